# compute-sanitizer memcheck / racecheck / synccheck / initcheck over every launch
# mode on small golden cases (only the library's fg_* kernels are instrumented).
# usage: bash scripts/sanitize.sh <outdir> [tool ...]
OUT=${1:-gpurun_out/sanitize}; shift
TOOLS=${@:-memcheck racecheck synccheck initcheck}
mkdir -p $OUT
SEL="tests/test_gpu_parity.py::test_launch_modes_bitwise_identical \
 tests/test_gpu_parity.py::test_temporal_blocking_modes_bitwise \
 tests/test_gpu_parity.py::test_subblock_launch_modes_bitwise \
 tests/test_gpu_parity.py::test_cached_graph_replay \
 tests/test_gpu_parity.py::test_graph_replay_after_a_larger_plan \
 tests/test_gpu_parity.py::test_temporal_blocking_divergence"
EXTRA="tests/test_gpu_parity.py::test_fused_pairs_bitwise tests/test_gpu_parity.py::test_item_widths_match_goldens \
 tests/test_gpu_parity.py::test_subblock_launches_match_goldens"
KSEL="c2_small-32 or c1-16 or 1d_adaptive-64 or batch_adaptive or 3d_sat_adaptive or c2_small-8 or c2_small_full-4 or c2_small-28 or point_short100-4"
for tool in $TOOLS; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 2400 compute-sanitizer --tool $tool $extra --kernel-name regex:fg_ --print-limit 200 \
     --target-processes all --log-file $OUT/$tool.log \
     python -m pytest -q -p no:cacheprovider $SEL > $OUT/${tool}_pytest.log 2>&1
  echo "$tool modes rc=$?"; tail -2 $OUT/${tool}_pytest.log
  timeout 2400 compute-sanitizer --tool $tool $extra --kernel-name regex:fg_ --print-limit 200 \
     --target-processes all --log-file $OUT/${tool}_extra.log \
     python -m pytest -q -p no:cacheprovider $EXTRA -k "$KSEL" > $OUT/${tool}_extra_pytest.log 2>&1
  echo "$tool extra rc=$?"; tail -2 $OUT/${tool}_extra_pytest.log
  timeout 2400 compute-sanitizer --tool $tool $extra --kernel-name regex:fg_ --print-limit 200 \
     --target-processes all --log-file $OUT/${tool}_block.log \
     python -m pytest -q -p no:cacheprovider tests/test_gpu_block.py -k "shape2 or shape4 or shape5" > $OUT/${tool}_block_pytest.log 2>&1
  echo "$tool block rc=$?"; tail -2 $OUT/${tool}_block_pytest.log
  grep -c "ERROR SUMMARY\|Hazard\|Invalid" $OUT/$tool.log $OUT/${tool}_extra.log $OUT/${tool}_block.log
  grep "SUMMARY" $OUT/$tool.log $OUT/${tool}_extra.log $OUT/${tool}_block.log | sort | uniq -c
done
