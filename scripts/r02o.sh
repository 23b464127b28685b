# dense block kernel A/B: tensor box (d1x) x k-step pipeline (dx1); parity of the default build first
mkdir -p gpurun_out/r02o
timeout 900 python -m pytest -q -x tests/test_gpu_block.py tests/test_gpu_parity.py -k "block or temporal" > gpurun_out/r02o/pytest_dense.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r02o/pytest_dense.log
timeout 900 python -m pytest -q -x tests/test_gpu_configs.py -k "c3_prefix or c4_prefix" > gpurun_out/r02o/pytest_cfg.log 2>&1; echo pytest_cfg=$?; tail -2 gpurun_out/r02o/pytest_cfg.log
for v in d00 d10 d01 default; do
  if [ $v = default ]; then L=""; else L=paper_1004_5128_b200/_lib/variants/libfgb200_$v.so; fi
  for c in c4-full c3-full; do
    FGB200_LIB=$L FGB200_TRACE=gpurun_out/r02o/trace_${v}_$c.txt timeout 600 python scripts/profile_run.py --config $c > gpurun_out/r02o/run_${v}_$c.log 2>&1; echo $v $c rc=$? $(tail -1 gpurun_out/r02o/run_${v}_$c.log)
  done
done
