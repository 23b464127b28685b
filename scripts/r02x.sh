# 16-column items: quarter-depth boxes too (short last stages read rows rounded up to 4) vs half-depth only
mkdir -p gpurun_out/r02x
timeout 900 python -m pytest -q -x tests/test_gpu_block.py tests/test_gpu_parity.py tests/test_gpu_configs.py -k "block or temporal or item or subblock or adaptive or c5" > gpurun_out/r02x/pytest_items.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r02x/pytest_items.log
for rep in 1 2; do
for v in default base; do
  if [ $v = default ]; then L=""; else L=paper_1004_5128_b200/_lib/variants/libfgb200_$v.so; fi
  for c in c4-adaptive c3-adaptive c5; do
    FGB200_LIB=$L timeout 600 python scripts/profile_run.py --config $c > gpurun_out/r02x/run_${v}_$c.log 2>&1; echo $v $c rc=$? $(tail -1 gpurun_out/r02x/run_${v}_$c.log)
  done
done
done
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:item_kernel<\(int\)96, \(int\)4, \(bool\)0>' -s 15 -c 1 -o gpurun_out/r02x/c4a_item_main python scripts/profile_run.py --config c4-adaptive --steps 2100 > gpurun_out/r02x/ncu_c4a.log 2>&1; echo ncu_c4a=$?
