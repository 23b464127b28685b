# 16-slice dense stages as default: dense parity, timings vs HEAD (8-slice stages), 3 reps; ncu of a mid-run main launch
mkdir -p gpurun_out/r02ap
timeout 900 python -m pytest -q -x tests/test_gpu_block.py tests/test_gpu_parity.py -k "block or temporal or subblock or modes" > gpurun_out/r02ap/pytest_dense.log 2>&1; echo pytest=$?; tail -1 gpurun_out/r02ap/pytest_dense.log
timeout 900 python -m pytest -q -x tests/test_gpu_configs.py -k "full or short" > gpurun_out/r02ap/pytest_cfg.log 2>&1; echo pytest_cfg=$?; tail -1 gpurun_out/r02ap/pytest_cfg.log
for rep in 1 2 3; do
for v in default head; do
  if [ $v = default ]; then L=""; else L=paper_1004_5128_b200/_lib/variants/libfgb200_$v.so; fi
  for c in c4-full c3-full c3-short; do
    FGB200_LIB=$L timeout 600 python scripts/profile_run.py --config $c > gpurun_out/r02ap/run.log 2>&1; echo $v $c rc=$? $(tail -1 gpurun_out/r02ap/run.log | cut -c1-45)
  done
done
done
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:tma_kernel<.*\(int\)3, \(int\)32>' -s 40 -c 1 -o gpurun_out/r02ap/c4f_ke16_main python scripts/profile_run.py --config c4-full --steps 1600 > gpurun_out/r02ap/ncu.log 2>&1; echo ncu=$?
