# dense kernel with the producer inside consumer warp 0 (8-warp CTAs, 96 registers: a step CTA fits beside two) vs producer warp
mkdir -p gpurun_out/r02v
timeout 900 python -m pytest -q -x tests/test_gpu_block.py tests/test_gpu_parity.py -k "block or temporal" > gpurun_out/r02v/pytest_dense.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r02v/pytest_dense.log
timeout 900 python -m pytest -q -x tests/test_gpu_configs.py -k "c3_prefix or c4_prefix" > gpurun_out/r02v/pytest_cfg.log 2>&1; echo pytest_cfg=$?; tail -2 gpurun_out/r02v/pytest_cfg.log
for v in default inl6 noinl; do
  if [ $v = default ]; then L=""; else L=paper_1004_5128_b200/_lib/variants/libfgb200_$v.so; fi
  for c in c4-full c3-full c3-short; do
    FGB200_LIB=$L FGB200_TRACE=gpurun_out/r02v/trace_${v}_$c.txt timeout 600 python scripts/profile_run.py --config $c > gpurun_out/r02v/run_${v}_$c.log 2>&1; echo $v $c rc=$? $(tail -1 gpurun_out/r02v/run_${v}_$c.log)
  done
done
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:tma_kernel<.*\(int\)5, \(int\)32>' -s 40 -c 1 -o gpurun_out/r02v/c4f_inl_main python scripts/profile_run.py --config c4-full --steps 1600 > gpurun_out/r02v/ncu.log 2>&1; echo ncu=$?
