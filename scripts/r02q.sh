# dense block kernel with 16-point consumer warps (TP 128, 16 consumer warps per SM) vs 32-point warps (TP 224)
mkdir -p gpurun_out/r02q
export FGB200_LIB=paper_1004_5128_b200/_lib/variants/libfgb200_wp16.so
timeout 900 python -m pytest -q -x tests/test_gpu_block.py tests/test_gpu_parity.py -k "block or temporal" > gpurun_out/r02q/pytest_dense.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r02q/pytest_dense.log
for c in c4-full c3-full c3-short; do
  FGB200_TRACE=gpurun_out/r02q/trace_wp16_$c.txt timeout 600 python scripts/profile_run.py --config $c > gpurun_out/r02q/run_wp16_$c.log 2>&1; echo wp16 $c rc=$? $(tail -1 gpurun_out/r02q/run_wp16_$c.log)
done
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:tma_kernel<.*\(int\)6, \(int\)16>' -s 40 -c 1 -o gpurun_out/r02q/c4f_wp16_main python scripts/profile_run.py --config c4-full --steps 1600 > gpurun_out/r02q/ncu.log 2>&1; echo ncu=$?
unset FGB200_LIB
for c in c4-full c3-full; do
  timeout 600 python scripts/profile_run.py --config $c > gpurun_out/r02q/run_base_$c.log 2>&1; echo base $c rc=$? $(tail -1 gpurun_out/r02q/run_base_$c.log)
done
