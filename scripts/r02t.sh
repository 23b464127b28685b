# dense block kernel, lean fragments + TP 256 (8 consumer warps per CTA, 16 per SM) vs default; parity of the lean build
mkdir -p gpurun_out/r02t
export FGB200_LIB=paper_1004_5128_b200/_lib/variants/libfgb200_lean.so
timeout 900 python -m pytest -q -x tests/test_gpu_block.py tests/test_gpu_parity.py -k "block or temporal" > gpurun_out/r02t/pytest_dense.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r02t/pytest_dense.log
timeout 900 python -m pytest -q -x tests/test_gpu_configs.py -k "c3_prefix or c4_prefix" > gpurun_out/r02t/pytest_cfg.log 2>&1; echo pytest_cfg=$?; tail -2 gpurun_out/r02t/pytest_cfg.log
for c in c4-full c3-full c3-short; do
  FGB200_TRACE=gpurun_out/r02t/trace_lean_$c.txt timeout 600 python scripts/profile_run.py --config $c > gpurun_out/r02t/run_lean_$c.log 2>&1; echo lean $c rc=$? $(tail -1 gpurun_out/r02t/run_lean_$c.log)
done
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:tma_kernel<.*\(int\)6, \(int\)32>' -s 40 -c 1 -o gpurun_out/r02t/c4f_lean_main python scripts/profile_run.py --config c4-full --steps 1600 > gpurun_out/r02t/ncu.log 2>&1; echo ncu=$?
unset FGB200_LIB
for c in c4-full c3-full c3-short; do
  timeout 600 python scripts/profile_run.py --config $c > gpurun_out/r02t/run_base_$c.log 2>&1; echo base $c rc=$? $(tail -1 gpurun_out/r02t/run_base_$c.log)
done
