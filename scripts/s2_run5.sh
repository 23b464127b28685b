mkdir -p gpurun_out
FGB200_TRACE=gpurun_out/c2_trace.txt timeout 300 python scripts/profile_run.py --config c2 > gpurun_out/c2_prof.log 2>&1
FGB200_TRACE=gpurun_out/c5_trace2.txt timeout 300 python scripts/profile_run.py --config c5 > gpurun_out/c5_prof2.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s2e_c2.log 2>&1
timeout 600 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s2e_c5.log 2>&1
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_parity.py -q -x -k "block or wide or batch or ensemble" > gpurun_out/s2e_tests.log 2>&1; echo tests=$?
