mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "modes_bitwise or divergence or chain" > gpurun_out/s2l_tests.log 2>&1; echo tests=$?
timeout 120 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --flags 34 > gpurun_out/s2l_c2_f34.log 2>&1; echo b34=$?
timeout 120 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --flags 2 > gpurun_out/s2l_c2_f2.log 2>&1; echo b2=$?
FGB200_RUN_FLAGS=34 FGB200_TRACE=gpurun_out/s2l_trace.txt timeout 120 python scripts/host_rate.py > gpurun_out/s2l_host.log 2>&1
