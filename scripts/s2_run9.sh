mkdir -p gpurun_out
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s2i_c2_f2.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --flags 3 > gpurun_out/s2i_c2_f3.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --flags 1 > gpurun_out/s2i_c2_f1.log 2>&1
FGB200_RUN_FLAGS=3 python scripts/host_rate.py > gpurun_out/s2i_host3.log 2>&1
