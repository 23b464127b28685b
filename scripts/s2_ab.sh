# A/B: current tree vs build/ab_head (HEAD of the branch), c2 bench alternated; c5 trace
mkdir -p gpurun_out
for i in 1 2; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_new_$i.log 2>&1
  (cd build/ab_head && timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > ../../gpurun_out/ab_head_$i.log 2>&1)
done
FGB200_TRACE=gpurun_out/c5_trace.txt timeout 300 python scripts/profile_run.py --config c5 > gpurun_out/c5_prof.log 2>&1
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_parity.py -q -x -k "block or wide or batch or ensemble" > gpurun_out/ab_tests.log 2>&1; echo tests=$?
