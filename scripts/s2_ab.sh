# A/B: current tree vs build/ab_head (HEAD of the branch)
mkdir -p gpurun_out
for i in 1 2; do
  for c in c2 c5 c3-adaptive; do
  timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ab_new_${c}_$i.log 2>&1
  (cd build/ab_head && timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > ../../gpurun_out/ab_head_${c}_$i.log 2>&1)
  done
done
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_parity.py -q -x > gpurun_out/ab_tests.log 2>&1; echo tests=$?
