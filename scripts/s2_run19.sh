mkdir -p gpurun_out
for per in 1 2; do
for c in c5 c3-adaptive c2; do
  FGB200_BLOCK_CTAS_PER_SM=$per timeout 300 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s2w_${c}_$per.log 2>&1
done; done
