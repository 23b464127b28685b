# A/B: current tree vs build/ab_head (HEAD of the branch): c2 bench alternated + host enqueue rate
mkdir -p gpurun_out
for i in 1 2; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_new_$i.log 2>&1
  (cd build/ab_head && timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > ../../gpurun_out/ab_head_$i.log 2>&1)
done
python scripts/host_rate.py > gpurun_out/ab_host_new.log 2>&1
(cd build/ab_head && python scripts/host_rate.py > ../../gpurun_out/ab_host_head.log 2>&1)
