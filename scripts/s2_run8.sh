mkdir -p gpurun_out
for fl in 2 3 4 6; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --flags $fl > gpurun_out/s2h_c2_f$fl.log 2>&1
done
timeout 300 python bench.py --config c4-adaptive --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s2h_c4a.log 2>&1
