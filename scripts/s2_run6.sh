mkdir -p gpurun_out
for tb in 48 64; do
  FGB200_TBLOCK=$tb timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s2f_c2_$tb.log 2>&1
  FGB200_TBLOCK=$tb timeout 300 python bench.py --config c3-adaptive --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s2f_c3a_$tb.log 2>&1
done
