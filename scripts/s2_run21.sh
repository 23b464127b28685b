mkdir -p gpurun_out
for tp in 112 96 128; do
  FGB200_ITEM_TP=$tp timeout 300 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s2y_c5_$tp.log 2>&1
done
