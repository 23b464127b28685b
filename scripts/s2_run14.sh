mkdir -p gpurun_out
for tb in 64 96 128; do
  FGB200_TBLOCK=$tb timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s2r_c2_$tb.log 2>&1
  FGB200_TBLOCK=$tb timeout 300 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s2r_c5_$tb.log 2>&1
done
timeout 300 python -m pytest tests/test_gpu_block.py -q -x > gpurun_out/s2r_tests.log 2>&1; echo tests=$?
