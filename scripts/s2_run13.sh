mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_parity.py -q -x > gpurun_out/s2o_tests.log 2>&1; echo tests=$?
for tb in 64 96 128; do
  FGB200_TBLOCK=$tb timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s2o_c2_$tb.log 2>&1
  FGB200_TBLOCK=$tb timeout 300 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s2o_c5_$tb.log 2>&1
  FGB200_TBLOCK=$tb timeout 300 python bench.py --config c3-adaptive --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s2o_c3a_$tb.log 2>&1
done
