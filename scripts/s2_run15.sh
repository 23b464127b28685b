mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -x -m gpu > gpurun_out/s2s_tests.log 2>&1; echo tests=$?
FGB200_TBLOCK=64 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s2s_c2_64.log 2>&1
FGB200_TBLOCK=128 timeout 300 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s2s_c5_128.log 2>&1
for cols in 8 16; do for tb in 64 128; do
  FGB200_ITEM_COLS=$cols FGB200_TBLOCK=$tb timeout 300 python bench.py --config c3-adaptive --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s2s_c3a_${cols}_$tb.log 2>&1
  FGB200_ITEM_COLS=$cols FGB200_TBLOCK=$tb timeout 300 python bench.py --config c4-adaptive --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s2s_c4a_${cols}_$tb.log 2>&1
done; done
FGB200_ITEM_COLS=16 FGB200_TBLOCK=128 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s2s_c2_16_128.log 2>&1
