mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_block.py -x -q -k ensemble > gpurun_out/s2b_block.log 2>&1; echo block=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "wide or blocking or batch" > gpurun_out/s2b_parity.log 2>&1; echo parity=$?
for tb in 24 32 48 64; do
  FGB200_TBLOCK=$tb timeout 600 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s2b_c5_$tb.log 2>&1; echo c5_$tb=$?
done
