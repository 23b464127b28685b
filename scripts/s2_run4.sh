mkdir -p gpurun_out
python scripts/debug_ens.py > gpurun_out/s2d_dbg.log 2>&1
timeout 900 python -m pytest tests/test_gpu_block.py -q > gpurun_out/s2d_block.log 2>&1; echo block=$?
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q > gpurun_out/s2d_parity.log 2>&1; echo parity=$?
for tb in 48 64; do
  FGB200_TBLOCK=$tb timeout 600 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s2d_c5_$tb.log 2>&1; echo c5_$tb=$?
done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s2d_c2.log 2>&1; echo c2=$?
