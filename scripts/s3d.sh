mkdir -p gpurun_out
for c in c3-full c4-full c3-short c2 c1; do
timeout 300 python bench.py --config $c --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/s3d_$c.log 2>&1
done
FGB200_BLOCK_TP=224 timeout 300 python bench.py --config c3-short --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/s3d_short224.log 2>&1
FGB200_BLOCK_TP=128 FGB200_BLOCK_CTAS_PER_SM=3 timeout 300 python bench.py --config c4-full --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/s3d_c4f_128_3.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_block.py -q -x > gpurun_out/s3d_tests.log 2>&1; echo tests=$?
