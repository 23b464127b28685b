mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "subblock" > gpurun_out/s2z_tests.log 2>&1; echo tests=$?
for sb in 16 8 32 0; do
  FGB200_SUBBLOCK=$sb timeout 300 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s2z_c5_$sb.log 2>&1
  FGB200_SUBBLOCK=$sb timeout 300 python bench.py --config c3-adaptive --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s2z_c3a_$sb.log 2>&1
done
FGB200_SUBBLOCK=16 FGB200_TRACE=gpurun_out/s2z_trace_c5.txt timeout 300 python scripts/profile_run.py --config c5 > gpurun_out/s2z_c5p.log 2>&1
