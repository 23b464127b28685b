mkdir -p gpurun_out
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s2j_c2.log 2>&1
FGB200_LIB=build/dbg/libfgb200.so timeout 300 python scripts/host_rate.py > gpurun_out/s2j_norecent.log 2>&1
FGB200_BLOCK_OVERLAP=0 timeout 300 python scripts/host_rate.py > gpurun_out/s2j_nooverlap.log 2>&1
FGB200_TRACE=gpurun_out/s2j_trace.txt timeout 300 python scripts/host_rate.py > gpurun_out/s2j_tr.log 2>&1
