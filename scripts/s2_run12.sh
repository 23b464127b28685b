mkdir -p gpurun_out
for v in dbg dbg2; do
FGB200_RUN_FLAGS=34 FGB200_BLOCK_OVERLAP=0 FGB200_LIB=build/$v/libfgb200.so FGB200_TRACE=gpurun_out/s2n_trace_$v.txt timeout 120 python scripts/host_rate.py > gpurun_out/s2n_$v.log 2>&1
done
FGB200_RUN_FLAGS=34 FGB200_TRACE=gpurun_out/s2n_trace_full.txt timeout 120 python scripts/host_rate.py > gpurun_out/s2n_full.log 2>&1
