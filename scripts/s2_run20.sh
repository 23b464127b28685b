mkdir -p gpurun_out
FGB200_LIB=build/dbg/libfgb200.so FGB200_TRACE=gpurun_out/s2x_trace_c5.txt timeout 300 python scripts/profile_run.py --config c5 > gpurun_out/s2x_c5.log 2>&1
FGB200_LIB=build/dbg/libfgb200.so FGB200_TRACE=gpurun_out/s2x_trace_c3a.txt timeout 300 python scripts/profile_run.py --config c3-adaptive > gpurun_out/s2x_c3a.log 2>&1
