# dense block kernel: main-launch times with the bulk copies removed (consumer + ring ceiling) vs real
mkdir -p gpurun_out/r02ae
FGB200_LIB=paper_1004_5128_b200/_lib/variants/libfgb200_nocopy.so FGB200_TRACE=gpurun_out/r02ae/trace_nocopy.txt timeout 600 python scripts/profile_run.py --config c4-full --steps 2000 > gpurun_out/r02ae/run_nocopy.log 2>&1; echo nocopy=$?; tail -1 gpurun_out/r02ae/run_nocopy.log
FGB200_TRACE=gpurun_out/r02ae/trace_base.txt timeout 600 python scripts/profile_run.py --config c4-full --steps 2000 > gpurun_out/r02ae/run_base.log 2>&1; echo base=$?; tail -1 gpurun_out/r02ae/run_base.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:tma_kernel<.*\(int\)6, \(int\)32>' -s 40 -c 1 -o gpurun_out/r02ae/nocopy_main env FGB200_LIB=paper_1004_5128_b200/_lib/variants/libfgb200_nocopy.so python scripts/profile_run.py --config c4-full --steps 1600 > gpurun_out/r02ae/ncu.log 2>&1; echo ncu=$?
