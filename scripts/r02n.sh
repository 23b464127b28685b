# dense block kernel: ncu of a mid-run main launch (c4-full); main-launch time with an L2-resident slice window (consumer ceiling)
mkdir -p gpurun_out/r02n
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:tma_kernel<.*\(int\)6>' -s 40 -c 1 -o gpurun_out/r02n/c4f_dense_main python scripts/profile_run.py --config c4-full --steps 1600 > gpurun_out/r02n/ncu_dense.log 2>&1; echo ncu_dense=$?
FGB200_LIB=paper_1004_5128_b200/_lib/variants/libfgb200_wrap4.so FGB200_TRACE=gpurun_out/r02n/trace_wrap4.txt timeout 600 python scripts/profile_run.py --config c4-full --steps 2000 > gpurun_out/r02n/run_wrap4.log 2>&1; echo wrap=$?; tail -2 gpurun_out/r02n/run_wrap4.log
FGB200_TRACE=gpurun_out/r02n/trace_base.txt timeout 600 python scripts/profile_run.py --config c4-full --steps 2000 > gpurun_out/r02n/run_base.log 2>&1; echo base=$?; tail -1 gpurun_out/r02n/run_base.log
