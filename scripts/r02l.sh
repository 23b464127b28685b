# block-pipeline timelines (FGB200_TRACE) of the large configs; ncu (full set + source) of mid-run MAIN launches
mkdir -p gpurun_out/r02l
for c in c4-full c4-adaptive c3-adaptive c3-full c5; do
  FGB200_TRACE=gpurun_out/r02l/trace_$c.txt timeout 600 python scripts/profile_run.py --config $c > gpurun_out/r02l/run_$c.log 2>&1; echo trace_$c=$?; tail -1 gpurun_out/r02l/run_$c.log
done
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:tma_kernel<32, 224, 1, 6" -s 60 -c 1 -o gpurun_out/r02l/c4f_dense_main python scripts/profile_run.py --config c4-full --steps 2000 > gpurun_out/r02l/ncu_dense.log 2>&1; echo ncu_dense=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:item_kernel<96, 4, 0" -s 15 -c 1 -o gpurun_out/r02l/c4a_item_main python scripts/profile_run.py --config c4-adaptive --steps 2100 > gpurun_out/r02l/ncu_c4a.log 2>&1; echo ncu_c4a=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:item_kernel<96, 4, 0" -s 15 -c 1 -o gpurun_out/r02l/c3a_item_main python scripts/profile_run.py --config c3-adaptive --steps 2100 > gpurun_out/r02l/ncu_c3a.log 2>&1; echo ncu_c3a=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:item_kernel<128, 4, 1" -s 40 -c 1 -o gpurun_out/r02l/c5_item_main python scripts/profile_run.py --config c5 --steps 6000 > gpurun_out/r02l/ncu_c5.log 2>&1; echo ncu_c5=$?
