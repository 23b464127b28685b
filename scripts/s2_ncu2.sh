mkdir -p gpurun_out
C="python scripts/profile_run.py --config c2"
$C > gpurun_out/s2q_p.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fg_block_item_kernel -s 120 -c 1 -o gpurun_out/s2q_item $C > gpurun_out/s2q_ncu.log 2>&1; echo n=$?
