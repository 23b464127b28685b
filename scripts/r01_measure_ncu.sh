mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
$B > gpurun_out/r1f_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -c 5420 --csv --log-file gpurun_out/r1f_c2_launches.csv $B > gpurun_out/r1f_ncu_l.log 2>&1; echo nl=$?
C="python scripts/profile_run.py --config c2"
$C > gpurun_out/r1f_p.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fg_block_item_kernel -s 160 -c 2 -o gpurun_out/r1f_c2_item $C > gpurun_out/r1f_ncu_1.log 2>&1; echo n1=$?
C3="python scripts/profile_run.py --config c3-full --steps 1600"
$C3 > gpurun_out/r1f_p3.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:fg_block_tma_kernel -s 90 -c 1 -o gpurun_out/r1f_c3f_dense $C3 > gpurun_out/r1f_ncu_4.log 2>&1; echo n4=$?
