mkdir -p gpurun_out
C3="python scripts/profile_run.py --config c3-full --steps 1600"
$C3 > gpurun_out/s2k_p3.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:fg_block_tma_kernel -s 90 -c 1 -o gpurun_out/s2k_c3f_dense $C3 > gpurun_out/s2k_ncu.log 2>&1; echo n=$?
