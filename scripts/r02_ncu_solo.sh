# ncu --set full capture of one mid-run dense main launch (solo kernel) of c4-full: block kb0=1344.
O=${OUT:-gpurun_out/r02m}
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fg_block_tma_solo_kernel -s 40 -c 1 \
  -o $O/c4f_solo python scripts/profile_run.py --config c4-full --steps 1600 > $O/ncu_c4f_solo.log 2>&1; echo ncu_solo=$?
