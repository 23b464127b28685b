O=gpurun_out/r01s; mkdir -p $O
P5="python scripts/profile_run.py --config c5 --steps 1536"
$P5 > $O/p5b.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:fg_block_item_kernel<.int.128, .int.8' -s 6 -c 1 -o $O/c5_item16_main $P5 > $O/ncu_f4.log 2>&1; echo f4=$?
