#!/bin/bash
# Round-1 measurement pass on one B200 (run through gpurun from the repo root).
# Bench lines -> gpurun_out/r1f_*.log, ncu launch list + full captures -> gpurun_out/r1f_*.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1f_smoke.log 2>&1; echo smoke=$?
python bench.py > gpurun_out/r1f_default.log 2>&1; echo default=$?
python bench.py --impl reference > gpurun_out/r1f_ref.log 2>&1; echo ref=$?
for c in c1 c3-full c3-short c3-adaptive c4-full c4-adaptive c5; do
  timeout 600 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r1f_$c.log 2>&1; echo $c=$?
done
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
$B > gpurun_out/r1f_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -c 6000 --csv --log-file gpurun_out/r1f_c2_launches.csv $B > gpurun_out/r1f_ncu_l.log 2>&1; echo nl=$?
C="python scripts/profile_run.py --config c2"
$C > gpurun_out/r1f_p.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:fg_block_item_kernel<224, 6>' -s 80 -c 1 -o gpurun_out/r1f_c2_item $C > gpurun_out/r1f_ncu_1.log 2>&1; echo n1=$?
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:fg_block_item_kernel<224, 2>' -s 80 -c 1 -o gpurun_out/r1f_c2_tail $C > gpurun_out/r1f_ncu_2.log 2>&1; echo n2=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fg_step -s 4000 -c 1 \
  -o gpurun_out/r1f_c2_step $C > gpurun_out/r1f_ncu_3.log 2>&1; echo n3=$?
C3="python scripts/profile_run.py --config c3-full --steps 1600"
$C3 > gpurun_out/r1f_p3.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on \
  --kernel-name-base demangled -k 'regex:fg_block_tma_kernel<32, \d+, true, 6>' -s 45 -c 1 \
  -o gpurun_out/r1f_c3f_dense $C3 > gpurun_out/r1f_ncu_4.log 2>&1; echo n4=$?
