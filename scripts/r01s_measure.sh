#!/bin/bash
# Round-1 final measurement pass on one B200 (gpurun, from the repo root).
# Bench lines, ncu launch lists and full captures -> gpurun_out/r01s/.
O=gpurun_out/r01s
mkdir -p $O
timeout 1800 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > $O/bench_default.log 2>&1; echo default=$?
timeout 900 python bench.py --impl reference > $O/bench_ref.log 2>&1; echo ref=$?
for c in c1 c3-full c3-short c3-adaptive c4-full c4-adaptive c5; do
  timeout 600 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_$c.log 2>&1; echo $c=$?
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
P2="python scripts/profile_run.py --config c2"
$P2 > $O/p2.log 2>&1
timeout 1200 ncu --metrics $M --clock-control none --csv --log-file $O/c2_launches.csv $P2 > $O/ncu_l2.log 2>&1; echo l2=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fg_block_item8_kernel -s 140 -c 1 \
  -o $O/c2_item8 $P2 > $O/ncu_f1.log 2>&1; echo f1=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fg_step_kernel -s 4000 -c 1 \
  -o $O/c2_step $P2 > $O/ncu_f2.log 2>&1; echo f2=$?
P5="python scripts/profile_run.py --config c5 --steps 1536"
$P5 > $O/p5.log 2>&1
timeout 1200 ncu --metrics $M --clock-control none --csv --log-file $O/c5_launches.csv $P5 > $O/ncu_l5.log 2>&1; echo l5=$?
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:fg_block_item_kernel<.int.128, .int.8' -s 6 -c 1 \
  -o $O/c5_item16 $P5 > $O/ncu_f3.log 2>&1; echo f3=$?
