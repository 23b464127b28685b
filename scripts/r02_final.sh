#!/bin/bash
# Round-2 final measurement pass on one B200 (gpurun, from the repo root): GPU suite with the
# config-scale parity log, smoke, default bench (c4) + reference arm, every other config, launch list.
O=${OUT:-gpurun_out/r02f}
mkdir -p $O
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > $O/gpu.txt; nproc >> $O/gpu.txt; free -g >> $O/gpu.txt
FGB200_PARITY_LOG=$O/parity.jsonl timeout 2400 python -m pytest tests -q -m gpu -rs > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; echo bench=$?
timeout 900 python bench.py --impl reference > $O/bench_ref_c4.json 2> $O/bench_ref_c4.err; echo ref=$?
for c in c1 c2 c3 c5; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo $c=$?
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_c4.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo launches=$?
