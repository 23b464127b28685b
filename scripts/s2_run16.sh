mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -x -m gpu > gpurun_out/s2t_tests.log 2>&1; echo tests=$?
for c in c2 c1 c3-full c3-short c3-adaptive c4-full c4-adaptive c5; do
  timeout 600 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s2t_$c.log 2>&1; echo $c=$?
done
