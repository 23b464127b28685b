# split tails: GPU suite, timelines of the blocked configs; dense-consumer microbenchmark
mkdir -p gpurun_out/r02p
./scripts/micro/dense_consumer > gpurun_out/r02p/dense_consumer.txt 2>&1; cat gpurun_out/r02p/dense_consumer.txt
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/r02p/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/r02p/pytest_gpu.log
for c in c4-adaptive c3-adaptive c5 c4-full c3-full c3-short; do
  FGB200_TRACE=gpurun_out/r02p/trace_$c.txt timeout 600 python scripts/profile_run.py --config $c > gpurun_out/r02p/run_$c.log 2>&1; echo $c rc=$? $(tail -1 gpurun_out/r02p/run_$c.log)
done
