mkdir -p gpurun_out
for c in c5 c3-adaptive c4-adaptive; do
FGB200_TRACE=gpurun_out/s2v_trace_$c.txt timeout 300 python scripts/profile_run.py --config $c > gpurun_out/s2v_$c.log 2>&1
done
