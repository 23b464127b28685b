# item tail/sub-block launches with 3 or 4 stages (critical-path tail vs its ring depth)
mkdir -p gpurun_out/r02al
for rep in 1 2; do
for v in default ts3 ts4; do
  if [ $v = default ]; then L=""; else L=paper_1004_5128_b200/_lib/variants/libfgb200_$v.so; fi
  for c in c4-adaptive c3-adaptive c5; do
    FGB200_LIB=$L FGB200_TRACE=gpurun_out/r02al/trace_${v}_$c.txt timeout 600 python scripts/profile_run.py --config $c > gpurun_out/r02al/run.log 2>&1; echo $v $c rc=$? $(tail -1 gpurun_out/r02al/run.log | cut -c1-45)
  done
done
done
