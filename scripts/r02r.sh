# step-kernel L2 bulk prefetch (large fields) A/B; checked-build GPU suite
mkdir -p gpurun_out/r02r
for v in nopf default; do
  if [ $v = default ]; then L=""; else L=paper_1004_5128_b200/_lib/variants/libfgb200_$v.so; fi
  for c in c4-adaptive c3-adaptive c5 c4-full; do
    FGB200_LIB=$L FGB200_TRACE=gpurun_out/r02r/trace_${v}_$c.txt timeout 600 python scripts/profile_run.py --config $c > gpurun_out/r02r/run_${v}_$c.log 2>&1; echo $v $c rc=$? $(tail -1 gpurun_out/r02r/run_${v}_$c.log)
  done
done
bash scripts/checked_suite.sh gpurun_out/r02r/checked
