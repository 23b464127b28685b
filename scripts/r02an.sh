# dense tail launches: ring depth 2 (default) / 3 / 4 / 6
mkdir -p gpurun_out/r02an
for rep in 1 2; do
for v in default dt3 dt4 dt6; do
  if [ $v = default ]; then L=""; else L=paper_1004_5128_b200/_lib/variants/libfgb200_$v.so; fi
  for c in c4-full c3-full c3-short; do
    FGB200_LIB=$L FGB200_TRACE=gpurun_out/r02an/trace_${v}_$c.txt timeout 600 python scripts/profile_run.py --config $c > gpurun_out/r02an/run.log 2>&1; echo $v $c rc=$? $(tail -1 gpurun_out/r02an/run.log | cut -c1-45)
  done
done
done
