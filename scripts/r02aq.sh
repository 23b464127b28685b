# dense stages of 24 slices (2-stage ring) vs 16 (default)
mkdir -p gpurun_out/r02aq
for rep in 1 2 3; do
for v in default ke24; do
  if [ $v = default ]; then L=""; else L=paper_1004_5128_b200/_lib/variants/libfgb200_$v.so; fi
  for c in c4-full c3-full; do
    FGB200_LIB=$L timeout 600 python scripts/profile_run.py --config $c > gpurun_out/r02aq/run.log 2>&1; echo $v $c rc=$? $(tail -1 gpurun_out/r02aq/run.log | cut -c1-45)
  done
done
done
