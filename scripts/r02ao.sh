# dense stages of 16 slices (3-stage ring, k-step loop not unrolled) vs 8 (default)
mkdir -p gpurun_out/r02ao
for rep in 1 2; do
for v in default ke16u1 ke8u1; do
  if [ $v = default ]; then L=""; else L=paper_1004_5128_b200/_lib/variants/libfgb200_$v.so; fi
  for c in c4-full c3-full; do
    FGB200_LIB=$L timeout 600 python scripts/profile_run.py --config $c > gpurun_out/r02ao/run.log 2>&1; echo $v $c rc=$? $(tail -1 gpurun_out/r02ao/run.log | cut -c1-45)
  done
done
done
