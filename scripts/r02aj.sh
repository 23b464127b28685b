# item kernel: release without an fp64 add (default) vs HEAD; main-ring depth 3/5/6 stages of 16 slices
mkdir -p gpurun_out/r02aj
for rep in 1 2; do
for v in default head is3 is5 is6; do
  if [ $v = default ]; then L=""; else L=paper_1004_5128_b200/_lib/variants/libfgb200_$v.so; fi
  for c in c4-adaptive c3-adaptive c5; do
    FGB200_LIB=$L timeout 600 python scripts/profile_run.py --config $c > gpurun_out/r02aj/run.log 2>&1; echo $v $c rc=$? $(tail -1 gpurun_out/r02aj/run.log | cut -c1-45)
  done
done
done
