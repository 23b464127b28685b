# recent-slice loads: newest offsets (m <= keep_m) evict_last, older evict_first, vs plain .cg loads (base)
mkdir -p gpurun_out/r02z
for v in default base keep0 keep3 keep9; do
  if [ $v = default ]; then L=""; else L=paper_1004_5128_b200/_lib/variants/libfgb200_$v.so; fi
  for c in c4-adaptive c3-adaptive c5 c4-full; do
    FGB200_LIB=$L timeout 600 python scripts/profile_run.py --config $c > gpurun_out/r02z/run_${v}_$c.log 2>&1; echo $v $c rc=$? $(tail -1 gpurun_out/r02z/run_${v}_$c.log)
  done
done
