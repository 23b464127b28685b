# L2 policy of P-row stores (evict_last vs normal above 32 MB of rows) and of δ^k stores (evict_last vs normal above 4 MB slices); c2 evict_first recent loads vs round-start build
mkdir -p gpurun_out/r02ac
Q="nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv,noheader"
for rep in 1 2; do
for v in default pk hk pkhk; do
  if [ $v = default ]; then L=""; else L=paper_1004_5128_b200/_lib/variants/libfgb200_$v.so; fi
  for c in c4-adaptive c3-adaptive c5 c4-full; do
    FGB200_LIB=$L timeout 600 python scripts/profile_run.py --config $c > gpurun_out/r02ac/run_${v}_$c.log 2>&1; echo $v $c rc=$? $(tail -1 gpurun_out/r02ac/run_${v}_$c.log | cut -c1-40) "| $($Q)"
  done
done
done
for v in default head; do
  if [ $v = default ]; then L=""; else L=paper_1004_5128_b200/_lib/variants/libfgb200_$v.so; fi
  FGB200_LIB=$L timeout 600 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02ac/bench_c2_$v.json 2>/dev/null; echo c2 $v $(python -c "import json;d=json.load(open('gpurun_out/r02ac/bench_c2_$v.json'));print(d['ms_per_step'], d['clocks'])")
done
