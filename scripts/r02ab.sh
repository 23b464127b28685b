# pipe2 vs lean dense consumers, alternating, with clocks/throttle reasons logged around each run; c2 with evict_first recent loads vs the previous build
mkdir -p gpurun_out/r02ab
Q="nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv,noheader"
for rep in 1 2; do
for v in default pipe2; do
  if [ $v = default ]; then L=""; else L=paper_1004_5128_b200/_lib/variants/libfgb200_$v.so; fi
  for c in c4-full c3-full; do
    FGB200_LIB=$L timeout 600 python scripts/profile_run.py --config $c > gpurun_out/r02ab/run_${v}_$c.log 2>&1; echo $v $c rc=$? $(tail -1 gpurun_out/r02ab/run_${v}_$c.log) "| $($Q)"
  done
done
done
for v in default base; do
  if [ $v = default ]; then L=""; else L=paper_1004_5128_b200/_lib/variants/libfgb200_$v.so; fi
  FGB200_LIB=$L timeout 600 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02ab/bench_c2_$v.json 2>/dev/null; echo c2 $v $(python -c "import json;d=json.load(open('gpurun_out/r02ab/bench_c2_$v.json'));print(d['ms_per_step'], d['clocks'])")
done
