# checked-build GPU suite; c2 step-chain variants (loads in flight per round, no recent sum)
mkdir -p gpurun_out/r02s
bash scripts/checked_suite.sh gpurun_out/r02s/checked
for v in default kr9 kr17 norecent; do
  if [ $v = default ]; then L=""; else L=paper_1004_5128_b200/_lib/variants/libfgb200_$v.so; fi
  FGB200_LIB=$L timeout 600 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02s/bench_c2_$v.json 2> gpurun_out/r02s/bench_c2_$v.err
  echo $v rc=$? $(python -c "import json,sys;d=json.load(open('gpurun_out/r02s/bench_c2_$v.json'));print(d['ms_per_step'], d['roofline']['runs'][0].get('block_stage',{}).get('total_ms'))")
done
FGB200_TRACE=gpurun_out/r02s/trace_c2.txt timeout 600 python scripts/profile_run.py --config c2 > /dev/null 2>&1
