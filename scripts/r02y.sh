# c4-full/c3-full: step kernel at 40 registers (a step CTA fits beside two dense block CTAs) + 5-stage dense ring
mkdir -p gpurun_out/r02y
for v in default ring5 s40k3 s40k2; do
  if [ $v = default ]; then L=""; else L=paper_1004_5128_b200/_lib/variants/libfgb200_$v.so; fi
  for c in c4-full c3-full; do
    FGB200_LIB=$L FGB200_TRACE=gpurun_out/r02y/trace_${v}_$c.txt timeout 600 python scripts/profile_run.py --config $c > gpurun_out/r02y/run_${v}_$c.log 2>&1; echo $v $c rc=$? $(tail -1 gpurun_out/r02y/run_${v}_$c.log)
  done
done
FGB200_LIB=paper_1004_5128_b200/_lib/variants/libfgb200_s40k3.so timeout 900 python -m pytest -q -x tests/test_gpu_configs.py -k "c4_prefix or c3_prefix" > gpurun_out/r02y/pytest_cfg.log 2>&1; echo pytest_cfg=$?; tail -1 gpurun_out/r02y/pytest_cfg.log
