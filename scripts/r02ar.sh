# dense producer: the warp's lanes issue a stage's row copies in parallel vs lane 0 alone
mkdir -p gpurun_out/r02ar
timeout 900 env FGB200_LIB=paper_1004_5128_b200/_lib/variants/libfgb200_pprod.so python -m pytest -q -x tests/test_gpu_block.py > gpurun_out/r02ar/pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/r02ar/pytest.log
for rep in 1 2 3; do
for v in default pprod; do
  if [ $v = default ]; then L=""; else L=paper_1004_5128_b200/_lib/variants/libfgb200_$v.so; fi
  for c in c4-full c3-full; do
    FGB200_LIB=$L timeout 600 python scripts/profile_run.py --config $c > gpurun_out/r02ar/run.log 2>&1; echo $v $c rc=$? $(tail -1 gpurun_out/r02ar/run.log | cut -c1-45)
  done
done
done
