# dense consumers with fragments one k-step ahead (pipe2, 96 registers + spills) vs lean; GPU suite on the evict_first build
mkdir -p gpurun_out/r02aa
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/r02aa/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r02aa/pytest_gpu.log
for v in default pipe2; do
  if [ $v = default ]; then L=""; else L=paper_1004_5128_b200/_lib/variants/libfgb200_$v.so; fi
  for c in c4-full c3-full; do
    FGB200_LIB=$L timeout 600 python scripts/profile_run.py --config $c > gpurun_out/r02aa/run_${v}_$c.log 2>&1; echo $v $c rc=$? $(tail -1 gpurun_out/r02aa/run_${v}_$c.log)
  done
done
