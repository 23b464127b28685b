# sub-block delay D (sub-block i feeds steps >= (i+1)S + D): parity with D = 7, 14; timings D = S / 14 / 7
mkdir -p gpurun_out/r02ag
for d in 7 14; do
  FGB200_SUBDELAY=$d timeout 900 python -m pytest -q -x tests/test_gpu_parity.py -k "subblock" > gpurun_out/r02ag/pytest_d$d.log 2>&1; echo pytest d=$d rc=$?; tail -1 gpurun_out/r02ag/pytest_d$d.log
done
FGB200_SUBDELAY=7 FGB200_PARITY_LOG=gpurun_out/r02ag/parity.jsonl timeout 900 python -m pytest -q -x tests/test_gpu_configs.py -k "c4_prefix and adaptive" > gpurun_out/r02ag/pytest_cfg.log 2>&1; echo cfg rc=$?; cat gpurun_out/r02ag/parity.jsonl
for rep in 1 2; do
for d in 0 14 7 4; do
  for c in c4-adaptive c3-adaptive c5 c4-full; do
    FGB200_SUBDELAY=$d timeout 600 python scripts/profile_run.py --config $c > gpurun_out/r02ag/run.log 2>&1; echo d=$d $c rc=$? $(tail -1 gpurun_out/r02ag/run.log | cut -c1-45)
  done
done
done
