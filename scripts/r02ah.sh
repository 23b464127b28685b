# sub-block delay defaults (adaptive S/4, full S/2): GPU suite; c3-short D sweep; timings
mkdir -p gpurun_out/r02ah
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/r02ah/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r02ah/pytest_gpu.log
for d in 0 1 2; do FGB200_SUBDELAY=$d timeout 600 python scripts/profile_run.py --config c3-short > gpurun_out/r02ah/run.log 2>&1; echo c3-short d=$d rc=$? $(tail -1 gpurun_out/r02ah/run.log | cut -c1-45); done
for c in c4-adaptive c3-adaptive c5 c4-full c3-full; do
  timeout 600 python scripts/profile_run.py --config $c > gpurun_out/r02ah/run.log 2>&1; echo default $c rc=$? $(tail -1 gpurun_out/r02ah/run.log | cut -c1-45)
done
