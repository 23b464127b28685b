# DMMA parallelism sweep; full GPU suite on the pruned library; c1/c2 timing
./scripts/micro/dmma_sweep > gpurun_out/r02g_dmma_sweep.txt 2>&1; echo sweep_rc=$?
cat gpurun_out/r02g_dmma_sweep.txt
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r02g_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r02g_pytest.log
for c in c1 c2; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02g_$c.json 2> gpurun_out/r02g_$c.err; echo $c rc=$?
  python -c "import json,sys; d=json.loads(open('gpurun_out/r02g_$c.json').read().strip().splitlines()[-1]); print('$c', d['ms_per_step'], d['value']/1e12)"
done
