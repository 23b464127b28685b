# item kernel: deferred release + shared-address loads
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_parity.py -x -q -m gpu -k "block or wide or item or subblock or ensemble" > gpurun_out/r02e_pytest.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/r02e_pytest.log
for c in c3-adaptive c5 c4-adaptive; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02e_$c.json 2> gpurun_out/r02e_$c.err; echo $c rc=$?
  python -c "import json,sys; d=json.loads(open('gpurun_out/r02e_$c.json').read().strip().splitlines()[-1]); x=d['roofline']['runs'][0]; print('$c', d['ms_per_step'], d['value']/1e12, x['block_stage']['hbm_frac'], x['block_stage']['total_ms'])"
done
