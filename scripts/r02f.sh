# dense kernel: deferred release + shared-address loads; item ncu after the release change
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r02f_pytest.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/r02f_pytest.log
for c in c4-full c3-full c3-short; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02f_$c.json 2> gpurun_out/r02f_$c.err; echo $c rc=$?
  python -c "import json,sys; d=json.loads(open('gpurun_out/r02f_$c.json').read().strip().splitlines()[-1]); x=d['roofline']['runs'][0]; print('$c', d['ms_per_step'], d['value']/1e12, x['block_stage']['hbm_frac'], x['block_stage']['fp64_frac'], x['block_stage']['total_ms'])"
done
python scripts/profile_run.py --config c3-adaptive --steps 1200 > gpurun_out/r02f_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fg_block_item_kernel -s 30 -c 4 -o gpurun_out/r02f_c3a_item16 python scripts/profile_run.py --config c3-adaptive --steps 1200 > gpurun_out/r02f_ncu.log 2>&1; echo ncu_rc=$?
