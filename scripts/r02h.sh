# item kernel: 16-row stages (default) vs 8-row stages (variant)
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_parity.py -x -q -m gpu -k "block or wide or item or subblock or ensemble or graph" > gpurun_out/r02h_pytest.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/r02h_pytest.log
for lib in default ir8; do
  if [ $lib = ir8 ]; then export FGB200_LIB=paper_1004_5128_b200/_lib/variants/libfgb200_ir8.so; else unset FGB200_LIB; fi
  for c in c3-adaptive c5 c4-adaptive; do
    timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02h_${lib}_$c.json 2> gpurun_out/r02h_${lib}_$c.err; echo $lib $c rc=$?
    python -c "import json,sys; d=json.loads(open('gpurun_out/r02h_${lib}_$c.json').read().strip().splitlines()[-1]); x=d['roofline']['runs'][0]; print('$lib $c', d['ms_per_step'], d['value']/1e12, x['block_stage']['hbm_frac'], x['block_stage']['total_ms'])"
  done
done
