# 32-column items at tblock 224 (single large adaptive fields): parity (goldens, config prefixes, c3-adaptive full length), timings vs 16-column items at 112
mkdir -p gpurun_out/r02ad
timeout 1500 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_block.py -k "block or temporal or item or subblock" > gpurun_out/r02ad/pytest_items.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r02ad/pytest_items.log
FGB200_PARITY_LOG=gpurun_out/r02ad/parity.jsonl timeout 1500 python -m pytest -q -x tests/test_gpu_configs.py -k "adaptive" > gpurun_out/r02ad/pytest_cfg.log 2>&1; echo pytest_cfg=$?; tail -2 gpurun_out/r02ad/pytest_cfg.log; cat gpurun_out/r02ad/parity.jsonl
for rep in 1 2; do
for c in c4-adaptive c3-adaptive; do
  FGB200_TRACE=gpurun_out/r02ad/trace_new_$c.txt timeout 600 python scripts/profile_run.py --config $c > gpurun_out/r02ad/run_new_$c.log 2>&1; echo new $c rc=$? $(tail -1 gpurun_out/r02ad/run_new_$c.log | cut -c1-50)
  FGB200_ITEM_COLS=16 FGB200_TBLOCK=112 timeout 600 python scripts/profile_run.py --config $c > gpurun_out/r02ad/run_w16_$c.log 2>&1; echo w16-112 $c rc=$? $(tail -1 gpurun_out/r02ad/run_w16_$c.log | cut -c1-50)
done
done
