mkdir -p gpurun_out
python scripts/debug_ens.py > gpurun_out/s2c_dbg.log 2>&1
FGB200_BLOCK_OVERLAP=0 python scripts/debug_ens.py >> gpurun_out/s2c_dbg.log 2>&1
FGB200_BLOCK_ITEMS=0 DBG_TB=16,24 python scripts/debug_ens.py >> gpurun_out/s2c_dbg.log 2>&1
timeout 900 python -m pytest tests/test_gpu_block.py -q -k ensemble > gpurun_out/s2c_block.log 2>&1; echo block=$?
