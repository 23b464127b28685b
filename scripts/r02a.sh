set -x
free -g; nproc; lscpu | grep -i "model name\|^CPU(s)\|Thread\|Socket"; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/r02a_pytest.log 2>&1; echo pytest_rc=$?
python scripts/profile_run.py --config c3-adaptive --steps 1200 > gpurun_out/r02a_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fg_block_item_kernel -s 30 -c 8 -o gpurun_out/r02a_c3a_item16 python scripts/profile_run.py --config c3-adaptive --steps 1200 > gpurun_out/r02a_ncu.log 2>&1; echo ncu_rc=$?
