# re-entry baseline: full GPU suite, smoke, default bench, reference arm, launch list, ncu of c4 dominant launches
mkdir -p gpurun_out/r02i
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/r02i/gpu.txt; nproc >> gpurun_out/r02i/gpu.txt; free -g >> gpurun_out/r02i/gpu.txt
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/r02i/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/r02i/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02i/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/r02i/bench.json 2> gpurun_out/r02i/bench.err; echo bench=$?; cat gpurun_out/r02i/bench.json
timeout 900 python bench.py --impl reference > gpurun_out/r02i/bench_ref.json 2> gpurun_out/r02i/bench_ref.err; echo ref=$?; cat gpurun_out/r02i/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02i/launches_c4.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r02i/ncu_launch.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fg_block_tma_kernel -s 90 -c 2 -o gpurun_out/r02i/c4f_dense python scripts/profile_run.py --config c4-full --steps 1600 > gpurun_out/r02i/ncu_dense.log 2>&1; echo ncu_dense=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fg_block_item_kernel -s 20 -c 2 -o gpurun_out/r02i/c4a_item python scripts/profile_run.py --config c4-adaptive --steps 1600 > gpurun_out/r02i/ncu_item.log 2>&1; echo ncu_item=$?
