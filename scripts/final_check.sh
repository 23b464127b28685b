# Round-end style check on one B200: GPU tests, smoke, default bench, reference arm.
mkdir -p gpurun_out/final
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/final/pytest_gpu.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/final/bench.log 2>&1; echo bench=$?
timeout 900 python bench.py --impl reference > gpurun_out/final/bench_ref.log 2>&1; echo ref=$?
