mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/s2_pytest.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2_smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/s2_default.log 2>&1; echo default=$?
timeout 600 python bench.py --impl reference > gpurun_out/s2_ref.log 2>&1; echo ref=$?
