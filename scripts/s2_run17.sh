mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/s2u_tests.log 2>&1; echo tests=$?
