# pad fix: full GPU suite (no -x), DMMA/DFMA microbenchmark, memcheck over every launch mode
mkdir -p gpurun_out/r02j
./scripts/micro/dmma_sweep > gpurun_out/r02j/dmma_sweep.txt 2>&1; echo sweep=$?; cat gpurun_out/r02j/dmma_sweep.txt
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r02j/pytest_gpu.log 2>&1; echo pytest=$?; tail -5 gpurun_out/r02j/pytest_gpu.log
bash scripts/sanitize.sh gpurun_out/r02j/sanitize memcheck
