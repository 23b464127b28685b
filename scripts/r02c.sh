# config-scale parity (parity log), c3-adaptive trace, dense-kernel ncu on c4-full
export FGB200_PARITY_LOG=gpurun_out/r02c_parity.jsonl
rm -f $FGB200_PARITY_LOG
timeout 1500 python -m pytest tests/test_gpu_configs.py -x -q -m gpu > gpurun_out/r02c_configs.log 2>&1; echo configs_rc=$?
tail -3 gpurun_out/r02c_configs.log
FGB200_TRACE=gpurun_out/r02c_c3a_trace.txt timeout 300 python scripts/profile_run.py --config c3-adaptive > gpurun_out/r02c_trace_run.log 2>&1; echo trace_rc=$?
timeout 300 python scripts/profile_run.py --config c4-full --steps 1600 > gpurun_out/r02c_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fg_block_tma_kernel -s 90 -c 2 -o gpurun_out/r02c_c4f_dense python scripts/profile_run.py --config c4-full --steps 1600 > gpurun_out/r02c_ncu.log 2>&1; echo ncu_rc=$?
