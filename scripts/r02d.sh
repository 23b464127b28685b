# new bench (c4 default, driver's K/W), reference arm, ncu of the TMA item kernel
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02d_ref.json 2> gpurun_out/r02d_ref.err; echo ref_rc=$?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err; echo bench_rc=$?
python scripts/profile_run.py --config c3-adaptive --steps 1200 > gpurun_out/r02d_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fg_block_item_kernel -s 30 -c 8 -o gpurun_out/r02d_c3a_item16 python scripts/profile_run.py --config c3-adaptive --steps 1200 > gpurun_out/r02d_ncu.log 2>&1; echo ncu_rc=$?
