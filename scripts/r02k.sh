# re-entry: GPU suite at HEAD, ncu of the 16-column item kernel main launches (c3/c4-adaptive, c5), sanitizers
mkdir -p gpurun_out/r02k
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/r02k/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/r02k/pytest_gpu.log
for c in c3-adaptive c4-adaptive; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fg_block_item_kernel -s 12 -c 2 -o gpurun_out/r02k/${c}_item python scripts/profile_run.py --config $c --steps 1200 > gpurun_out/r02k/ncu_$c.log 2>&1; echo ncu_$c=$?
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fg_block_item_kernel -s 40 -c 2 -o gpurun_out/r02k/c5_item python scripts/profile_run.py --config c5 --steps 3000 > gpurun_out/r02k/ncu_c5.log 2>&1; echo ncu_c5=$?
bash scripts/sanitize.sh gpurun_out/r02k/sanitize memcheck synccheck racecheck
