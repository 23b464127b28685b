# DRAM bytes of every launch of two mid-run temporal blocks (serialised, L2 state kept): the
# traffic a block really moves, to set against its in-run time (traces)
mkdir -p gpurun_out/r02u
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 1200 ncu --metrics $M --cache-control none --clock-control none -s 2300 -c 240 --csv --log-file gpurun_out/r02u/c4a_block.csv python scripts/profile_run.py --config c4-adaptive --steps 2600 > gpurun_out/r02u/c4a.log 2>&1; echo c4a=$?
timeout 1200 ncu --metrics $M --cache-control none --clock-control none -s 2400 -c 80 --csv --log-file gpurun_out/r02u/c4f_block.csv python scripts/profile_run.py --config c4-full --steps 2600 > gpurun_out/r02u/c4f.log 2>&1; echo c4f=$?
timeout 1200 ncu --metrics $M --cache-control none --clock-control none -s 2300 -c 240 --csv --log-file gpurun_out/r02u/c3a_block.csv python scripts/profile_run.py --config c3-adaptive --steps 2600 > gpurun_out/r02u/c3a.log 2>&1; echo c3a=$?
