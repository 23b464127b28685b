# ncu --set full of the UNBLOCKED fused step kernel (FGB200_TBLOCK=0: one history pass per step,
# the north star's literal kernel) at a mid-run step of c3-full, c4-full and c3-adaptive.
O=${OUT:-gpurun_out/r02u0}
mkdir -p $O
export FGB200_TBLOCK=0
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fg_step_kernel -s 1500 -c 1 \
  -o $O/c3f_step python scripts/profile_run.py --config c3-full --steps 1502 > $O/ncu_c3f.log 2>&1; echo c3f=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fg_step_kernel -s 1500 -c 1 \
  -o $O/c4f_step python scripts/profile_run.py --config c4-full --steps 1502 > $O/ncu_c4f.log 2>&1; echo c4f=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fg_step_kernel -s 3000 -c 1 \
  -o $O/c3a_step python scripts/profile_run.py --config c3-adaptive --steps 3002 > $O/ncu_c3a.log 2>&1; echo c3a=$?
for c in c3-full c4-full c3-adaptive; do python scripts/profile_run.py --config $c --steps 1502 | tail -1; done
