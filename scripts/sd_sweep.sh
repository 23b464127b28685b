# (S, D) sweep of the sub-block launches on one B200 (gpurun, from the repo root).
# usage: CONFIGS="c4-full c3-full" PAIRS="8:2 8:4 16:4" [LIBV=variant] bash scripts/sd_sweep.sh <outdir>
O=${1:?outdir}
CONFIGS=${CONFIGS:-c4-full}
PAIRS=${PAIRS:-"8:2 8:4 16:4"}
REPS=${REPS:-2}
mkdir -p $O
[ -n "$LIBV" ] && export FGB200_LIB=paper_1004_5128_b200/_lib/variants/libfgb200_$LIBV.so
for rep in $(seq $REPS); do
  for sd in $PAIRS; do
    for c in $CONFIGS; do
      FGB200_SUBBLOCK=${sd%%:*} FGB200_SUBDELAY=${sd##*:} timeout 900 python scripts/profile_run.py --config $c > $O/run_${sd/:/_}_$c.log 2>&1
      echo "S:D=$sd $c rc=$? $(tail -1 $O/run_${sd/:/_}_$c.log | cut -c1-60)"
    done
  done
done
