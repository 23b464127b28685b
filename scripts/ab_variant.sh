# A/B timing of library variants on one B200 (gpurun, from the repo root).
# Variants are builds of the same sources with extra defines, e.g.
#   python -c "from paper_1004_5128_b200 import build as B; \
#     B.build(out='paper_1004_5128_b200/_lib/variants/libfgb200_x.so', defines=('FG_X=1',))"
# usage: REPS=3 CONFIGS="c4-full c3-full" TEST=tests/test_gpu_block.py bash scripts/ab_variant.sh <out> default x [...]
# Each variant runs its parity test selection first (TEST, optional), then every config
# REPS times, interleaved with the other variants so box drift hits all of them alike.
O=${1:?outdir}; shift
VARIANTS=${@:-default}
REPS=${REPS:-3}
CONFIGS=${CONFIGS:-c4-full c4-adaptive}
mkdir -p $O
lib() { [ $1 = default ] && echo "" || echo paper_1004_5128_b200/_lib/variants/libfgb200_$1.so; }
if [ -n "$TEST" ]; then
  for v in $VARIANTS; do
    FGB200_LIB=$(lib $v) timeout 1200 python -m pytest -q -x $TEST > $O/pytest_$v.log 2>&1
    echo "$v pytest rc=$? $(tail -1 $O/pytest_$v.log)"
  done
fi
for rep in $(seq $REPS); do
  for v in $VARIANTS; do
    for c in $CONFIGS; do
      FGB200_LIB=$(lib $v) timeout 900 python scripts/profile_run.py --config $c > $O/run_${v}_$c.log 2>&1
      echo "$v $c rc=$? $(tail -1 $O/run_${v}_$c.log | cut -c1-60)"
    done
  done
done
