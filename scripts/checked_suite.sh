# GPU test suite against the bounds-checked build (FG_CHECKS: every kernel index
# checked against its buffer, trap on violation) — the stand-in for
# compute-sanitizer, which is closed on the GPU pool.
# usage: bash scripts/checked_suite.sh <outdir>
OUT=${1:-gpurun_out/checked}
mkdir -p $OUT
export FGB200_LIB=paper_1004_5128_b200/_lib/variants/libfgb200_checked.so
timeout 3000 python -m pytest tests -q -m gpu -p no:cacheprovider > $OUT/pytest_checked.log 2>&1
echo "checked suite rc=$?"; tail -3 $OUT/pytest_checked.log
grep -c "FG_CHECK failed" $OUT/pytest_checked.log || true
