# (sub-block S, delay D) sweep around the new defaults
mkdir -p gpurun_out/r02ai
sw() { c=$1; S=$2; D=$3; FGB200_SUBBLOCK=$S FGB200_SUBDELAY=$D timeout 600 python scripts/profile_run.py --config $c > gpurun_out/r02ai/run.log 2>&1; echo $c S=$S D=$D rc=$? $(tail -1 gpurun_out/r02ai/run.log | cut -c1-45); }
for rep in 1 2; do
sw c4-adaptive 28 7; sw c4-adaptive 14 7; sw c4-adaptive 14 4; sw c4-adaptive 56 14; sw c4-adaptive 56 7; sw c4-adaptive 16 4
sw c5 32 8; sw c5 16 8; sw c5 16 4; sw c5 64 16; sw c5 64 8
sw c4-full 8 4; sw c4-full 4 2; sw c4-full 16 4; sw c4-full 16 8; sw c4-full 8 2
done
