# c2 (small field) with sub-block launches: steps sum fewer recent offsets
mkdir -p gpurun_out/r02ak
b() { FGB200_SUBBLOCK=$1 FGB200_SUBDELAY=$2 timeout 600 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02ak/c2.json 2>gpurun_out/r02ak/c2.err; echo c2 S=$1 D=$2 $(python -c "import json;d=json.load(open('gpurun_out/r02ak/c2.json'));print(d['ms_per_step'])" 2>&1 | tail -1); }
for rep in 1 2; do
b 0 0; b 8 2; b 8 4; b 14 4; b 14 7; b 28 7; b 4 1; b 4 2
done
