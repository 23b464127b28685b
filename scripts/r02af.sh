# parameter sweeps on the defaults' neighbours: sub-block length and tblock (c5, c4-adaptive, c3-adaptive), fused pairs for c2
mkdir -p gpurun_out/r02af
for c in c5 c4-adaptive; do
  for tb in 96 112 128; do
    for sb in 16 24 28 32 48; do
      if [ $((tb % sb)) -ne 0 ]; then continue; fi
      FGB200_TBLOCK=$tb FGB200_SUBBLOCK=$sb timeout 600 python scripts/profile_run.py --config $c > gpurun_out/r02af/run.log 2>&1; echo $c tb=$tb S=$sb rc=$? $(tail -1 gpurun_out/r02af/run.log | cut -c1-45)
    done
  done
done
for fl in 2 258; do
  timeout 600 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline --flags $fl > gpurun_out/r02af/c2_$fl.json 2>/dev/null; echo c2 flags=$fl $(python -c "import json;d=json.load(open('gpurun_out/r02af/c2_$fl.json'));print(d['ms_per_step'])")
done
