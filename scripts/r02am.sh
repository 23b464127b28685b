# bench.py after the sharded-c5 change: default line and c5 line (one GPU)
mkdir -p gpurun_out/r02am
timeout 900 python bench.py --steps 2 --warmup 3 > gpurun_out/r02am/bench_c4.json 2> gpurun_out/r02am/bench_c4.err; echo c4=$?; python -c "import json;d=json.load(open('gpurun_out/r02am/bench_c4.json'));print(d['value']/1e12, d['scaling'], d['config']['parallelism'])"
timeout 900 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02am/bench_c5.json 2> gpurun_out/r02am/bench_c5.err; echo c5=$?; python -c "import json;d=json.load(open('gpurun_out/r02am/bench_c5.json'));print(d['value']/1e12, d['scaling'], d['config']['parallelism'])"
