set -x
timeout 900 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-float-sim > gpurun_out/r2_bench48.json 2> gpurun_out/r2_bench48.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r2_bench48.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['kernels']['keyswitch']['ms'], d['clocks']); print({k:(v['ms'],v['frac']) for k,v in d['c2_microbench'].items() if isinstance(v,dict)})"
