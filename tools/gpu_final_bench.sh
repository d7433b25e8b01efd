set -x
date
timeout 1500 python bench.py --impl reference --gpus 1 --steps 3 --warmup 1 > gpurun_out/r2_bench_reference_final.json 2> gpurun_out/r2_bench_reference_final.err; echo "ref rc=$?"
date
timeout 1500 python bench.py > gpurun_out/r2_bench_final.json 2> gpurun_out/r2_bench_final.err; echo "bench rc=$?"
date
python -c "import json; d=json.load(open('gpurun_out/r2_bench_final.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['ms'], d['kernels']['keyswitch']['ms'], d['kernels']['keyswitch']['traffic'], d['cpu_baseline']['value'], d['clocks'], d['gpu_launches']); print({k:(v['ms'],v['frac']) for k,v in d['c2_microbench'].items() if isinstance(v,dict)})"
python -c "import json; d=json.load(open('gpurun_out/r2_bench_reference_final.json')); print(d['value'], d['ms_per_step'], d['cpu_baseline'], d.get('float_simulator'))"
