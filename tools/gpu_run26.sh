set -x
for cpp in 4 8; do
HK_CPP_EPI=$cpp timeout 1200 python bench.py --steps 6 --warmup 3 > gpurun_out/r2_bench26_$cpp.json 2> gpurun_out/r2_bench26_$cpp.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r2_bench26_$cpp.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['kernels']['keyswitch']['ms'], d['cpu_baseline']['value'], d['clocks'])"
done
