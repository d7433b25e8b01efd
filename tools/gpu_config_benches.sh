set -x
for cfg in "c5" "c5 --log-n 17" "c4" "c3" "c1 --log-n 17"; do
  name=$(echo $cfg | tr -d ' -')
  timeout 1500 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-float-sim --no-c2 > gpurun_out/r2_bench_$name.json 2> gpurun_out/r2_bench_$name.err; echo "bench $cfg rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/r2_bench_$name.json')); print(d['config']['workload'], d['value'], d['e2e']['value'], d.get('max_abs_err_vs_reference_mirrored'))"
done
