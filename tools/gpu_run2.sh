set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_params.py -q -m gpu -k "not c4_layer1" > gpurun_out/r2_gputest2.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2_gputest2.log
timeout 900 python bench.py --steps 3 --warmup 1 --no-c2 --no-cpu-baseline > gpurun_out/r2_bench2.json 2> gpurun_out/r2_bench2.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r2_bench2.json')); print(d['value'], d['e2e']['value'], d['kernels']['ntt']['ms'], d['kernels']['keyswitch']['ms'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_mul_launches.csv python tools/prof_ntt.py mul 37 128 > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fwd_kernel -c 1 -o gpurun_out/r2_ntt_fwd python tools/prof_ntt.py ntt 37 128 > gpurun_out/r2_ncu_ntt.log 2>&1; echo "ncu2 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:EpiMdRsT2 -c 1 -o gpurun_out/r2_mdrs python tools/prof_ntt.py mul 37 128 > gpurun_out/r2_ncu_mdrs.log 2>&1; echo "ncu3 rc=$?"
ls -la gpurun_out/
