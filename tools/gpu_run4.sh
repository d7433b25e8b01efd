set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_params.py -q -m gpu -x -k "not c4_layer1 and not full_inference" > gpurun_out/r2_gputest4.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2_gputest4.log
timeout 900 python bench.py --steps 3 --warmup 1 --no-c2 --no-cpu-baseline > gpurun_out/r2_bench4.json 2> gpurun_out/r2_bench4.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r2_bench4.json')); print(d['value'], d['e2e']['value'], d['kernels']['ntt']['ms'], d['kernels']['keyswitch']['ms'], d['max_abs_err_vs_reference_mirrored'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_mul_launches4.csv python tools/prof_ntt.py mul 37 128 > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 900 python -m pytest tests/test_gpu_bench_params.py -q -m gpu -x -k "full_inference" >> gpurun_out/r2_gputest4.log 2>&1; echo "pytest2 rc=$?"
tail -3 gpurun_out/r2_gputest4.log
