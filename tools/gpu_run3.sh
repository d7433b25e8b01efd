set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/r2_gputest3.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2_gputest3.log
timeout 600 python -m pytest tests/test_gpu_bench_params.py -q -m gpu -x -k "c1_params_ops or c5_params_ops" >> gpurun_out/r2_gputest3.log 2>&1; echo "pytest2 rc=$?"
tail -3 gpurun_out/r2_gputest3.log
timeout 900 python bench.py --steps 3 --warmup 1 --no-c2 --no-cpu-baseline > gpurun_out/r2_bench3.json 2> gpurun_out/r2_bench3.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r2_bench3.json')); print(d['value'], d['e2e']['value'], d['kernels']['ntt']['ms'], d['kernels']['keyswitch']['ms'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_mul_launches3.csv python tools/prof_ntt.py mul 37 128 > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fwd_kernel -c 1 -o gpurun_out/r2_ntt_fwd3 python tools/prof_ntt.py ntt 37 128 > gpurun_out/r2_ncu_ntt3.log 2>&1; echo "ncu2 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:EpiMdRsT2 -c 1 -o gpurun_out/r2_mdrs3 python tools/prof_ntt.py mul 37 128 > gpurun_out/r2_ncu_mdrs3.log 2>&1; echo "ncu3 rc=$?"
