set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "ops_bitexact" > gpurun_out/r2_gputest13.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/r2_gputest13.log
timeout 600 python -m pytest tests/test_gpu_bench_params.py -q -m gpu -x -k "c1_params_ops or bsgs" >> gpurun_out/r2_gputest13.log 2>&1; echo "pytest2 rc=$?"
tail -3 gpurun_out/r2_gputest13.log
for tc in 0 1; do
  HK_CONV_TC=$tc timeout 600 python bench.py --steps 3 --warmup 1 --no-c2 --no-cpu-baseline > gpurun_out/r2_ab13_$tc.json 2>gpurun_out/r2_ab13_$tc.err
  python -c "import json; d=json.load(open('gpurun_out/r2_ab13_$tc.json')); print('tc=$tc', d['value'], d['e2e']['value'], d['kernels']['keyswitch']['ms'], d['max_abs_err_vs_reference_mirrored'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_mul_launches13.csv python tools/prof_ntt.py mul 37 128 > /dev/null 2>&1; echo "ncu1 rc=$?"
