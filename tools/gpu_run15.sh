set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "ops_bitexact" > gpurun_out/r2_gputest15.log 2>&1; echo "pytest rc=$?"
HK_CONV_EPI=16 timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "ops_bitexact" >> gpurun_out/r2_gputest15.log 2>&1; echo "pytest16 rc=$?"
tail -3 gpurun_out/r2_gputest15.log
for ew in 8 12 16; do
  HK_CONV_EPI=$ew timeout 600 python bench.py --steps 3 --warmup 1 --no-c2 --no-cpu-baseline > gpurun_out/r2_ab15_$ew.json 2>gpurun_out/r2_ab15_$ew.err
  python -c "import json; d=json.load(open('gpurun_out/r2_ab15_$ew.json')); print('epi=$ew', d['value'], d['e2e']['value'], d['kernels']['keyswitch']['ms'])"
  HK_CONV_EPI=$ew timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_mul_launches15_$ew.csv python tools/prof_ntt.py mul 37 128 > /dev/null 2>&1
done
