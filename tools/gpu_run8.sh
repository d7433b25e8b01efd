set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "ops_bitexact or bsgs or rotate_sum" > gpurun_out/r2_gputest8.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2_gputest8.log
for cfg in "0 4" "4 4" "8 4" "4 1" "4 2"; do
  set -- $cfg
  HK_CONV_WAVES=$1 HK_KEYIP_BB=$2 timeout 600 python bench.py --steps 3 --warmup 1 --no-c2 --no-cpu-baseline > gpurun_out/r2_ab8_$1_$2.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/r2_ab8_$1_$2.json')); print('waves=$1 bb=$2', d['value'], d['e2e']['value'], d['kernels']['keyswitch']['ms'])"
done
