set -x
for z in 16 24 16 24 12; do echo "EPI $z"; HK_CONV_EPI=$z timeout 600 python tools/time_prims.py --batch 128 2>&1 | grep -E "mul_ct|rotate"; done
HK_CONV_EPI=24 timeout 900 python -m pytest tests/test_gpu_bench_params.py -q -m gpu -x -k "ops_bitexact" 2>&1 | tail -2
HK_CONV_EPI=24 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_mul_launches59.csv python tools/prof_ntt.py mul 37 128 > /dev/null 2>&1; echo "ncu mul rc=$?"
