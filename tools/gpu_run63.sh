set -x
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_rot63.csv python tools/prof_rot.py 128 > /dev/null 2>&1; python tools/launches.py gpurun_out/r2_rot63.csv | grep -E "conv|total"
timeout 900 python -m pytest tests/test_gpu_bench_params.py -q -m gpu -x -k "ops_bitexact" 2>&1 | tail -2
