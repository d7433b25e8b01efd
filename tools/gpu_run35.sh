set -x
timeout 900 python -m pytest tests/test_gpu_bench_params.py -q -m gpu -x -k "ops_bitexact" 2>&1 | tail -3
timeout 600 python tools/time_prims.py --batch 128 > gpurun_out/r2_prims35.log 2>&1; cat gpurun_out/r2_prims35.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_mul_launches35.csv python tools/prof_ntt.py mul 37 128 > /dev/null 2>&1; echo "ncu mul rc=$?"
