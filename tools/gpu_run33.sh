set -x
timeout 600 python tools/time_prims.py --batch 128 > gpurun_out/r2_prims33.log 2>&1; cat gpurun_out/r2_prims33.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "ops_bitexact" 2>&1 | tail -3
