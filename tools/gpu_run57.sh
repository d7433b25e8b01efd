set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_params.py -q -m gpu -x --deselect tests/test_gpu_bench_params.py::test_c4_layer1_bitexact --deselect tests/test_gpu_bench_params.py::test_c1_full_inference_bitexact > gpurun_out/r2_gputest57.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2_gputest57.log
for z in 1 0 1 0; do HK_CONV_LAZY=$z timeout 600 python tools/time_prims.py --batch 128 2>&1 | grep -E "mul_ct|rotate"; done
