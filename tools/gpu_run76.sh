set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_params.py -q -m gpu -x --deselect tests/test_gpu_bench_params.py::test_c4_layer1_bitexact --deselect tests/test_gpu_bench_params.py::test_c1_full_inference_bitexact > gpurun_out/r2_gputest76.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2_gputest76.log
timeout 600 python tools/time_prims.py --batch 128
for bbv in 4 8 4 8; do echo "BB $bbv"; HK_KEYIP_BB=$bbv timeout 600 python tools/time_prims.py --batch 128 2>&1 | grep -E "mul_ct|rotate"; done
