set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_params.py -q -m gpu -x --deselect tests/test_gpu_bench_params.py::test_c4_layer1_bitexact --deselect tests/test_gpu_bench_params.py::test_c1_full_inference_bitexact > gpurun_out/r2_gputest58.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2_gputest58.log
for z in 0 1 0 1; do HK_CONV_STRIDE=$z timeout 600 python tools/time_prims.py --batch 128 2>&1 | grep -E "mul_ct|rotate"; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_mul_launches58.csv python tools/prof_ntt.py mul 37 128 > /dev/null 2>&1; echo "ncu mul rc=$?"
