set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_params.py -q -m gpu -x --deselect tests/test_gpu_bench_params.py::test_c4_layer1_bitexact --deselect tests/test_gpu_bench_params.py::test_c1_full_inference_bitexact > gpurun_out/r2_gputest_parity.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2_gputest_parity.log
timeout 600 python tools/time_prims.py --batch 128 > gpurun_out/r2_prims.log 2>&1; cat gpurun_out/r2_prims.log
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_rot_launches.csv python tools/prof_rot.py 128 > /dev/null 2>&1; echo "ncu rot rc=$?"
