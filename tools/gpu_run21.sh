set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_params.py -q -m gpu -x --deselect tests/test_gpu_bench_params.py::test_c4_layer1_bitexact > gpurun_out/r2_gputest21.log 2>&1; echo "pytest rc=$?"
tail -12 gpurun_out/r2_gputest21.log
timeout 600 python tools/time_prims.py --batch 128 > gpurun_out/r2_prims21.log 2>&1; cat gpurun_out/r2_prims21.log
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_conv_tc -c 1 -o gpurun_out/r2_convtc2_modup python tools/prof_rot.py 128 > gpurun_out/r2_ncu_convtc2.log 2>&1; echo "ncu1 rc=$?"
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_mul_launches21.csv python tools/prof_rot.py 128 > /dev/null 2>&1; echo "ncu rot rc=$?"
