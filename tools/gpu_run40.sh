set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_params.py -q -m gpu -x --deselect tests/test_gpu_bench_params.py::test_c4_layer1_bitexact --deselect tests/test_gpu_bench_params.py::test_c1_full_inference_bitexact > gpurun_out/r2_gputest40.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2_gputest40.log
timeout 600 python tools/time_prims.py --batch 128 > gpurun_out/r2_prims40.log 2>&1; cat gpurun_out/r2_prims40.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-float-sim > gpurun_out/r2_bench40.json 2> gpurun_out/r2_bench40.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r2_bench40.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['kernels']['keyswitch']['ms']); print({k:(v['ms'],v['frac']) for k,v in d['c2_microbench'].items() if isinstance(v,dict)})"
