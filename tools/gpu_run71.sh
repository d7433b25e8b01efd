set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_params.py -q -m gpu -x --deselect tests/test_gpu_bench_params.py::test_c4_layer1_bitexact --deselect tests/test_gpu_bench_params.py::test_c1_full_inference_bitexact > gpurun_out/r2_gputest71.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2_gputest71.log
for z in 1 0; do
HK_CONV_TC32=$z timeout 900 python bench.py --config c3 --steps 3 --warmup 2 --no-cpu-baseline --no-float-sim --no-c2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('TC32 $z', d['value'], d['e2e']['value'], d.get('max_abs_err_vs_reference_mirrored'))"
done
