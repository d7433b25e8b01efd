set -x
nproc
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/r2_gputest1.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/r2_gputest1.log
timeout 900 python bench.py --steps 3 --warmup 1 > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r2_bench1.json
tail -20 gpurun_out/r2_bench1.err
