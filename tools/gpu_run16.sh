set -x
timeout 2400 python -m pytest tests -q -m gpu --durations=10 > gpurun_out/r2_gputest16.log 2>&1; echo "pytest rc=$?"
tail -16 gpurun_out/r2_gputest16.log
timeout 600 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_rotate_traffic.csv python tools/prof_rot.py 128 > /dev/null 2>&1; echo "ncu rot rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_step_launches16.csv python tools/prof_step.py --batch 128 --passes 2 > gpurun_out/r2_step16.log 2>&1; echo "ncu step rc=$?"
tail -1 gpurun_out/r2_step16.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench16.json 2> gpurun_out/r2_bench16.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r2_bench16.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['kernels']['keyswitch']['ms'], d['cpu_baseline']['value'], d['clocks'])"
