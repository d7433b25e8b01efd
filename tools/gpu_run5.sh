set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/r2_gputest5.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2_gputest5.log
timeout 900 python bench.py --steps 3 --warmup 1 --no-c2 --no-cpu-baseline > gpurun_out/r2_bench5.json 2> gpurun_out/r2_bench5.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r2_bench5.json')); print(d['value'], d['e2e']['value'], d['kernels']['ntt']['ms'], d['kernels']['keyswitch']['ms'], d['max_abs_err_vs_reference_mirrored'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_mul_launches5.csv python tools/prof_ntt.py mul 37 128 > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"k_conv<14>" -c 1 -o gpurun_out/r2_kconv14 python tools/prof_ntt.py mul 37 128 > gpurun_out/r2_ncu_kconv.log 2>&1; echo "ncu2 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"k_key_ip<3, 1>" -c 1 -o gpurun_out/r2_keyip python tools/prof_ntt.py mul 37 128 > gpurun_out/r2_ncu_keyip.log 2>&1; echo "ncu3 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"ProD2" -c 1 -o gpurun_out/r2_prod2 python tools/prof_ntt.py mul 37 128 > gpurun_out/r2_ncu_prod2.log 2>&1; echo "ncu4 rc=$?"
