set -x
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_conv --launch-skip 3 -c 1 -o gpurun_out/r2_kconv14 python tools/prof_ntt.py mul 37 128 > gpurun_out/r2_ncu_kconv.log 2>&1; echo "ncu2 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_key_ip -c 1 -o gpurun_out/r2_keyip python tools/prof_ntt.py mul 37 128 > gpurun_out/r2_ncu_keyip.log 2>&1; echo "ncu3 rc=$?"
ls gpurun_out
