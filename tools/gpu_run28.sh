set -x
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:EpiMdRsY2 --launch-skip 1 -c 1 -o gpurun_out/r2_mdrsy2 python tools/prof_ntt.py mul 37 128 > gpurun_out/r2_ncu_mdrsy2.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:ProD2 --launch-skip 1 -c 1 -o gpurun_out/r2_prod2 python tools/prof_ntt.py mul 37 128 > gpurun_out/r2_ncu_prod2.log 2>&1; echo "ncu2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:k_key_ip --launch-skip 1 -c 1 -o gpurun_out/r2_keyip python tools/prof_ntt.py mul 37 128 > gpurun_out/r2_ncu_keyip.log 2>&1; echo "ncu3 rc=$?"
