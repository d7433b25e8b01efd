set -x
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_conv_tc -c 1 -o gpurun_out/r2_convtc3 python tools/prof_ntt.py mul 37 128 > gpurun_out/r2_ncu_convtc3.log 2>&1; echo "ncu rc=$?"
