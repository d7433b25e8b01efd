set -x
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_conv_tc -c 1 -o gpurun_out/r2_convtc_modup python tools/prof_rot.py 128 > gpurun_out/r2_ncu_convtc.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_conv_tc --launch-skip 3 -c 1 -o gpurun_out/r2_convtc_moddown python tools/prof_rot.py 128 > gpurun_out/r2_ncu_convtc2.log 2>&1; echo "ncu2 rc=$?"
tail -3 gpurun_out/r2_ncu_convtc.log
