set -x
timeout 2400 python -m pytest tests -q -m gpu -x --durations=5 > gpurun_out/r2_gputest20.log 2>&1; echo "pytest rc=$?"
tail -12 gpurun_out/r2_gputest20.log
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_conv_tc -c 1 -o gpurun_out/r2_convtc_modup python tools/prof_rot.py 128 > gpurun_out/r2_ncu_convtc.log 2>&1; echo "ncu1 rc=$?"
tail -3 gpurun_out/r2_ncu_convtc.log
