set -x
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:fwd_kernel --launch-skip 2 -c 1 -o gpurun_out/r2_ntt_fwd_head python tools/prof_ntt.py ntt 37 128 > gpurun_out/r2_ncu_ntt_head.log 2>&1; echo "ncu ntt rc=$?"
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_step_launches54.csv python tools/prof_step.py --batch 128 --passes 2 > gpurun_out/r2_step54.log 2>&1; echo "ncu step rc=$?"
tail -2 gpurun_out/r2_step54.log
gzip -9 gpurun_out/r2_step_launches54.csv
ls -la gpurun_out/
