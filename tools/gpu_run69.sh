set -x
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_step_c4.csv python tools/prof_step.py --config c4 --batch 32 --passes 2 > gpurun_out/r2_step_c4.log 2>&1; echo "ncu step rc=$?"
tail -2 gpurun_out/r2_step_c4.log
gzip -9 gpurun_out/r2_step_c4.csv
