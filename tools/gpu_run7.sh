set -x
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_step_launches.csv python tools/prof_step.py --batch 128 --passes 2 > gpurun_out/r2_step.log 2>&1; echo "ncu rc=$?"
tail -2 gpurun_out/r2_step.log
