set -x
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:fwd_kernel --launch-skip 1 -c 1 -o gpurun_out/r2_ntt_fwd_final python tools/prof_ntt.py ntt 37 128 > gpurun_out/r2_ncu_ntt_final.log 2>&1; echo "ncu ntt rc=$?"
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_rot_launches_final.csv python tools/prof_rot.py 128 > /dev/null 2>&1; echo "ncu rot rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_mul_launches_final.csv python tools/prof_ntt.py mul 37 128 > /dev/null 2>&1; echo "ncu mul rc=$?"
