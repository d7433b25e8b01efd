set -x
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_mul_launches52.csv python tools/prof_ntt.py mul 37 128 > /dev/null 2>&1; echo "ncu mul rc=$?"
