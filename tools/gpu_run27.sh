set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:EpiMdRsY2 --launch-skip 1 -c 1 -o gpurun_out/r2_mdrsy2 python tools/prof_ntt.py mul 37 128 > gpurun_out/r2_ncu_mdrsy2.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ProD2 --launch-skip 1 -c 1 -o gpurun_out/r2_prod2 python tools/prof_ntt.py mul 37 128 > gpurun_out/r2_ncu_prod2.log 2>&1; echo "ncu2 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_mul_launches27.csv python tools/prof_ntt.py mul 37 128 > /dev/null 2>&1; echo "ncu mul rc=$?"
