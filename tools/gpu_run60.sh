set -x
for z in 0 1 2 3 4 7; do echo "DBG $z"; HK_CONV_DBG=$z timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_dbg$z.csv python tools/prof_rot.py 128 > /dev/null 2>&1; python tools/launches.py gpurun_out/r2_dbg$z.csv | grep conv; done
