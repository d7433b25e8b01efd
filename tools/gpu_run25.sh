set -x
for cpp in 4 8; do
HK_CPP_EPI=$cpp timeout 600 python tools/time_prims.py --batch 128 > gpurun_out/r2_prims25_$cpp.log 2>&1; cat gpurun_out/r2_prims25_$cpp.log
done
HK_CPP_EPI=8 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_rot_launches25.csv python tools/prof_rot.py 128 > /dev/null 2>&1; echo "ncu rot rc=$?"
