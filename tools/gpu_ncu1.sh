# usage: gpu_ncu1.sh <kernel regex> <out name> <launch-skip> <cmd...>
set -x
rx=$1; out=$2; skip=$3; shift 3
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:$rx --launch-skip $skip -c 1 -o gpurun_out/$out "$@" > gpurun_out/$out.log 2>&1; echo "ncu rc=$?"
ls -la gpurun_out/
