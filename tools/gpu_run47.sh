set -x
for f in 1 0 1 0; do HK_RS_FAST=$f timeout 600 python tools/time_prims.py --batch 128 2>&1 | grep -E "mul_plain|rescale-only"; done
