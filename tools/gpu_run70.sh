set -x
for cpp in 8 4 8 4; do
HK_CPP_EPI=$cpp timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-float-sim --no-c2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('CPP $cpp', d['value'], d['e2e']['value'], d['clocks']['sm_mhz'])"
done
