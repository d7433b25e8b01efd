set -x
for dn in 2 3 4; do
timeout 900 python bench.py --dnum $dn --steps 3 --warmup 2 --no-cpu-baseline --no-float-sim --no-c2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('DNUM $dn', d['value'], d['e2e']['value'], d.get('max_abs_err_vs_reference_mirrored'), d['config']['workload'][-30:], d['config']['security'][:40])"
done
