timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/contention_probe.py
for i in 1 2; do
KOT_BENCH_DEBUG=1 timeout 300 python bench.py --no-cpu-baseline --no-ttt 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value',d['value'],'e2e',d['e2e']['value'], 'cg', d['trace']['cg_iters'], 'res', [round(x,3) for x in d['trace']['res']])
    else: print(l.rstrip()[:400])"
done
