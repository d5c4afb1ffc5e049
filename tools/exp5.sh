timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2 3 4; do
KOT_BENCH_DEBUG=1 timeout 300 python bench.py --no-cpu-baseline --no-ttt 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value %.3f e2e %.3f' % (d['value'],d['e2e']['value']))
    elif l.startswith('e2e'): print(l.strip()[:400])"
done
