timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
echo "== eigbench 2000"; timeout 200 python tools/eigbench.py 2000 2>&1 | head -21
echo "== eigbench 1000"; timeout 200 python tools/eigbench.py 1000 2>&1 | head -21 | grep -v "^  [a-z.]* *calls"
for i in 1 2; do
KOT_BENCH_DEBUG=1 timeout 300 python bench.py --no-cpu-baseline --no-ttt 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value',d['value'],'e2e',d['e2e']['value'], 'roof', d['roofline']['achieved'], d['roofline']['avg_launch_ms'])
    else: print(l.rstrip()[:400])"
done
