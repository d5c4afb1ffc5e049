for g in 148 96; do echo "== one-stage 2000 grid $g"; KOT_TRD_GRID=$g timeout 200 python tools/eigbench.py 2000 2>&1 | grep "sytrd_panel\|Q:\|S:\|grid.sync"; done
timeout 600 python -m pytest tests -m gpu -x -q -k "eig or sym or tridiag" 2>&1 | tail -2
KOT_BENCH_DEBUG=1 timeout 300 python bench.py --no-cpu-baseline --no-ttt 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value %.3f e2e %.3f' % (d['value'],d['e2e']['value']))
    elif l.startswith('e2e'): print(l.strip()[:400])"
