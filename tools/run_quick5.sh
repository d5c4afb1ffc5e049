timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash tools/e2e_var.sh 2>&1 | head -4
KOT_BENCH_DEBUG=1 timeout 600 python bench.py --config cfg4 --no-cpu-baseline --no-ttt --steps 6 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); e=d['e2e']; print('cfg4 value %.3f e2e %.3f wall %.0f solve %.0f iters %.0f' % (d['value'], e['value'], e['wall_ms'], e['solve_ms'], e['iterations_ms']))
    elif l.startswith('e2e'): print(l.strip()[:300])"
KOT_TRD_GRID=48 timeout 300 python tools/conc_probe.py 8 40 4 2>&1 | tail -1
