for i in 1 2 3 4 5; do KOT_BENCH_DEBUG=1 timeout 200 python bench.py --no-cpu-baseline --no-ttt 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); e=d['e2e']; print('value %.3f e2e %.3f wall %.0f solve %.0f iters %.0f' % (d['value'], e['value'], e['wall_ms'], e['solve_ms'], e['iterations_ms']))
    elif l.startswith('e2e'): print(l.strip()[:300])"; done
