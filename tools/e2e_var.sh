# e2e variance: the e2e leg (first solve in a fresh process) several times, with its per-iteration times
for i in 1 2 3 4 5 6; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-ttt --no-cpu-baseline --no-batch 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); e=d['e2e']
        print(round(d['value'],2), 'e2e', round(e['value'],2), 'wall', e['wall_ms'], 'asm', e['assemble_ms'], 'setup', e['setup_ms'], 'steps', e['step_ms'])
"
done
