# quick GPU check: parity suite + contention probe + cfg3 bench (value, e2e)
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/contention_probe.py 2>&1 | grep "safeguard\|matvec\|newton "
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --no-ttt 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); p=d['phases']
print('value %.3f e2e %.3f newton %.1f trial %.1f pipe_eg %.1f matvec %.1f/%d' % (d['value'], d['e2e']['value'], p['host.newton']['ms_per_step'], p['host.trial_resid']['ms_per_step'], p['host.pipe_eg']['ms_per_step'], p['matvec']['ms_per_step'], p['matvec']['calls_per_step']))"; done
