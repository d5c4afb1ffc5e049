timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2 3; do timeout 300 python bench.py --no-cpu-baseline --no-ttt 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); p=d['phases']
print('value %.3f e2e %.3f newton %.1f trial %.1f pipe_eg %.1f pipe_res %.1f' % (d['value'], d['e2e']['value'], p['host.newton']['ms_per_step'], p['host.trial_resid']['ms_per_step'], p['host.pipe_eg']['ms_per_step'], p['host.pipe_resid']['ms_per_step']))"; done
timeout 600 python bench.py --config cfg4 --no-cpu-baseline --no-ttt --steps 6 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('cfg4 value %.3f e2e %.3f' % (d['value'], d['e2e']['value']))"
timeout 600 python bench.py --config cfg5 --batch 16 --max-iter 100 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('cfg5 %.3f' % d['value'])"
