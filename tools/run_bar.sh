timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for n in 2000; do echo "== eig $n"; timeout 200 python tools/eigbench.py $n 2>&1 | grep "err\|eigh \|eig.sytrd\|sytrd_panel\|sytrd_tail \|Q:\|S:\|grid.sync"; done
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --no-ttt 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); p=d['phases']
print('value %.3f e2e %.3f newton %.1f trial %.1f pipe_eg %.1f pipe_res %.1f' % (d['value'], d['e2e']['value'], p['host.newton']['ms_per_step'], p['host.trial_resid']['ms_per_step'], p['host.pipe_eg']['ms_per_step'], p['host.pipe_resid']['ms_per_step']))"; done
KOT_TRD_GRID=48 timeout 300 python tools/conc_probe.py 6 40 3 2>&1 | tail -1
