timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
run() { echo "== $*"; env "$@" timeout 200 python bench.py --no-cpu-baseline --no-ttt 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); p=d['phases']
print('value %.3f e2e %.3f newton %.1f trial %.1f pipe_eg %.1f pipe_res %.1f wait %.1f' % (d['value'], d['e2e']['value'], p['host.newton']['ms_per_step'], p['host.trial_resid']['ms_per_step'], p['host.pipe_eg']['ms_per_step'], p['host.pipe_resid']['ms_per_step'], p['host.eg_wait']['ms_per_step']))"; }
run KOT_X=0
run KOT_TRD_GRID_BG=64
run KOT_TRD_GRID_BG=64 KOT_TRD_GRID_BG2=48
run KOT_TRD_GRID_FG=112 KOT_TRD_GRID_BG=56 KOT_TRD_GRID_BG2=48
run KOT_TRD_GRID_FG=128 KOT_TRD_GRID_BG=48 KOT_TRD_GRID_BG2=48
run KOT_TRD_GRID_FG=148 KOT_TRD_GRID_BG=48 KOT_TRD_GRID_BG2=48
KOT_TRD_GRID=48 timeout 300 python tools/conc_probe.py 6 40 3 2>&1 | tail -1
