run() { echo "== $*"; env "$@" timeout 200 python bench.py --no-cpu-baseline --no-ttt 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); p=d['phases']
print('value %.3f e2e %.3f newton %.1f trial %.1f pipe_eg %.1f pipe_res %.1f' % (d['value'], d['e2e']['value'], p['host.newton']['ms_per_step'], p['host.trial_resid']['ms_per_step'], p['host.pipe_eg']['ms_per_step'], p['host.pipe_resid']['ms_per_step']))"; }
run KOT_X=0
run KOT_EG_PRIORITY=high
run KOT_TRD_GRID_BG=112 KOT_TRD_GRID_BG2=48
run KOT_TRD_GRID_FG=80 KOT_TRD_GRID_BG=112 KOT_TRD_GRID_BG2=48
run KOT_TRD_GRID_FG=112 KOT_TRD_GRID_BG=112 KOT_TRD_GRID_BG2=32
run KOT_MV_SPLIT=2
run KOT_MV_SPLIT=1
