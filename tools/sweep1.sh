run() { echo "== $*"; env "$@" timeout 200 python bench.py --no-cpu-baseline --no-ttt 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); p=d['phases']; print('value %.3f e2e %.3f newton %.1f trial %.1f pipe_eg %.1f pipe_res %.1f wait %.1f' % (d['value'],d['e2e']['value'],p['host.newton']['ms_per_step'],p['host.trial_resid']['ms_per_step'],p['host.pipe_eg']['ms_per_step'],p['host.pipe_resid']['ms_per_step'],p['host.eg_wait']['ms_per_step']))"; }
run KOT_X=0
run KOT_EG_PRIORITY=high
run KOT_TRD_GRID_BG=96
run KOT_TRD_GRID_BG=96 KOT_TRD_GRID_BG2=64
run KOT_TRD_GRID_BG=148 KOT_TRD_GRID_BG2=64
run KOT_TRD_GRID_BG=96 KOT_EG_PRIORITY=high
run KOT_TRD_GRID_BG=128 KOT_TRD_GRID_BG2=48 KOT_EG_PRIORITY=high
run KOT_TRD_GRID=96 KOT_TRD_GRID_BG=96 KOT_TRD_GRID_BG2=64
