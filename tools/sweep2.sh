run() { echo "== $*"; env KOT_BENCH_DEBUG=1 "$@" timeout 200 python bench.py --no-cpu-baseline --no-ttt 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); p=d['phases']; print('value %.3f e2e %.3f newton %.1f trial %.1f pipe_eg %.1f pipe_res %.1f wait %.1f' % (d['value'],d['e2e']['value'],p['host.newton']['ms_per_step'],p['host.trial_resid']['ms_per_step'],p['host.pipe_eg']['ms_per_step'],p['host.pipe_resid']['ms_per_step'],p['host.eg_wait']['ms_per_step']))
    elif l.startswith('e2e'): print(l.strip()[:300])"; }
run KOT_TRD_GRID=96 KOT_TRD_GRID_BG=96 KOT_TRD_GRID_BG2=64
run KOT_TRD_GRID=80 KOT_TRD_GRID_BG=96 KOT_TRD_GRID_BG2=64
run KOT_TRD_GRID=112 KOT_TRD_GRID_BG=96 KOT_TRD_GRID_BG2=64
run KOT_TRD_GRID=96 KOT_TRD_GRID_BG=112 KOT_TRD_GRID_BG2=64
run KOT_TRD_GRID=96 KOT_TRD_GRID_BG=96 KOT_TRD_GRID_BG2=80
run KOT_TRD_GRID=96 KOT_TRD_GRID_BG=96 KOT_TRD_GRID_BG2=48
run KOT_TRD_GRID=112 KOT_TRD_GRID_BG=112 KOT_TRD_GRID_BG2=64
run KOT_TRD_GRID=96 KOT_TRD_GRID_BG=128 KOT_TRD_GRID_BG2=64
run KOT_TRD_GRID=96 KOT_TRD_GRID_BG=96 KOT_TRD_GRID_BG2=64 KOT_EG_PRIORITY=high
