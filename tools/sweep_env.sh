# env-knob sweep of the cfg3 iteration rate (diagnostic): one bench line per setting
run() { echo "== $*"; env "$@" timeout 300 python bench.py --steps 12 --warmup 3 --no-ttt --no-cpu-baseline 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); p=d['phases']
        print(round(d['value'],2), 'it/s  e2e', round(d['e2e']['value'],2), ' newton', round(p['host.newton']['ms_per_step'],1), 'trial', round(p['host.trial_resid']['ms_per_step'],1), 'eg', round(p['host.pipe_eg']['ms_per_step'],1), 'resid', round(p['host.pipe_resid']['ms_per_step'],1))
"; }
run KOT_X=0
run KOT_TRD_GRID_BG=32 KOT_TRD_GRID_BG2=24
run KOT_TRD_GRID_BG=24 KOT_TRD_GRID_BG2=16
run KOT_TRD_GRID_BG=16 KOT_TRD_GRID_BG2=16
run KOT_TRD_GRID_FG=148
run KOT_TRD_GRID_FG=64
run KOT_MV_SPLIT=1
run KOT_MV_SPLIT=2
run KOT_MV_SPLIT=4
run KOT_CG_BATCH=8
run KOT_EIG_STAGES=3
run KOT_X=0
