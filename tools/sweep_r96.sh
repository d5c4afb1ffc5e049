R96=$PWD/paper_2310_14087_b200/libkotgpu_r96.so
run() { echo "== $*"; env "$@" timeout 300 python bench.py --steps 16 --warmup 4 --no-ttt --no-cpu-baseline --no-batch 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); p=d['phases']; e=d['e2e']
        print(round(d['value'],2), 'it/s  e2e', round(e['value'],2), ' newton', round(p['host.newton']['ms_per_step'],1), 'trial', round(p['host.trial_resid']['ms_per_step'],1), 'eg', round(p['host.pipe_eg']['ms_per_step'],1), 'resid', round(p['host.pipe_resid']['ms_per_step'],1))
"; }
run KOT_X=0
run KOT_CARVEOUT=1
run KOT_LIB_PATH=$R96
run KOT_LIB_PATH=$R96 KOT_CARVEOUT=1
run KOT_LIB_PATH=$R96 KOT_CARVEOUT=1 KOT_TRD_GRID_BG=32 KOT_TRD_GRID_BG2=24
run KOT_X=0
run KOT_LIB_PATH=$R96 KOT_CARVEOUT=1
