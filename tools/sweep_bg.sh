run() { echo "== $*"; env "$@" timeout 300 python bench.py --steps 12 --warmup 3 --no-ttt --no-cpu-baseline --no-batch 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); p=d['phases']
        print(round(d['value'],2), 'it/s  e2e', round(d['e2e']['value'],2), ' newton', round(p['host.newton']['ms_per_step'],1), 'trial', round(p['host.trial_resid']['ms_per_step'],1), 'eg', round(p['host.pipe_eg']['ms_per_step'],1), 'resid', round(p['host.pipe_resid']['ms_per_step'],1))
"; }
run KOT_BG_GEMM_CTAS=0
run KOT_BG_GEMM_CTAS=96
run KOT_BG_GEMM_CTAS=64
run KOT_BG_GEMM_CTAS=32
run KOT_BG_GEMM_CTAS=16
run KOT_BG_GEMM_CTAS=48 KOT_TRD_GRID_BG=32 KOT_TRD_GRID_BG2=24
run KOT_BG_GEMM_CTAS=0
