# config-5 batch: panel grid cap and concurrency (64 members, tol 5e-3, tight profile)
run() { echo "== $*"; env "$@" timeout 600 python bench.py --config cfg5 --batch 64 --max-iter 100 --tol 5e-3 --profile tight --concurrency ${CONC:-6} 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); b=d['batch']; print(round(d['value'],3),'problems/s', b['converged'],'converged', b['iterations_mean'],'it/problem')
"; }
run KOT_BATCH_GRID=32
run KOT_BATCH_GRID=16
run KOT_BATCH_GRID=24
CONC=8 run KOT_BATCH_GRID=16
CONC=4 run KOT_BATCH_GRID=16
