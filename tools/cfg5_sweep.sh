# config-5 batch variants (64 members, paper threshold, tight profile)
run() { echo "== $*"; env "$@" timeout 600 python bench.py --config cfg5 --batch 64 --max-iter 100 --tol 5e-3 --profile tight 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); b=d['batch']; print(round(d['value'],3),'problems/s', b['converged'],'converged', b['iterations_mean'],'it/problem')
"; }
run KOT_X=0
run KOT_EG_PARALLEL=0
run KOT_NO_PIPE=1
run KOT_NO_PIPE=1 KOT_EG_PARALLEL=0
