# config-5 batch rate at the paper threshold (tight profile), several concurrency levels
for c in 6 8 12; do
  echo "== concurrency $c"
  timeout 600 python bench.py --config cfg5 --batch 64 --max-iter 100 --tol 5e-3 --profile tight --concurrency $c 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(round(d['value'],3),'problems/s', d['converged'],'converged', sum(d['iterations']),'iterations', d['clocks'])
"
done
