for e in "KOT_EG_PARALLEL=1" "KOT_EG_PARALLEL=0"; do for g in 32 24; do
echo "== $e grid $g"; env $e KOT_TRD_GRID=$g timeout 300 python bench.py --config cfg5 --batch 16 --max-iter 100 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('problems/s %.3f' % d['value'])"; done; done
