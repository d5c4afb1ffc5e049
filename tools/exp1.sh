B="python bench.py --no-cpu-baseline --no-ttt"
for a in 1 0; do
  echo "== cfg3 KOT_PIPE_ALPHA=$a" 
  KOT_PIPE_ALPHA=$a KOT_BENCH_DEBUG=1 timeout 300 $B 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value',d['value'],'e2e',d['e2e']['value'])
    else: print(l.rstrip()[:400])"
done
echo "== eigbench 2000"; timeout 200 python tools/eigbench.py 2000 2>&1 | head -30
for a in 1 0; do
  echo "== cfg4 KOT_PIPE_ALPHA=$a"
  KOT_PIPE_ALPHA=$a KOT_BENCH_DEBUG=1 timeout 400 $B --config cfg4 --steps 6 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value',d['value'],'e2e',d['e2e']['value'])
    else: print(l.rstrip()[:400])"
done
