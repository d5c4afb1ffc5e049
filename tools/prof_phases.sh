# per-phase breakdown of the cfg3 iteration (every library scope timed; ~14 % slower than the bench)
KOT_BENCH_PROFILE=full timeout 300 python bench.py --steps 10 --warmup 3 --no-ttt --no-cpu-baseline 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l)
        print('it/s', round(d['value'],2))
        for k,v in sorted(d['phases'].items(), key=lambda kv:-kv[1]['ms_per_step']):
            print(f\"{k:32s} {v['ms_per_step']:8.2f} ms/it  {v['calls_per_step']:8.1f} calls/it  {v.get('tflops','')}\")
"
