mkdir -p gpurun_out; rm -f gpurun_out/bench_tight.txt
for t in 2 3 4 6; do
for p in paper tight; do
  echo "== $p throttle $t" >> gpurun_out/bench_tight.txt
  env KOT_TRD_THROTTLE=$t timeout 300 python bench.py --gpus 1 --steps 20 --warmup 10 --profile $p --no-batch --no-ttt --no-cpu-baseline 2>> gpurun_out/bench_mid.err | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value']); print({k:round(v['ms_per_step'],2) for k,v in sorted(d.get('phases',{}).items()) if v['ms_per_step']>0.05})" >> gpurun_out/bench_tight.txt 2>&1
done
done
