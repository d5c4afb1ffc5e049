mkdir -p gpurun_out; rm -f gpurun_out/bench_tight.txt
for g in 96 112 128 148; do
  echo "== tight MID_GRID $g" >> gpurun_out/bench_tight.txt
  env KOT_TRD_MID_GRID=$g timeout 300 python bench.py --gpus 1 --steps 20 --warmup 10 --profile tight --no-batch --no-ttt --no-cpu-baseline 2>> gpurun_out/bench_mid.err | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value']); print({k:round(v['ms_per_step'],2) for k,v in sorted(d.get('phases',{}).items()) if v['ms_per_step']>0.05})" >> gpurun_out/bench_tight.txt 2>&1
done
python - > gpurun_out/assemble_prof.txt 2>&1 <<'PY'
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2310_14087_b200 as K
from paper_2310_14087_b200 import configs, _lib
wl = configs.config3()
sx, sy, sxy = K.build_kernel_specs(wl.d, wl.bandwidth_sq)
def asm():
    t0 = time.perf_counter()
    pd = K.assemble(K.SampleSet(wl.xs), K.SampleSet(wl.ys), K.FillingPoints(wl.xt, wl.yt), wl.lambda1, wl.lambda2, sx, sy, sxy)
    return pd, (time.perf_counter() - t0) * 1e3
pd, t = asm(); print("first assemble ms", t)
_lib.profile_enable(True)
pd2, t = asm(); print("second assemble ms", t)
prof = _lib.profile_read()
for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"]): print(f"  {k:20s} calls {v['calls']:4d} ms {v['ms']:8.3f}")
PY
