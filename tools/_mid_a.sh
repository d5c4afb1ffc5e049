mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/bench_mid.txt
for v in "KOT_TRD_MID=1" "KOT_TRD_MID=1 KOT_TRD_GRID_BG=32 KOT_TRD_GRID_BG2=24" "KOT_TRD_MID=1 KOT_TRD_GRID_BG=16 KOT_TRD_GRID_BG2=16" "KOT_TRD_MID=1 KOT_TRD_GRID_FG=128" "KOT_TRD_MID=1 KOT_TRD_MID_GRID=148" "KOT_TRD_MID=1 KOT_TRD_MID_GRID=64"; do
  echo "== $v" >> gpurun_out/bench_mid.txt
  env $v timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --no-batch --no-ttt --no-cpu-baseline 2>> gpurun_out/bench_mid.err | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], {k:round(v['ms_per_step'],2) for k,v in d.get('phases',{}).items() if k.startswith('host.') or k in ('sytrd_mid','sytrd_panel','eigh')})" >> gpurun_out/bench_mid.txt 2>&1
done
