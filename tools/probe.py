"""Quick GPU probe: assemble a config, run a few SSN iterations with the phase profiler on."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import json
import sys
import time

import numpy as np

import paper_2310_14087_b200 as K
from paper_2310_14087_b200 import _lib, configs, solver

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
n = int(sys.argv[3]) if len(sys.argv) > 3 else None
wl = {"cfg1": configs.config1, "cfg2": configs.config2, "cfg3": configs.config3, "cfg4": configs.config4}[cfg_name]()
if n and cfg_name == "cfg3":
    wl = configs.config3(n=n)
sx, sy, sxy = K.build_kernel_specs(wl.d, wl.bandwidth_sq)
t0 = time.perf_counter()
pd = K.assemble(K.SampleSet(wl.xs), K.SampleSet(wl.ys), K.FillingPoints(wl.xt, wl.yt), wl.lambda1, wl.lambda2,
                sx, sy, sxy)
t_asm = time.perf_counter() - t0
step = configs.eg_stepsize(pd.q_mat, pd.pair_gram(), pd.lambda2)
print(f"{wl.name}: l={pd.n} assemble {t_asm*1e3:.1f} ms jitter {pd.jitter} eg_step {step:.3e}", flush=True)
cfg = K.SolverConfig(eg=K.EgConfig(step), residual_tol=1e-6, max_iter=10000)
se = solver.Session(pd, cfg)
se.step(1)
_lib.profile_enable(True)
t0 = time.perf_counter()
done = se.step(iters)
dt = time.perf_counter() - t0
prof = _lib.profile_read()
print(f"{done} iterations in {dt*1e3:.1f} ms -> {done/dt:.2f} it/s")
for r in se.records:
    print(f"  it {r.iteration}: res {r.res_accepted:.3e} acc {r.accepted} cg {r.cg_iters} att {r.attempts} "
          f"npos {r.n_pos} step {r.step_ms:.1f} ms (eg {r.eg_ms:.1f} newton {r.newton_ms:.1f} cg {r.cg_ms:.1f} "
          f"resid {r.resid_ms:.1f})")
for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"]):
    tf = v["flops"] / (v["ms"] * 1e-3) / 1e12 if v["ms"] > 0 and v["flops"] > 0 else 0
    print(f"  {k:16s} calls {v['calls']:6d}  ms {v['ms']:9.2f}  per-call {v['ms']/max(v['calls'],1):8.3f} ms  {tf:6.2f} TF/s")
