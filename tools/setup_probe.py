"""Where the first solve of a process spends its setup (e2e's setup_ms): host phase timers of the
library for a first and a second solve of cfg3 in one process (tools/setup_probe.py [config])."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2310_14087_b200 as K  # noqa: E402
from paper_2310_14087_b200 import _lib, configs  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
t0 = time.perf_counter()
_lib.lib()
print(f"library load {1e3 * (time.perf_counter() - t0):.1f} ms")
wl = configs.config3() if cfgname == "cfg3" else configs.config2()
sx, sy, sxy = K.build_kernel_specs(wl.d, wl.bandwidth_sq)
for rep in range(2):
    _lib.profile_enable(True, 2)
    t0 = time.perf_counter()
    pd = K.assemble(K.SampleSet(wl.xs), K.SampleSet(wl.ys), K.FillingPoints(wl.xt, wl.yt), wl.lambda1, wl.lambda2,
                    sx, sy, sxy, device=0)
    t_asm = time.perf_counter() - t0
    step = configs.eg_stepsize(pd.q_mat, pd.pair_gram(), pd.lambda2)
    t1 = time.perf_counter()
    r = K.solve(pd, K.SolverConfig(eg=K.EgConfig(step), residual_tol=1e-300, max_iter=2))
    t_solve = time.perf_counter() - t1
    prof = _lib.profile_read()
    _lib.profile_enable(False)
    steps = sum(x.step_ms for x in r.trace)
    print(f"solve #{rep}: assemble {1e3 * t_asm:.1f} ms, solve call {1e3 * t_solve:.1f} ms, total_ms {r.total_ms:.1f},"
          f" steps {steps:.1f} ({[round(x.step_ms, 1) for x in r.trace]}), setup {r.total_ms - steps:.1f} ms")
    for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"]):
        if k.startswith(("solve.", "host.", "asm", "problem")):
            print(f"   {k:20s} calls {v['calls']:4d}  {v['ms']:9.2f} ms")
    pd.release_device()
