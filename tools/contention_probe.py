"""Newton-chain cost with and without the concurrent EG safeguard chain (cfg3, diagnostic):
safeguard_every=10**6 runs the EG step only at iteration 0, so later iterations time the Newton chain
(Newton direction + trial residual) alone on the GPU."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2310_14087_b200 as K  # noqa: E402
from paper_2310_14087_b200 import _lib, configs, solver  # noqa: E402

wl = configs.config3()
sx, sy, sxy = K.build_kernel_specs(wl.d, wl.bandwidth_sq)
pd = K.assemble(K.SampleSet(wl.xs), K.SampleSet(wl.ys), K.FillingPoints(wl.xt, wl.yt), wl.lambda1, wl.lambda2,
                sx, sy, sxy)
step = configs.eg_stepsize(pd.q_mat, pd.pair_gram(), pd.lambda2)
for every in (1, 10 ** 6):
    cfg = K.SolverConfig(eg=K.EgConfig(step), residual_tol=1e-300, max_iter=10 ** 6, safeguard_every=every)
    se = solver.Session(pd, cfg)
    se.step(4)
    _lib.profile_enable(True, 1)
    t0 = time.perf_counter()
    se.step(8)
    dt = time.perf_counter() - t0
    prof = _lib.profile_read()
    _lib.profile_enable(False)
    se.close()
    pick = {k: round(prof[k]["ms"] / 8, 2) for k in ("host.newton", "host.trial_resid", "matvec", "newton.criterion",
                                                       "eigh", "sytrd_panel") if k in prof}
    mv = prof.get("matvec", {"calls": 1})["calls"] / 8
    print(f"safeguard_every={every}: {8 / dt:.2f} it/s  per iteration {pick}  matvecs/it {mv:.1f}", flush=True)
