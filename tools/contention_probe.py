"""Newton-chain cost with and without the concurrent EG safeguard pipeline (cfg3).

safeguard_every=10**6 stalls the pipeline after its 4-slot ring fills, so the
Newton chain then runs alone: the difference is what co-running costs it."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import time

import paper_2310_14087_b200 as K
from paper_2310_14087_b200 import _lib, configs, solver

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
wl = configs.config3(n=n)
sx, sy, sxy = K.build_kernel_specs(wl.d, wl.bandwidth_sq)
pd = K.assemble(K.SampleSet(wl.xs), K.SampleSet(wl.ys), K.FillingPoints(wl.xt, wl.yt), wl.lambda1, wl.lambda2,
                sx, sy, sxy)
step = configs.eg_stepsize(pd.q_mat, pd.pair_gram(), pd.lambda2)
for every in (1, 10 ** 6):
    cfg = K.SolverConfig(newton=K.NewtonConfig(), eg=K.EgConfig(step), residual_tol=1e-300, max_iter=10 ** 6,
                         safeguard_every=every)
    se = solver.Session(pd, cfg)
    se.step(8)
    _lib.profile_enable(True)
    t0 = time.perf_counter()
    se.step(10)
    dt = time.perf_counter() - t0
    prof = _lib.profile_read()
    _lib.profile_enable(False)
    se.close()
    print(f"safeguard_every={every}: {dt / 10 * 1e3:.1f} ms/iter")
    for k in ("ssn_iteration", "newton", "newton.prologue", "matvec", "newton.criterion", "residual", "eigh",
              "eig.sytrd", "host.trial_resid", "host.newton"):
        if k in prof:
            v = prof[k]
            print(f"   {k:18s} {v['ms'] / 10:8.2f} ms/iter  calls {v['calls'] / 10:6.1f}")
