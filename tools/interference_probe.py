"""Which background work slows the Newton chain (diagnostic): the cfg3 Newton chain alone
(safeguard_every=10**6) while a background host thread loops (a) l=2000 eigensolves, (b) l=2000 GEMMs
(phi_adjoint), (c) nothing."""
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2310_14087_b200 as K  # noqa: E402
from paper_2310_14087_b200 import _lib, configs, linalg, problem, solver  # noqa: E402

wl = configs.config3()
sx, sy, sxy = K.build_kernel_specs(wl.d, wl.bandwidth_sq)
pd = K.assemble(K.SampleSet(wl.xs), K.SampleSet(wl.ys), K.FillingPoints(wl.xt, wl.yt), wl.lambda1, wl.lambda2,
                sx, sy, sxy)
pd2 = K.assemble(K.SampleSet(wl.xs), K.SampleSet(wl.ys), K.FillingPoints(wl.xt, wl.yt), wl.lambda1, wl.lambda2,
                 sx, sy, sxy)
step = configs.eg_stepsize(pd.q_mat, pd.pair_gram(), pd.lambda2)
rng = np.random.default_rng(0)
a = rng.standard_normal((2000, 2000))
z = 0.5 * (a + a.T)
g = rng.standard_normal(2000)



def bg_loop(kind, stop):
    n = 0
    while not stop.is_set():
        if kind == "eig":
            linalg.sym_eig(z)
        elif kind == "gemm":
            problem.phi_adjoint(pd2, g)
        n += 1
    return n


for kind in ("none", "eig", "gemm", "none"):
    cfg = K.SolverConfig(eg=K.EgConfig(step), residual_tol=1e-300, max_iter=10 ** 6, safeguard_every=10 ** 6)
    se = solver.Session(pd, cfg)
    se.step(3)
    stop = threading.Event()
    th = threading.Thread(target=bg_loop, args=(kind, stop)) if kind != "none" else None
    if th:
        th.start()
        time.sleep(0.5)
    _lib.profile_enable(True, 1)
    t0 = time.perf_counter()
    se.step(6)
    dt = time.perf_counter() - t0
    prof = _lib.profile_read()
    _lib.profile_enable(False)
    stop.set()
    if th:
        th.join()
    se.close()
    pick = {k: round(prof[k]["ms"] / 6, 2) for k in ("host.newton", "host.trial_resid", "matvec") if k in prof}
    print(f"background={kind}: {6 / dt:.2f} it/s  per iteration {pick}", flush=True)
