"""Where the e2e time outside the iterations goes (upload, setup, download)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import paper_2310_14087_b200 as K
from paper_2310_14087_b200 import configs
from paper_2310_14087_b200.solver import _run

wl = configs.config3()
sx, sy, sxy = K.build_kernel_specs(wl.d, wl.bandwidth_sq)
pd = K.assemble(K.SampleSet(wl.xs), K.SampleSet(wl.ys), K.FillingPoints(wl.xt, wl.yt), wl.lambda1, wl.lambda2,
                sx, sy, sxy)
step = configs.eg_stepsize(pd.q_mat, pd.pair_gram(), pd.lambda2)
cfg = K.SolverConfig(eg=K.EgConfig(step), residual_tol=1e-300, max_iter=2)
K.solve(pd, cfg)
pd.release_device()
for rep in range(3):
    ph = K.ProblemData(q_mat=pd.q_mat.copy(), z=pd.z.copy(), q_sq=pd.q_sq, chol_upper=pd.chol_upper.copy(),
                       lambda1=pd.lambda1, lambda2=pd.lambda2, embed_sum=pd.embed_sum.copy())
    t0 = time.perf_counter()
    ph.device_problem()
    t1 = time.perf_counter()
    r = _run(ph, cfg, None, False, want_x=False)
    t2 = time.perf_counter()
    r2 = _run(ph, cfg, None, False, want_x=True)
    t3 = time.perf_counter()
    print(f"upload {1e3*(t1-t0):.1f} ms; solve(2 it, no X) {1e3*(t2-t1):.1f} ms (lib {r.total_ms:.1f}); "
          f"solve(2 it, with X) {1e3*(t3-t2):.1f} ms (lib {r2.total_ms:.1f})", flush=True)
    ph.release_device()
