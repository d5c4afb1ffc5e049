"""Where the e2e (solve from host arrays) time goes: setup vs per-iteration."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import paper_2310_14087_b200 as K
from paper_2310_14087_b200 import _lib, configs

wl = configs.config3()
sx, sy, sxy = K.build_kernel_specs(wl.d, wl.bandwidth_sq)
pd0 = K.assemble(K.SampleSet(wl.xs), K.SampleSet(wl.ys), K.FillingPoints(wl.xt, wl.yt), wl.lambda1, wl.lambda2,
                 sx, sy, sxy)
step = configs.eg_stepsize(pd0.q_mat, pd0.pair_gram(), pd0.lambda2)
import ctypes as C
for it in (1, 1, 5, 10, 20):
    pd = K.ProblemData(q_mat=pd0.q_mat.copy(), z=pd0.z.copy(), q_sq=pd0.q_sq, chol_upper=pd0.chol_upper.copy(),
                       lambda1=pd0.lambda1, lambda2=pd0.lambda2, embed_sum=pd0.embed_sum.copy())
    cfg = K.SolverConfig(eg=K.EgConfig(step), residual_tol=1e-300, max_iter=it)
    t0 = time.perf_counter()
    dp = pd.device_problem()
    t1 = time.perf_counter()
    rep = K.solve(pd, cfg)
    t2 = time.perf_counter()
    print(f"max_iter {it:3d}: upload {1e3*(t1-t0):7.1f} ms, solve {1e3*(t2-t1):8.1f} ms "
          f"({rep.iterations} it, {1e3*(t2-t1)/max(rep.iterations,1):6.1f} ms/it), total_ms {rep.total_ms:.1f}")
    del dp, pd
