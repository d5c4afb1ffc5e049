"""Reproduce bench.py's e2e leg: Session steps on problem A, then solve() on a fresh host copy B."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2310_14087_b200 as K
from paper_2310_14087_b200 import configs, solver

wl = configs.config3()
sx, sy, sxy = K.build_kernel_specs(wl.d, wl.bandwidth_sq)
pd = K.assemble(K.SampleSet(wl.xs), K.SampleSet(wl.ys), K.FillingPoints(wl.xt, wl.yt), wl.lambda1, wl.lambda2,
                sx, sy, sxy)
step = configs.eg_stepsize(pd.q_mat, pd.pair_gram(), pd.lambda2)
cfg = K.SolverConfig(eg=K.EgConfig(step), residual_tol=1e-300, max_iter=10 ** 6)
se = solver.Session(pd, cfg)
t0 = time.perf_counter()
se.step(13)
print(f"session 13 steps {time.perf_counter() - t0:.2f} s")
se.close()
for trial in range(3):
    pdh = K.ProblemData(q_mat=pd.q_mat.copy(), z=pd.z.copy(), q_sq=pd.q_sq, chol_upper=pd.chol_upper.copy(),
                        lambda1=pd.lambda1, lambda2=pd.lambda2, embed_sum=pd.embed_sum.copy())
    cfg_e = K.SolverConfig(eg=K.EgConfig(step), residual_tol=1e-300, max_iter=10)
    t0 = time.perf_counter()
    dp = pdh.device_problem()
    t1 = time.perf_counter()
    rep = K.solve(pdh, cfg_e)
    t2 = time.perf_counter()
    print(f"e2e trial {trial}: upload {1e3*(t1-t0):.1f} ms, solve {1e3*(t2-t1):.1f} ms, total_ms {rep.total_ms:.1f}, "
          f"first step {rep.trace[0].step_ms:.1f} ms, steps {[round(r.step_ms) for r in rep.trace]}")
    del dp, pdh
