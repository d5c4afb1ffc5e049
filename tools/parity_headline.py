"""Trace parity at the headline size (cfg3, l = 2000, paper profile): the GPU solver and the NumPy
oracle (restatement of the reference) from the same host instance, first K iterations side by side.

The trajectory is chaotic (±2-ulp perturbations of R move the residual trace by
>1e-6 relative within a few iterations), so the expected agreement is tight for the first iterations
and then within the oracle's own ulp spread; CG counts and accept decisions must match.
python tools/parity_headline.py [K] [l]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import paper_2310_14087_b200 as K
from oracle import kot_port as O
from paper_2310_14087_b200 import configs

k_it = int(sys.argv[1]) if len(sys.argv) > 1 else 6
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
wl = configs.config3(n=n)
sx, sy, sxy = K.build_kernel_specs(wl.d, wl.bandwidth_sq)
pd = K.assemble(K.SampleSet(wl.xs), K.SampleSet(wl.ys), K.FillingPoints(wl.xt, wl.yt), wl.lambda1, wl.lambda2,
                sx, sy, sxy)
step = configs.eg_stepsize(pd.q_mat, pd.pair_gram(), pd.lambda2)
t0 = time.perf_counter()
rep = K.solve(pd, K.SolverConfig(eg=K.EgConfig(step), residual_tol=1e-300, max_iter=k_it))
t_gpu = time.perf_counter() - t0
po = O.Problem(q=pd.q_mat, z=pd.z, q_sq=pd.q_sq, r=pd.chol_upper, l1=pd.lambda1, l2=pd.lambda2, embed=pd.embed_sum)
t0 = time.perf_counter()
orep = O.solve(po, O.SolverCfg(eg_stepsize=step, residual_tol=1e-300, max_iter=k_it))
t_cpu = time.perf_counter() - t0
# the oracle's own sensitivity: the same solve with R perturbed by ±1 ulp (relative 2.2e-16)
rng = np.random.default_rng(1)
pp = O.Problem(q=pd.q_mat, z=pd.z, q_sq=pd.q_sq, r=pd.chol_upper * (1 + rng.choice([-1.0, 1.0], pd.chol_upper.shape)
               * 2.2e-16), l1=pd.lambda1, l2=pd.lambda2, embed=pd.embed_sum)
prep = O.solve(pp, O.SolverCfg(eg_stepsize=step, residual_tol=1e-300, max_iter=k_it))
print(f"cfg3 l={n}: {k_it} iterations, GPU {t_gpu:.2f} s, oracle {t_cpu:.1f} s")
print(" it  accepted    res (GPU)               res (oracle)            GPU-oracle  1ulp-oracle  cg GPU/oracle/1ulp")
for g, o, u in zip(rep.trace, orep.trace, prep.trace):
    d = abs(g.res_accepted - o.res_accepted) / abs(o.res_accepted)
    du = abs(u.res_accepted - o.res_accepted) / abs(o.res_accepted)
    print(f"{g.iteration:3d}  {g.accepted:>3s}/{o.accepted:<3s}  {g.res_accepted:.17g}  {o.res_accepted:.17g}  "
          f"{d:.1e}     {du:.1e}      {g.cg_iters:3d}/{o.cg_iters:<3d}/{u.cg_iters:<3d}")
print(f"gamma rel diff {np.linalg.norm(rep.gamma_hat - orep.gamma) / np.linalg.norm(orep.gamma):.2e}, "
      f"objective rel diff {abs(K.objective(pd, rep.gamma_hat) - O.objective(po, orep.gamma)) / abs(O.objective(po, orep.gamma)):.2e}")
