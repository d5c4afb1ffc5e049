"""Diagnostic: tight-profile cfg1 solve to 1e-10 on the GPU, iteration count + residual checkpoints."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np

import paper_2310_14087_b200 as K
from paper_2310_14087_b200 import problem as GP

import sys

d = dict(np.load("tests/golden/cfg1.npz"))
seed = int(sys.argv[1]) if len(sys.argv) > 1 else 0
r = d["r"]
if seed:
    rng = np.random.default_rng(seed)
    r = r * (1.0 + rng.choice([-1.0, 1.0], r.shape) * 2.2e-16)
pd = GP.ProblemData(q_mat=d["q"], z=d["z"], q_sq=float(d["q_sq"]), chol_upper=r, lambda1=float(d["l1"]),
                    lambda2=float(d["l2"]), embed_sum=d["embed"])
cfg = K.SolverConfig(newton=K.NewtonConfig(alpha1=1e-8, alpha2=1e-4, cg_max=500), eg=K.EgConfig(float(d["eg_stepsize"])),
                     residual_tol=1e-10, max_iter=1000)
rep = K.solve(pd, cfg)
res = np.array([t.res_accepted for t in rep.trace])
hit = np.nonzero(res <= 1e-6)[0]
print("seed", seed, "iterations", rep.iterations, "first<=1e-6", hit[0] + 1 if hit.size else None, "ref", int(d["tight_iters"]),
      int(d["tight_first_1e6"]))
ref = d["tight_res_accepted"]
for k in ():
    if k < len(res):
        print(f"  it {k}: gpu {res[k]:.3e}  ref {ref[k] if k < len(ref) else float('nan'):.3e}  cg {rep.trace[k].cg_iters} "
              f"ref cg {d['tight_cg_iters'][k] if k < len(ref) else -1}")
