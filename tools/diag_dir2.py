import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import paper_2310_14087_b200 as K
from paper_2310_14087_b200 import newton as GN, problem as GP

d = dict(np.load(os.path.join(ROOT, "tests", "golden", "cfg1.npz")))
i = int(sys.argv[1]) if len(sys.argv) > 1 else 2
pd = GP.ProblemData(q_mat=d["q"], z=d["z"], q_sq=float(d["q_sq"]), chol_upper=d["r"], lambda1=float(d["l1"]),
                    lambda2=float(d["l2"]), embed_sum=d.get("embed"))
theta = float(d[f"rp{i}_theta"])
rng = np.random.default_rng(0)
for eps in (0.0, 1e-14, 1e-13, 1e-12):
    x = d[f"rp{i}_wx"] * (1 + eps * rng.standard_normal(d[f"rp{i}_wx"].shape))
    x = 0.5 * (x + x.T)
    w = GP.IteratePair(d[f"rp{i}_wg"], x)
    st = GN.newton_direction_at(pd, w, theta, K.NewtonConfig(cg_max=20, cg_restarts=1))
    print(f"eps {eps:g}: lhs {st.crit_lhs:.6e} cg {st.cg_iters}")
