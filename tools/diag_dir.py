"""Newton direction at replay state i: compare GPU (current eig config) with the oracle per CG attempt."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import paper_2310_14087_b200 as K
from paper_2310_14087_b200 import newton as GN, problem as GP
from oracle import kot_port as O

d = dict(np.load(os.path.join(ROOT, "tests", "golden", "cfg1.npz")))
i = int(sys.argv[1]) if len(sys.argv) > 1 else 2
pd = GP.ProblemData(q_mat=d["q"], z=d["z"], q_sq=float(d["q_sq"]), chol_upper=d["r"], lambda1=float(d["l1"]),
                    lambda2=float(d["l2"]), embed_sum=d.get("embed"))
po = O.Problem(q=d["q"], z=d["z"], q_sq=float(d["q_sq"]), r=d["r"], l1=float(d["l1"]), l2=float(d["l2"]),
               embed=d.get("embed"))
w = GP.IteratePair(d[f"rp{i}_wg"], d[f"rp{i}_wx"])
theta = float(d[f"rp{i}_theta"])
r, dc = O.residual_parts(po, O.Pair(w.gamma, w.x_mat))
ctx = O.newton_context(dc, r.norm(), theta)
for cgmax, rest in ((20, 0), (40, 0), (20, 2), (3000, 0)):
    cfgg = K.NewtonConfig(cg_max=cgmax, cg_restarts=rest, **({"cg_tol": 1e-14} if cgmax == 3000 else {}))
    cfgo = O.NewtonCfg(cg_max=cgmax, cg_restarts=rest, **({"cg_tol": 1e-14} if cgmax == 3000 else {}))
    st = GN.newton_direction_at(pd, w, theta, cfgg)
    so = O.newton_direction(po, r, ctx, cfgo)
    rel = np.linalg.norm(st.dw.gamma - so.dw.g) / np.linalg.norm(so.dw.g)
    print(f"cg_max {cgmax} restarts {rest}: gpu cg {st.cg_iters} lhs {st.crit_lhs:.4e} | oracle cg {so.cg_iters} "
          f"lhs {so.lhs:.4e} | rel dg {rel:.2e}")
v = np.random.default_rng(0).standard_normal(pd.n)
out, mu = GN.middle_operator_at(pd, w, theta, v)
ref = O.middle_operator(po, ctx.op, ctx.mu)(v)
print("middle op rel", np.linalg.norm(out - ref) / np.linalg.norm(ref))
for cgmax, rest in ((20, 1), (20, 1)):
    st = GN.newton_direction_at(pd, w, theta, K.NewtonConfig(cg_max=cgmax, cg_restarts=rest))
    so = O.newton_direction(po, r, ctx, O.NewtonCfg(cg_max=cgmax, cg_restarts=rest))
    print(f"2 attempts: gpu cg {st.cg_iters} lhs {st.crit_lhs:.6e} oracle lhs {so.lhs:.6e} rel dg "
          f"{np.linalg.norm(st.dw.gamma - so.dw.g) / np.linalg.norm(so.dw.g):.2e}")
from paper_2310_14087_b200 import linalg as GL
zarg = O.sym(w.x_mat) - O.constraint_matrix(po, w.gamma)
g = GL.sym_eig(zarg)
P = g.eigvecs
Pn = dc.vecs
ov = np.abs(P.T @ Pn)
print("basis overlap: min diag", ov.diagonal().min(), "max offdiag", (ov - np.diag(ov.diagonal())).max())
gaps = np.diff(np.sort(dc.vals))
print("min eigen gap", gaps.min())
# oracle direction using the GPU decomposition of Z (instead of LAPACK's)
dg_ = O.Decomp(vecs=g.eigvecs.copy(), vals=g.eigvals.copy(), k=int(np.count_nonzero(g.eigvals > 0)))
r_g = O.Pair(r.g, w.x_mat - O.proj(dg_))
ctx_g = O.newton_context(dg_, r_g.norm(), theta)
so2 = O.newton_direction(po, r_g, ctx_g, O.NewtonCfg(cg_max=20, cg_restarts=1))
print(f"oracle with GPU decomposition: lhs {so2.lhs:.6e}")
# and with a random rotation inside each near-degenerate pair (gap < 1e-4)
vals = dc.vals
V = dc.vecs.copy()
rng = np.random.default_rng(1)
for a in range(len(vals) - 1):
    if abs(vals[a] - vals[a + 1]) < 1e-4:
        th = rng.uniform(-1e-10, 1e-10)
        c, s = np.cos(th), np.sin(th)
        V[:, [a, a + 1]] = V[:, [a, a + 1]] @ np.array([[c, -s], [s, c]])
dr = O.Decomp(vecs=V, vals=vals.copy(), k=dc.k)
so3 = O.newton_direction(po, O.Pair(r.g, w.x_mat - O.proj(dr)), O.newton_context(dr, r.norm(), theta),
                         O.NewtonCfg(cg_max=20, cg_restarts=1))
print(f"oracle with 1e-10 rotations in close pairs: lhs {so3.lhs:.6e}")
print("‖P_gpu − P_np (sign-aligned)‖ per column max:",
      np.max(np.linalg.norm(g.eigvecs * np.sign(np.sum(g.eigvecs * dc.vecs, 0)) - dc.vecs, axis=0)))
