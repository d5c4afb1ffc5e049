"""Replay state i of the cfg1 golden fixture: GPU record vs oracle ensembles (knife-edge diagnosis)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np

import paper_2310_14087_b200 as K
from paper_2310_14087_b200 import problem as GP, solver as GS, linalg as GL
from paper_2310_14087_b200.eg import EgConfig
from oracle import kot_port as O

d = dict(np.load(os.path.join(ROOT, "tests", "golden", "cfg1.npz")))
i = int(sys.argv[1]) if len(sys.argv) > 1 else 2
pd = GP.ProblemData(q_mat=d["q"], z=d["z"], q_sq=float(d["q_sq"]), chol_upper=d["r"], lambda1=float(d["l1"]),
                    lambda2=float(d["l2"]), embed_sum=d.get("embed"))
cfg = K.SolverConfig(eg=EgConfig(float(d["eg_stepsize"])), residual_tol=1e-12, max_iter=40)
ocfg = O.SolverCfg(eg_stepsize=float(d["eg_stepsize"]), residual_tol=1e-12, max_iter=40)
w = GP.IteratePair(d[f"rp{i}_wg"], d[f"rp{i}_wx"])
v = GP.IteratePair(d[f"rp{i}_vg"], d[f"rp{i}_vx"])
theta = float(d[f"rp{i}_theta"])
w2, v2, th2, rec = GS.iterate(pd, cfg, w, v, theta, i)
print(f"GPU: cg {rec.cg_iters} att {rec.attempts} lhs {rec.crit_lhs:.6e} rhs {rec.crit_rhs:.6e} acc {rec.accepted}")
print(f"ref: cg {int(d['paper_cg_iters'][i])}")
for eps in (1e-13, 1e-12, 1e-11):
    out = []
    for seed in (11, 12, 13, 14, 15, 16):
        rng = np.random.default_rng(seed)
        r = d["r"] * (1.0 + rng.choice([-1.0, 1.0], d["r"].shape) * eps)
        po = O.Problem(q=d["q"], z=d["z"], q_sq=float(d["q_sq"]), r=r, l1=float(d["l1"]), l2=float(d["l2"]),
                       embed=d.get("embed"))
        ow = O.Pair(w.gamma.copy(), w.x_mat.copy())
        r_w, dc_w = O.residual_parts(po, ow)
        st0 = O.State(ow, O.Pair(v.gamma.copy(), v.x_mat.copy()), r_w, dc_w, r_w.norm(), None, None, r_w.norm(),
                      theta)
        ost, orec, _ = O.iterate_once(po, st0, i, ocfg)
        out.append((orec.cg_iters, f"{orec.crit_lhs:.4e}/{orec.crit_rhs:.4e}"))
    print(f"oracle eps={eps:g}:", out)
# eigensolver accuracy on the residual matrix at w
rng = np.random.default_rng(0)
for n in (100, 300, 1000):
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.sort(rng.standard_normal(n))[::-1]
    z = (q * lam) @ q.T
    z = 0.5 * (z + z.T)
    dc = GL.sym_eig(z)
    P, vals = dc.eigvecs, dc.eigvals
    print(f"n={n}: recon {np.linalg.norm(P @ np.diag(vals) @ P.T - z) / np.linalg.norm(z):.2e} "
          f"orth {np.linalg.norm(P.T @ P - np.eye(n)):.2e} vals {np.max(np.abs(vals - lam)):.2e}")

# spectrum of Z at w (and at the Newton trial point) near zero: numpy vs GPU
po = O.Problem(q=d["q"], z=d["z"], q_sq=float(d["q_sq"]), r=d["r"], l1=float(d["l1"]), l2=float(d["l2"]),
               embed=d.get("embed"))
zarg = O.sym(w.x_mat) - O.constraint_matrix(po, w.gamma)
ref = np.sort(np.linalg.eigvalsh(zarg))[::-1]
g = GL.sym_eig(zarg)
print("k numpy", int(np.sum(ref > 0)), "k gpu", int(np.sum(g.eigvals > 0)))
idx = np.argsort(np.abs(ref))[:6]
print("smallest |σ| numpy:", ref[idx])
print("gpu at same idx:  ", g.eigvals[idx])
print("max |Δσ|", np.max(np.abs(g.eigvals - ref)), "‖Z‖", np.abs(ref).max())
pr = GL.proj_psd(zarg) if hasattr(GL, "proj_psd") else None
