"""Diagnostic: accuracy of the GPU eigensolver / PSD projection on the first EG argument of config-5
member 0 (σ = 0.5): A = −s·C(ĝ), spectrum [−1.4e-8, 4.8e-10], 11 positive eigenvalues."""
import numpy as np

from oracle import kot_port as O
from paper_2310_14087_b200 import configs
from paper_2310_14087_b200 import linalg as GL
from paper_2310_14087_b200 import psdcone as GC

wl = configs.config5_member(0)
po, kmat = O.assemble(wl.xs, wl.ys, wl.xt, wl.yt, wl.lambda1, wl.lambda2, wl.bandwidth_sq)
s = configs.eg_stepsize(po.q, kmat, po.l2)
g0 = np.zeros(po.q.shape[0])
x0 = np.zeros_like(po.q)
gv = O.objective_grad(po, g0) - O.phi(po, x0)
gh = g0 - s * gv
A = O.sym(-s * O.constraint_matrix(po, gh))
P = O.proj_psd(A)
ref = np.linalg.eigvalsh(A)
for scale in (1.0, 1e8):
    B = A * scale
    dc = GL.sym_eig(B)
    V, lam = dc.eigvecs, dc.eigvals
    nb = np.linalg.norm(B, 2)
    print(f"scale {scale:g}: orth {np.abs(V.T @ V - np.eye(len(lam))).max():.2e} "
          f"recon {np.abs((V * lam) @ V.T - B).max() / nb:.2e} eigerr {np.abs(np.sort(lam) - ref * scale).max() / nb:.2e} "
          f"k {dc.n_pos} vs {(ref > 0).sum()}")
    Pg = GC.proj_psd(B) / scale
    print(f"   proj rel {np.linalg.norm(Pg - P) / np.linalg.norm(P):.2e}  top eig gpu {np.sort(lam)[-3:] / scale} ref {ref[-3:]}")
