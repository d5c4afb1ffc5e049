"""Small workload for compute-sanitizer (one tool per gpurun call): the cluster-resident sytrd tail
(DSMEM pushes), the cooperative panel kernel, the two-stage path (sb2st cluster flags), the TMA GEMM
core (mbarrier ring), the grouped D&C GEMMs and a short pipelined solve (EG contexts on their own
threads and streams)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2310_14087_b200 as K  # noqa: E402
from paper_2310_14087_b200 import _lib, configs, linalg, problem  # noqa: E402

rng = np.random.default_rng(0)
for n in (200, 700):  # tail only; panels + tail
    a = rng.standard_normal((n, n))
    z = 0.5 * (a + a.T)
    dc = linalg.sym_eig(z)
    print(n, "eig err", np.max(np.abs(dc.eigvals - np.sort(np.linalg.eigvalsh(z))[::-1])), flush=True)
L = _lib.lib()
L.kot_debug_eig_stages(2)
z = 0.5 * (lambda a: a + a.T)(rng.standard_normal((300, 300)))
dc = linalg.sym_eig(z)
print("two-stage 300 eig err", np.max(np.abs(dc.eigvals - np.sort(np.linalg.eigvalsh(z))[::-1])), flush=True)
L.kot_debug_eig_stages(0)
wl = configs.config3(n=256)
sx, sy, sxy = K.build_kernel_specs(wl.d, wl.bandwidth_sq)
pd = K.assemble(K.SampleSet(wl.xs), K.SampleSet(wl.ys), K.FillingPoints(wl.xt, wl.yt), wl.lambda1, wl.lambda2,
                sx, sy, sxy)
g = rng.standard_normal(256)
print("phi* sym", np.array_equal(problem.phi_adjoint(pd, g), problem.phi_adjoint(pd, g).T), flush=True)
step = configs.eg_stepsize(pd.q_mat, pd.pair_gram(), pd.lambda2)
rep = K.solve(pd, K.SolverConfig(eg=K.EgConfig(step), residual_tol=1e-12, max_iter=3))
print("solve", [t.res_accepted for t in rep.trace], flush=True)
