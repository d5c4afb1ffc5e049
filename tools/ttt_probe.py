"""Time-to-tolerance: solve() from host arrays to ‖R‖ ≤ tol (BASELINE metric part 1)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import paper_2310_14087_b200 as K
from paper_2310_14087_b200 import configs

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
profile = sys.argv[2] if len(sys.argv) > 2 else "tight"
tol = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-6
max_iter = int(sys.argv[4]) if len(sys.argv) > 4 else 2000
wl = (configs.config5_member(int(cfg_name.split(":")[1])) if cfg_name.startswith("cfg5")
      else {"cfg1": configs.config1, "cfg2": configs.config2, "cfg3": configs.config3}[cfg_name]())
sx, sy, sxy = K.build_kernel_specs(wl.d, wl.bandwidth_sq)
t0 = time.perf_counter()
pd = K.assemble(K.SampleSet(wl.xs), K.SampleSet(wl.ys), K.FillingPoints(wl.xt, wl.yt), wl.lambda1, wl.lambda2,
                sx, sy, sxy)
step = configs.eg_stepsize(pd.q_mat, pd.pair_gram(), pd.lambda2)
t1 = time.perf_counter()
cfg = K.SolverConfig(newton=K.NewtonConfig(**configs.PROFILES[profile]), eg=K.EgConfig(step), residual_tol=tol,
                     max_iter=max_iter)
rep = K.solve(pd, cfg)
t2 = time.perf_counter()
res = [r.res_accepted for r in rep.trace]
first = next((i for i, r in enumerate(res) if r <= tol), None)
cg = [r.cg_iters for r in rep.trace]
print(f"{cfg_name} {profile} tol {tol}: {rep.termination} after {rep.iterations} iterations; assemble {t1-t0:.2f} s, "
      f"solve {t2-t1:.2f} s ({rep.iterations/(t2-t1):.2f} it/s), first ≤tol at {first}; mean CG {np.mean(cg):.1f}; "
      f"final res {rep.residual_norm:.3e}; ot {rep.ot_estimate:.6f}; EG accepted "
      f"{sum(1 for r in rep.trace if r.accepted != 'ssn')}; min res {min(res):.3e}")
