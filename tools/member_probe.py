"""Solve config-5 members one at a time (diagnostic): python tools/member_probe.py SEED [MAX_ITER] [PROFILE]."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import time

from paper_2310_14087_b200 import batch

seed = int(sys.argv[1])
mi = int(sys.argv[2]) if len(sys.argv) > 2 else 100
prof = sys.argv[3] if len(sys.argv) > 3 else "paper"
t0 = time.perf_counter()
r = batch.gpu_solve_member(seed, dict(profile=prof, residual_tol=1e-6, max_iter=mi), 0)
print(f"seed {seed}: it {r.iterations} conv {r.converged} res {r.residual_norm:.3e} {time.perf_counter() - t0:.1f}s",
      flush=True)
