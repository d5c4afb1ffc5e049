"""One n=2000 eigensolve after one warm-up (for ncu launch lists)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2310_14087_b200 import linalg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
rng = np.random.default_rng(0)
q, _ = np.linalg.qr(rng.standard_normal((n, n)))
vals = np.concatenate([np.linspace(1, 100, n // 2), -np.linspace(1e-4, 1, n - n // 2)])
z = (q * vals) @ q.T
z = 0.5 * (z + z.T)
linalg.sym_eig(z)
linalg.sym_eig(z)
