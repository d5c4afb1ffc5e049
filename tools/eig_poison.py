"""Eigensolver on fresh (poisoned) workspaces at several orders (diagnostic, KOT_POISON)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

from paper_2310_14087_b200 import linalg

for n in [int(a) for a in sys.argv[1:]]:
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n))
    z = a + a.T
    dc = linalg.sym_eig(z)
    ref = np.linalg.eigvalsh(z)[::-1]
    print(n, f"{np.max(np.abs(dc.eigvals - ref)) / np.abs(ref).max():.2e}", flush=True)
