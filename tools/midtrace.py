"""Per-warp clock64 trace of the sytrd mid kernel (argv: n, first columns, CTA)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

from paper_2310_14087_b200 import _lib, linalg

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
c0s = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [10, 600, 1200, 1700]
cta = int(sys.argv[3]) if len(sys.argv) > 3 else 0
L = _lib.lib()
rng = np.random.default_rng(0)
a = rng.standard_normal((n, n))
z = (a + a.T) / 2
linalg.sym_eig(z)
names = ["top", "symv done", "sync", "published", "update done", "gathered", "red1 sync", "red2 sync", "scal sync", "end", "s:sums", "s:sqrt", "s:div", "s:stores", "-", "-"]
for c0 in c0s:
    buf = (C.c_longlong * (8 * 16 * 16))()
    L.kot_debug_mid_trace(1, c0, cta, buf)
    linalg.sym_eig(z)
    L.kot_debug_mid_trace(0, c0, cta, buf)
    t = np.array(buf[:], dtype=np.int64).reshape(8, 16, 16)
    print(f"n={n} columns {c0}..{c0+7} CTA {cta}: cycles since the column's top (warp 0 | warp 7 | warp 15), mean over 8 columns")
    base = t[:, 0:1, 0:1]
    rel = (t - base).astype(float)
    rel[t == 0] = np.nan
    m = np.nanmean(rel, axis=0)
    for k, nm in enumerate(names):
        print(f"  {nm:12s} w0 {m[0, k]:8.0f}  w7 {m[7, k]:8.0f}  w15 {m[15, k]:8.0f}   max over warps {np.nanmax(m[:, k]):8.0f}")
    per_col = np.diff(t[:, 0, 0])
    print("  column period (cycles):", per_col)
