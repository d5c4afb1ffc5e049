"""Isolated eigensolver timing (library phase profiler), n from argv."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import sys

import numpy as np

from paper_2310_14087_b200 import _lib, linalg

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
rng = np.random.default_rng(0)
q, _ = np.linalg.qr(rng.standard_normal((n, n)))
vals = np.concatenate([np.linspace(1, 100, n // 2), -np.linspace(1e-4, 1, n - n // 2)])
z = (q * vals) @ q.T
z = 0.5 * (z + z.T)
linalg.sym_eig(z)
_lib.profile_enable(True)
reps = 3
for _ in range(reps):
    dc = linalg.sym_eig(z)
prof = _lib.profile_read()
print(f"n={n}  max|eig err| = {np.max(np.abs(dc.eigvals - np.sort(vals)[::-1])):.2e}")
for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"]):
    tf = v["flops"] / (v["ms"] * 1e-3) / 1e12 if v["ms"] > 0 and v["flops"] > 0 else 0
    print(f"  {k:16s} calls/eig {v['calls']/reps:7.1f}  ms/eig {v['ms']/reps:9.3f}  {tf:6.2f} TF/s")

# per-segment timing of the sytrd panel kernel (CTA 0, thread 0)
import ctypes as C
L = _lib.lib()
buf = (C.c_ulonglong * 8)()
L.kot_debug_sytrd_timing(1, buf)
linalg.sym_eig(z)
L.kot_debug_sytrd_timing(0, buf)
names = ["Q:partials+prefetch", "Q:finish W", "Q:col update+partn", "grid.sync#1", "S:norm+householder",
         "S:scale+symv+partials", "S:part write", "grid.sync#2"]
tot = sum(buf) or 1
for nm, v in zip(names, buf):
    print(f"  {nm:24s} {v/1e6:8.3f} ms  {v/tot*100:5.1f}%  ({v/1e3/(n-1):.2f} us/col)")

# per-segment timing of the cluster-resident tail kernel (CTA 0 thread 0)
f = getattr(L, "kot_debug_tail_timing", None)
if f is not None:
    bt = (C.c_ulonglong * 8)()
    f(1, bt)
    linalg.sym_eig(z)
    f(0, bt)
    names = ["A:publish+norm", "cluster.sync#1", "B:gather+house", "B:Vall", "C:symv", "cluster.sync#2",
             "D:gather y+w", "E:rank-2 update"]
    for nm, v in zip(names, bt):
        print(f"  tail {nm:18s} {v / 1e6:8.3f} ms")

# per-segment cycles of the bulge-chasing kernel (every CTA × warp)
f = getattr(L, "kot_debug_sb2st_timing", None)
if f is not None:
    buf2 = (C.c_ulonglong * (16 * 32 * 8))()
    f(1, buf2)
    linalg.sym_eig(z)
    f(0, buf2)
    a = np.array(buf2[:], dtype=float).reshape(16, 32, 8)
    names = ["enum/idle", "load", "(1) C·Hp", "(2) house+bcast", "(3) C left", "(4) D two-sided", "store+slot",
             "cluster.sync"]
    busy = a[:, :, :7].sum(axis=2)
    print("  sb2st busy Mcyc per CTA (max over warps):", np.round(busy.max(axis=1) / 1e6, 2))
    print("  sb2st sync Mcyc per CTA (warp 0):", np.round(a[:, 0, 7] / 1e6, 2))
    w = np.unravel_index(np.argmax(busy), busy.shape)
    for k, nm in enumerate(names):
        print(f"  sb2st busiest warp {w}: {nm:18s} {a[w[0], w[1], k]/1e6:9.3f} Mcyc")
f = getattr(L, "kot_debug_pqr_timing", None)
if f is not None:
    b3 = (C.c_ulonglong * 8)()
    f(1, b3)
    linalg.sym_eig(z)
    f(0, b3)
    names = ["load+prologue", "sync#1", "gather+house", "dots", "sync#2", "gather+update", "next norm", "T+out+sync"]
    for nm, v in zip(names, b3):
        print(f"  panel {nm:16s} {v / 1e6:8.3f} Mcyc  ({v / max(1, (n // 16)) / 16:8.1f} cyc/col)")
