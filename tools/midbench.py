"""Grid-resident sytrd mid kernel: correctness against LAPACK over sizes / hand-over points, and the
isolated eigensolve time with and without it (argv: sizes; default a sweep + 2000)."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np

from paper_2310_14087_b200 import _lib, linalg

L = _lib.lib()
rng = np.random.default_rng(3)


def check(z, tag):
    dc = linalg.sym_eig(z)
    n = z.shape[0]
    ref = np.linalg.eigvalsh(z)[::-1]
    p = dc.eigvecs
    nz = max(1.0, np.max(np.abs(ref)))
    ev = np.max(np.abs(dc.eigvals - ref)) / nz
    orth = np.max(np.abs(p.T @ p - np.eye(n)))
    rec = np.max(np.abs((p * dc.eigvals) @ p.T - z)) / nz
    ok = ev < 1e-12 and orth < 1e-12 and rec < 1e-12
    print(f"  {tag:28s} n={n:5d} eig {ev:.1e} orth {orth:.1e} rec {rec:.1e} {'ok' if ok else 'FAIL'}", flush=True)
    return ok


def cases(n):
    a = rng.standard_normal((n, n))
    yield "gauss", (a + a.T) / 2
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    vals = np.concatenate([np.linspace(1, 100, n // 2), -np.linspace(1e-4, 1, n - n // 2)])
    z = (q * vals) @ q.T
    yield "split-spectrum", (z + z.T) / 2


sizes = [int(x) for x in sys.argv[1:]] or [3, 4, 33, 100, 257, 640, 641, 700, 999, 1000, 1500, 1776, 1777, 2000]
ok = True
for n in sizes:
    for mode, tail in ((2, 0), (2, 200), (2, 640)):
        L.kot_debug_trd_mid(mode, tail)
        for name, z in cases(n):
            ok &= check(z, f"mid tail={tail} {name}")
        if n > 1000:
            break
# H = I columns: diagonal and block matrices
L.kot_debug_trd_mid(2, 0)
ok &= check(np.diag(rng.standard_normal(700)), "diag700")
b = np.zeros((800, 800))
x = rng.standard_normal((400, 400))
b[:400, :400] = (x + x.T) / 2
b[600:, 600:] = np.eye(200) * 3.0
ok &= check(b, "block800")
print("ALL OK" if ok else "FAILURES", flush=True)

# timing
for n in (2000, 1000):
    z = next(iter(cases(n)))[1]
    for mode, tail in ((0, 0), (1, 0), (1, 320), (1, 640)):
        L.kot_debug_trd_mid(mode, tail)
        linalg.sym_eig(z)
        _lib.profile_enable(True)
        reps = 3
        for _ in range(reps):
            linalg.sym_eig(z)
        prof = _lib.profile_read()
        _lib.profile_enable(False)
        keys = ["eigh", "eig.sytrd", "sytrd_panel", "sytrd_mid", "sytrd_tail", "eig.stedc", "eig.ormtr"]
        print(f"n={n} mode={mode} tail={tail}: " + "  ".join(
            f"{k} {prof[k]['ms'] / reps:.2f}" for k in keys if k in prof), flush=True)
    L.kot_debug_trd_mid(1, 0)
    buf = (C.c_ulonglong * 8)()
    L.kot_debug_mid_timing(1, buf)
    linalg.sym_eig(z)
    L.kot_debug_mid_timing(0, buf)
    names = ["symv pass", "publish + update", "gather + finish"]
    for nm, v in zip(names, buf):
        print(f"  mid {nm:26s} {v / 1e6:8.3f} ms")
