"""Bit-identity check of two libkotgpu builds on kot_sym_eig (argv: old.so new.so)."""
import ctypes as C
import sys

import numpy as np


def run(path, z):
    L = C.CDLL(path)
    n = z.shape[0]
    vecs = np.zeros((n, n))
    vals = np.zeros(n)
    k = C.c_int(0)
    P = C.POINTER(C.c_double)
    st = L.kot_sym_eig(np.ascontiguousarray(z).ctypes.data_as(P), n, 0, vecs.ctypes.data_as(P),
                       vals.ctypes.data_as(P), C.byref(k))
    assert st == 0, st
    return vecs, vals


rng = np.random.default_rng(1)
cases = []
for n in (2, 3, 33, 100, 501, 640, 641, 1000, 2000):
    a = rng.standard_normal((n, n))
    cases.append((f"gauss{n}", (a + a.T) / 2))
cases.append(("diag700", np.diag(rng.standard_normal(700))))  # every reflector H = I
b = np.zeros((800, 800))
b[:400, :400] = cases[5][1][:400, :400] if False else (lambda x: (x + x.T) / 2)(rng.standard_normal((400, 400)))
b[600:, 600:] = np.eye(200) * 3.0
cases.append(("block800", b))  # mixes H = I columns into the tail
ok = True
for name, z in cases:
    v0, e0 = run(sys.argv[1], z)
    v1, e1 = run(sys.argv[2], z)
    same = np.array_equal(v0, v1) and np.array_equal(e0, e1)
    err = np.max(np.abs(np.sort(e1) - np.linalg.eigvalsh(z)))
    print(f"{name:10s} bit-identical={same}  max|eig - eigvalsh|={err:.2e}")
    ok &= same
print("ALL BIT-IDENTICAL" if ok else "DIFFERENCES")
