"""Dense symmetric linear algebra on the B200 (mirror of reference ``kot.linalg``).

Reference: ``pkg/src/kot/linalg.py``.  ``sym_eig`` is the hand-written
sytrd + divide-and-conquer + back-transform eigensolver (csrc/eig.cu);
``cholesky_psd`` the blocked DMMA Cholesky with the same jitter ladder
(csrc/chol.cu); ``cg_solve`` runs the CG recurrence on the device — entirely so
for the solver's own middle operator (``newton.middle_operator``), with one
host round trip per matvec for an arbitrary Python callable.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np

from paper_2310_14087_b200 import _lib
from paper_2310_14087_b200._lib import EigenSolveError, IndefiniteKernelError  # noqa: F401


def symmetrize(a: np.ndarray) -> np.ndarray:
    """Return the symmetric part (a + a.T) / 2 (linalg.py:25-27; host helper)."""
    return 0.5 * (a + a.T)


@dataclass(frozen=True)
class SpectralDecomp:
    """Eigendecomposition, eigenvalues descending; pos_idx = strictly positive prefix (linalg.py:30-49)."""

    eigvecs: np.ndarray
    eigvals: np.ndarray
    pos_idx: np.ndarray
    nonpos_idx: np.ndarray

    @property
    def order(self) -> int:
        return self.eigvals.shape[0]

    @property
    def n_pos(self) -> int:
        return self.pos_idx.shape[0]


@dataclass(frozen=True)
class CholeskyFactor:
    """Upper-triangular R with R.T @ R = input + jitter_applied * I (linalg.py:52-57)."""

    upper: np.ndarray
    jitter_applied: float


def sym_eig(z, device: int | None = None) -> SpectralDecomp:
    """Eigendecompose sym(z) on the GPU; descending order, strict σ>0 split (linalg.py:60-83)."""
    zs = _lib.f64(z)
    if zs.ndim != 2 or zs.shape[0] != zs.shape[1]:
        raise ValueError("expected a square matrix")
    n = zs.shape[0]
    vecs = np.empty((n, n))
    vals = np.empty(n)
    k = _lib.C.c_int(0)
    _lib.check(_lib.lib().kot_sym_eig(_lib.ptr(zs), n, _lib.default_device() if device is None else device,
                                      _lib.ptr(vecs), _lib.ptr(vals), _lib.C.byref(k)))
    kk = int(k.value)
    return SpectralDecomp(eigvecs=vecs, eigvals=vals, pos_idx=np.arange(kk), nonpos_idx=np.arange(kk, n))


def cg_solve(apply: Callable[[np.ndarray], np.ndarray], rhs, tol: float, max_iter: int,
             device: int | None = None) -> tuple[np.ndarray, int, float]:
    """Conjugate gradient for an SPD operator (linalg.py:117-162): stops once the recursive residual
    ‖r‖ ≤ tol·‖rhs‖ or after ``max_iter`` matvecs; pᵀAp ≤ 0 ends it one step early; NaN/Inf raise
    FloatingPointError.

    ``apply`` built by :func:`paper_2310_14087_b200.newton.middle_operator` runs wholly on the GPU
    (the solver's fused CG); any other callable is evaluated on host copies of p, with the CG vector
    algebra on the device."""
    if max_iter < 1:
        raise ValueError("max_iter must be >= 1")
    b = _lib.f64(rhs)
    n = b.shape[0]
    x = np.empty(n)
    iters, res = _lib.C.c_int(0), _lib.C.c_double(0.0)
    dev = getattr(apply, "_kot_middle", None)
    if dev is not None:  # (ProblemData, SpectralDecomp, mu): everything stays in HBM
        pd, dc, mu = dev
        _lib.check(_lib.lib().kot_cg_solve_middle(pd.device_problem().handle, _lib.ptr(_lib.f64(dc.eigvecs)),
                                                  _lib.ptr(_lib.f64(dc.eigvals)), dc.n_pos, float(mu), _lib.ptr(b),
                                                  float(tol), int(max_iter), _lib.ptr(x), _lib.C.byref(iters),
                                                  _lib.C.byref(res)))
        return x, int(iters.value), float(res.value)
    raised: list[BaseException] = []

    def _mv(_user, p, ap):
        try:
            out = np.asarray(apply(np.ctypeslib.as_array(p, shape=(n,)).copy()), dtype=float)
            if out.shape != (n,):
                raise ValueError(f"operator returned shape {out.shape}, expected ({n},)")
            np.ctypeslib.as_array(ap, shape=(n,))[:] = out
            return 0
        except BaseException as e:  # noqa: BLE001 — re-raised below
            raised.append(e)
            return 1

    cb = _lib.MatvecFn(_mv)
    st = _lib.lib().kot_cg_solve(cb, None, _lib.ptr(b), n, float(tol), int(max_iter),
                                 _lib.default_device() if device is None else device, _lib.ptr(x),
                                 _lib.C.byref(iters), _lib.C.byref(res))
    if raised:
        raise raised[0]
    _lib.check(st)
    return x, int(iters.value), float(res.value)


def cholesky_psd(k, device: int | None = None) -> CholeskyFactor:
    """Upper Cholesky factor with the 0, 1e-10·s … 1e-6·s jitter ladder (linalg.py:91-114)."""
    ks = _lib.f64(k)
    n = ks.shape[0]
    up = np.empty((n, n))
    jit = _lib.C.c_double(0.0)
    _lib.check(_lib.lib().kot_cholesky_psd(_lib.ptr(ks), n, _lib.default_device() if device is None else device,
                                           _lib.ptr(up), _lib.C.byref(jit)))
    return CholeskyFactor(upper=up, jitter_applied=float(jit.value))
