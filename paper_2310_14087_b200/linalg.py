"""Dense symmetric linear algebra on the B200 (mirror of reference ``kot.linalg``).

Reference: ``pkg/src/kot/linalg.py``.  ``sym_eig`` is the hand-written
sytrd + divide-and-conquer + back-transform eigensolver (csrc/eig.cu);
``cholesky_psd`` the blocked DMMA Cholesky with the same jitter ladder
(csrc/chol.cu).  The reference's Python-callable ``cg_solve`` has no device
equivalent: CG runs fused inside the device Newton step (csrc/solver.cu).
"""

from __future__ import annotations

from dataclasses import dataclass

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


def cholesky_psd(k, device: int | None = None) -> CholeskyFactor:
    """Upper Cholesky factor with the 0, 1e-10·s … 1e-6·s jitter ladder (linalg.py:91-114)."""
    ks = _lib.f64(k)
    n = ks.shape[0]
    up = np.empty((n, n))
    jit = _lib.C.c_double(0.0)
    _lib.check(_lib.lib().kot_cholesky_psd(_lib.ptr(ks), n, _lib.default_device() if device is None else device,
                                           _lib.ptr(up), _lib.C.byref(jit)))
    return CholeskyFactor(upper=up, jitter_applied=float(jit.value))
