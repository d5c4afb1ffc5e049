"""PSD-cone spectral operators on the B200 (mirror of reference ``kot.psdcone``).

Reference: ``pkg/src/kot/psdcone.py``.  Same names, dataclasses and call
signatures: ``proj_from_decomp`` (:52-59), ``proj_psd`` (:62-64),
``proj_jacobian_coeffs`` (:67-80), ``apply_proj_jacobian`` (:94-100),
``make_eliminator`` (:103-110) and ``apply_eliminator`` (:124-151) with both
low-rank paths.  The operators run on the GPU from the decomposition
(``kot_spectral_apply_decomp``); their coefficients η = σ_α/(σ_α − σ_ᾱ) and
ξ = η/(μ + 1 − η) are formed inside the DMMA GEMM epilogues from σ, so the
k×(ℓ−k) ``cross`` / ``cross_scaled`` arrays of the reference dataclasses are
host views built only when a caller reads them.  ``*_at`` variants take the
matrix z and decompose it on the device first.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from paper_2310_14087_b200 import _lib
from paper_2310_14087_b200.linalg import SpectralDecomp

POS_BLOCK = "pos_block"
NONPOS_COMPLEMENT = "nonpos_complement"
_PATH = {None: -1, POS_BLOCK: 0, NONPOS_COMPLEMENT: 1}


def _dev(device):
    return _lib.default_device() if device is None else device


@dataclass(frozen=True)
class ProjJacobianCoeffs:
    """Spectral coefficients of the projection's generalized Jacobian (psdcone.py:22-32)."""

    decomp: SpectralDecomp
    _cross: np.ndarray | None = field(default=None, repr=False, compare=False)

    @property
    def cross(self) -> np.ndarray:
        """cross[i, j] = σ_i/(σ_i − σ_j), i positive, j nonpositive (host view; lies in (0, 1])."""
        if self._cross is None:
            k = self.decomp.n_pos
            pos, non = self.decomp.eigvals[:k], self.decomp.eigvals[k:]
            object.__setattr__(self, "_cross", pos[:, None] / (pos[:, None] - non[None, :]))
        return self._cross


@dataclass(frozen=True)
class NewtonEliminator:
    """M((μ+1)I − M)⁻¹ at the decomposition; ``path`` picks the cheap route (psdcone.py:35-49)."""

    coeffs: ProjJacobianCoeffs
    mu: float
    path: str

    @property
    def cross_scaled(self) -> np.ndarray:
        """ξ = η/(μ + 1 − η) ∈ (0, 1/μ] (host view)."""
        c = self.coeffs.cross
        return c / (self.mu + 1.0 - c)


def _decomp_call(decomp: SpectralDecomp, mode: int, mu: float, path, s, device) -> np.ndarray:
    n = decomp.order
    vecs, vals = _lib.f64(decomp.eigvecs), _lib.f64(decomp.eigvals)
    ss = None
    if mode != 2:
        ss = _lib.f64(s)
        if ss.shape != (n, n):
            raise ValueError(f"expected matrix of order {n}, got shape {ss.shape}")
    out = np.empty((n, n))
    _lib.check(_lib.lib().kot_spectral_apply_decomp(_lib.ptr(vecs), _lib.ptr(vals), n, decomp.n_pos, _dev(device),
                                                    mode, float(mu), _PATH[path], _lib.ptr(ss), _lib.ptr(out)))
    return out


def proj_from_decomp(decomp: SpectralDecomp, device: int | None = None) -> np.ndarray:
    """sym(P_α diag(σ_α) P_αᵀ) from a precomputed decomposition; zeros if k = 0 (psdcone.py:52-59)."""
    return _decomp_call(decomp, 2, 0.0, None, None, device)


def proj_psd(z, device: int | None = None) -> np.ndarray:
    """Frobenius-nearest PSD matrix to sym(z) (psdcone.py:62-64)."""
    zs = _lib.f64(z)
    n = zs.shape[0]
    out = np.empty((n, n))
    _lib.check(_lib.lib().kot_proj_psd(_lib.ptr(zs), n, _dev(device), _lib.ptr(out)))
    return out


def proj_jacobian_coeffs(decomp: SpectralDecomp) -> ProjJacobianCoeffs:
    """Coefficients of the projection's directional derivative (psdcone.py:67-80).

    The sign-group gap σ_α − σ_ᾱ is structurally positive; like the reference, a non-positive
    (NaN) gap raises AssertionError."""
    k = decomp.n_pos
    if 0 < k < decomp.order and not decomp.eigvals[k - 1] - decomp.eigvals[k] > 0.0:
        raise AssertionError("eigenvalue gap between sign groups must be positive")
    return ProjJacobianCoeffs(decomp=decomp)


def jacobian_coeff_matrix(coeffs: ProjJacobianCoeffs) -> np.ndarray:
    """Dense n×n Hadamard coefficient matrix of M (psdcone.py:83-91; host helper for the dense formula)."""
    n, k = coeffs.decomp.order, coeffs.decomp.n_pos
    w = np.zeros((n, n))
    w[:k, :k] = 1.0
    w[:k, k:] = coeffs.cross
    w[k:, :k] = coeffs.cross.T
    return w


def apply_proj_jacobian(coeffs: ProjJacobianCoeffs, s, device: int | None = None) -> np.ndarray:
    """M(Z)[S] = P(Ω∘PᵀSP)Pᵀ (psdcone.py:94-100), by the low-rank G + Gᵀ route on the GPU."""
    return _decomp_call(coeffs.decomp, 1, 1.0, None, s, device)


def make_eliminator(coeffs: ProjJacobianCoeffs, mu: float) -> NewtonEliminator:
    """ξ = η/(μ+1−η); POS_BLOCK iff k ≤ ℓ − k (psdcone.py:103-110)."""
    if mu <= 0.0:
        raise ValueError("regularization mu must be positive")
    k, n = coeffs.decomp.n_pos, coeffs.decomp.order
    return NewtonEliminator(coeffs=coeffs, mu=float(mu), path=POS_BLOCK if k <= n - k else NONPOS_COMPLEMENT)


def eliminator_coeff_matrix(op: NewtonEliminator) -> np.ndarray:
    """Dense Hadamard coefficient matrix of 𝒯 (psdcone.py:113-121; host helper for the dense formula)."""
    n, k = op.coeffs.decomp.order, op.coeffs.decomp.n_pos
    w = np.zeros((n, n))
    w[:k, :k] = 1.0 / op.mu
    w[:k, k:] = op.cross_scaled
    w[k:, :k] = op.cross_scaled.T
    return w


def apply_eliminator(op: NewtonEliminator, s, device: int | None = None) -> np.ndarray:
    """𝒯[S] along ``op.path`` (psdcone.py:124-151), on the GPU."""
    return _decomp_call(op.coeffs.decomp, 0, op.mu, op.path, s, device)


def _spectral(z, s, mode: int, mu: float, path, device) -> np.ndarray:
    zs = _lib.f64(z)
    n = zs.shape[0]
    ss = _lib.f64(s)
    if ss.shape != (n, n):
        raise ValueError(f"expected matrix of order {n}, got shape {ss.shape}")
    out = np.empty((n, n))
    _lib.check(_lib.lib().kot_spectral_apply(_lib.ptr(zs), n, _dev(device), mode, float(mu), _PATH[path],
                                             _lib.ptr(ss), _lib.ptr(out)))
    return out


def apply_proj_jacobian_at(z, s, path=None, device: int | None = None) -> np.ndarray:
    """M(z)[S] at the device decomposition of z (no host eigenvectors)."""
    return _spectral(z, s, 1, 1.0, path, device)


def apply_eliminator_at(z, s, mu: float, path=None, device: int | None = None) -> np.ndarray:
    """𝒯[S] = M((μ+1)I − M)⁻¹[S] at the device decomposition of z."""
    if mu <= 0.0:
        raise ValueError("regularization mu must be positive")
    return _spectral(z, s, 0, mu, path, device)
