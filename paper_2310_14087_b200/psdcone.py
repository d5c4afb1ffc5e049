"""PSD-cone spectral operators on the B200 (mirror of reference ``kot.psdcone``).

Reference: ``pkg/src/kot/psdcone.py``.  The operators are applied at the
eigendecomposition of a given symmetric matrix ``z`` (computed on device):
``proj_psd`` (:62-64), the projection Jacobian M(z)[S] (:94-100) and the
Newton eliminator 𝒯[S] (:103-151) with both low-rank paths.
"""

from __future__ import annotations

import numpy as np

from paper_2310_14087_b200 import _lib

POS_BLOCK = "pos_block"
NONPOS_COMPLEMENT = "nonpos_complement"
_PATH = {None: -1, POS_BLOCK: 0, NONPOS_COMPLEMENT: 1}


def proj_psd(z, device: int | None = None) -> np.ndarray:
    """Frobenius-nearest PSD matrix to sym(z)."""
    zs = _lib.f64(z)
    n = zs.shape[0]
    out = np.empty((n, n))
    _lib.check(_lib.lib().kot_proj_psd(_lib.ptr(zs), n, _lib.default_device() if device is None else device,
                                       _lib.ptr(out)))
    return out


def _spectral(z, s, mode: int, mu: float, path, device) -> np.ndarray:
    zs = _lib.f64(z)
    n = zs.shape[0]
    ss = _lib.f64(s)
    if ss.shape != (n, n):
        raise ValueError(f"expected matrix of order {n}, got shape {ss.shape}")
    out = np.empty((n, n))
    _lib.check(_lib.lib().kot_spectral_apply(_lib.ptr(zs), n, _lib.default_device() if device is None else device,
                                             mode, float(mu), _PATH[path], _lib.ptr(ss), _lib.ptr(out)))
    return out


def apply_proj_jacobian_at(z, s, path=None, device: int | None = None) -> np.ndarray:
    """M(z)[S] = P(Ω∘PᵀSP)Pᵀ evaluated by the low-rank route (psdcone.py:94-100)."""
    return _spectral(z, s, 1, 1.0, path, device)


def apply_eliminator_at(z, s, mu: float, path=None, device: int | None = None) -> np.ndarray:
    """𝒯[S] = M((μ+1)I − M)⁻¹[S] at the decomposition of z (psdcone.py:103-151)."""
    if mu <= 0.0:
        raise ValueError("regularization mu must be positive")
    return _spectral(z, s, 0, mu, path, device)
