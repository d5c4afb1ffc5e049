"""Regularized semismooth Newton direction (mirror of reference ``kot.newton``).

Reference: ``pkg/src/kot/newton.py``.  The Newton step (eliminator, reduced
ℓ×ℓ SPD system, CG with restarts, Eq.(9) criterion) runs on the device; this
module carries the configuration and host entry points.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from paper_2310_14087_b200 import _lib
from paper_2310_14087_b200.linalg import SpectralDecomp
from paper_2310_14087_b200.problem import IteratePair, ProblemData, residual_parts
from paper_2310_14087_b200.psdcone import NewtonEliminator, ProjJacobianCoeffs, make_eliminator, proj_jacobian_coeffs


@dataclass(frozen=True)
class NewtonConfig:
    """Constants of the Newton step (newton.py:36-71; same defaults and validation)."""

    tau: float = 0.5
    kappa: float = 0.1
    alpha1: float = 1e-6
    alpha2: float = 1.0
    beta0: float = 0.5
    beta1: float = 1.2
    beta2: float = 5.0
    theta_min: float = 1e-4
    theta_max: float = 1e4
    theta0: float = 1.0
    cg_max: int = 20
    cg_restarts: int = 2
    cg_tol: float | None = None

    def __post_init__(self) -> None:
        if not (0.0 < self.tau < 1.0 and 0.0 < self.kappa < 1.0):
            raise ValueError("tau and kappa must lie in (0, 1)")
        if not (0.0 < self.alpha1 <= self.alpha2):
            raise ValueError("need 0 < alpha1 <= alpha2")
        if not (self.beta0 < 1.0 < self.beta2):
            raise ValueError("need beta0 < 1 < beta2")
        if not (0.0 < self.theta_min <= self.theta_max):
            raise ValueError("need 0 < theta_min <= theta_max")
        if self.cg_max < 1 or self.cg_restarts < 0:
            raise ValueError("invalid CG budget")


@dataclass(frozen=True)
class NewtonContext:
    """Per-iteration spectral objects at the current iterate (newton.py:74-82)."""

    decomp: SpectralDecomp
    coeffs: ProjJacobianCoeffs
    eliminator: NewtonEliminator
    mu: float
    theta: float


@dataclass(frozen=True)
class NewtonStep:
    """newton.py:85-92."""

    dw: IteratePair
    cg_iters: int
    criterion_met: bool
    crit_lhs: float
    crit_rhs: float
    cg_ms: float = 0.0


def cfg_struct(newton: NewtonConfig, eg_stepsize: float = 0.01, residual_tol: float = 0.005, max_iter: int = 500,
               safeguard_every: int = 1) -> _lib.SolverCfgC:
    c = _lib.SolverCfgC()
    for f in ("tau", "kappa", "alpha1", "alpha2", "beta0", "beta1", "beta2", "theta_min", "theta_max", "theta0"):
        setattr(c, f, float(getattr(newton, f)))
    c.cg_max, c.cg_restarts = int(newton.cg_max), int(newton.cg_restarts)
    c.cg_tol = 0.0 if newton.cg_tol is None else float(newton.cg_tol)
    c.has_cg_tol = 0 if newton.cg_tol is None else 1
    c.eg_stepsize, c.residual_tol = float(eg_stepsize), float(residual_tol)
    c.max_iter, c.safeguard_every = int(max_iter), int(safeguard_every)
    return c


def newton_context(decomp: SpectralDecomp, res_norm: float, theta: float) -> NewtonContext:
    """μ = θ‖r‖ and the spectral operators at the decomposition (newton.py:95-107)."""
    if res_norm <= 0.0:
        raise ValueError("context requires a nonzero residual")
    mu = theta * res_norm
    coeffs = proj_jacobian_coeffs(decomp)
    return NewtonContext(decomp=decomp, coeffs=coeffs, eliminator=make_eliminator(coeffs, mu), mu=mu, theta=theta)


def newton_context_at(pd: ProblemData, w: IteratePair, theta: float) -> NewtonContext:
    """Evaluate the residual at ``w`` (on the GPU) and build its context (newton.py:110-113)."""
    r, decomp = residual_parts(pd, w)
    return newton_context(decomp, r.norm(), theta)


def middle_operator(pd: ProblemData, elim: NewtonEliminator, mu: float):
    """SPD operator of the reduced system v ↦ Qv/(2λ₂) + μv + Φ(𝒯[Φ*(v)]) (newton.py:116-128).

    The returned callable evaluates on the GPU (the solver's structure-reduced form); passed to
    :func:`paper_2310_14087_b200.linalg.cg_solve` it runs the whole CG in HBM."""
    dc = elim.coeffs.decomp
    vecs, vals = _lib.f64(dc.eigvecs), _lib.f64(dc.eigvals)

    def apply(v):
        vv = _lib.f64(v, (pd.n,))
        out = np.empty(pd.n)
        _lib.check(_lib.lib().kot_middle_operator_decomp(pd.device_problem().handle, _lib.ptr(vecs), _lib.ptr(vals),
                                                         dc.n_pos, float(mu), _lib.ptr(vv), _lib.ptr(out)))
        return out

    apply._kot_middle = (pd, dc, float(mu))
    return apply


def newton_direction(pd: ProblemData, r: IteratePair, ctx: NewtonContext, cfg: NewtonConfig) -> NewtonStep:
    """Algorithm 1 (newton.py:144-195) at ``ctx`` for the residual ``r``, on the GPU."""
    r1, r2 = _lib.f64(r.gamma, (pd.n,)), _lib.f64(r.x_mat, (pd.n, pd.n))
    dc = ctx.decomp
    dg, dx = np.empty(pd.n), np.empty((pd.n, pd.n))
    it, met, lhs, rhs = C.c_int(), C.c_int(), C.c_double(), C.c_double()
    c = cfg_struct(cfg)
    _lib.check(_lib.lib().kot_newton_direction_decomp(
        pd.device_problem().handle, C.byref(c), _lib.ptr(r1), _lib.ptr(r2), _lib.ptr(_lib.f64(dc.eigvecs)),
        _lib.ptr(_lib.f64(dc.eigvals)), dc.n_pos, float(ctx.mu), _lib.ptr(dg), _lib.ptr(dx), C.byref(it),
        C.byref(met), C.byref(lhs), C.byref(rhs)))
    return NewtonStep(IteratePair(dg, dx), int(it.value), bool(met.value), float(lhs.value), float(rhs.value))


def middle_operator_at(pd: ProblemData, w: IteratePair, theta: float, v, form: str = "reduced"
                       ) -> tuple[np.ndarray, float]:
    """Q v/(2λ₂) + μv + Φ(𝒯[Φ*(v)]) at the context of w (μ = θ‖R(w)‖) (newton.py:95-128).

    ``form="reduced"``: the solver's structure-reduced B = R·P evaluation (same-sign block as
    the GEMV (G_α∘G_α)v/μ, mixed-sign block as two GEMMs);
    ``form="blocked"``: the structure-reduced form with the whole smaller sign block in the GEMMs
    (the row-sharded layout, rowshard.py);
    ``form="direct"``: the reference's Φ* → 𝒯 → Φ chain."""
    code = {"reduced": 0, "direct": 1, "blocked": 2}[form]
    g, x = _lib.f64(w.gamma, (pd.n,)), _lib.f64(w.x_mat, (pd.n, pd.n))
    vv = _lib.f64(v, (pd.n,))
    out, mu = np.empty(pd.n), C.c_double()
    _lib.check(_lib.lib().kot_middle_operator(pd.device_problem().handle, _lib.ptr(g), _lib.ptr(x), float(theta),
                                              _lib.ptr(vv), code, _lib.ptr(out),
                                              C.byref(mu)))
    return out, float(mu.value)


def newton_direction_at(pd: ProblemData, w: IteratePair, theta: float, cfg: NewtonConfig) -> NewtonStep:
    """Algorithm 1 at w with damping θ (newton.py:144-195), on device."""
    g, x = _lib.f64(w.gamma, (pd.n,)), _lib.f64(w.x_mat, (pd.n, pd.n))
    dg, dx = np.empty(pd.n), np.empty((pd.n, pd.n))
    it, met, lhs, rhs = C.c_int(), C.c_int(), C.c_double(), C.c_double()
    c = cfg_struct(cfg)
    _lib.check(_lib.lib().kot_newton_direction(pd.device_problem().handle, C.byref(c), _lib.ptr(g), _lib.ptr(x),
                                               float(theta), _lib.ptr(dg), _lib.ptr(dx), C.byref(it),
                                               C.byref(met), C.byref(lhs), C.byref(rhs)))
    return NewtonStep(IteratePair(dg, dx), int(it.value), bool(met.value), float(lhs.value), float(rhs.value))


def theta_update(theta: float, rho: float, dw_norm_sq: float, cfg: NewtonConfig) -> float:
    """Three-branch damping update (newton.py:198-211); host scalar logic."""
    if rho >= cfg.alpha2 * dw_norm_sq:
        new = max(cfg.theta_min, cfg.beta0 * theta)
    elif rho >= cfg.alpha1 * dw_norm_sq:
        new = cfg.beta1 * theta
    else:
        new = min(cfg.theta_max, cfg.beta2 * theta)
    return float(min(max(new, cfg.theta_min), cfg.theta_max))
