"""NumPy restatement of the reference SSN kernel-OT solver (oracle; test-only).

Every function cites the reference ``file:line`` it restates (paths relative
to ``/root/reference/pkg/src/kot``).  The arithmetic is performed with the
same NumPy/LAPACK primitives in the same order, so that on identical inputs
this port reproduces the reference bit-for-bit on the machine that generated
``tests/golden`` (checked by ``tests/test_oracle_golden.py``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field, replace
from typing import Callable

import numpy as np
import scipy.linalg
from scipy.spatial.distance import cdist

__all__ = [
    "OracleEigenError", "OracleIndefiniteKernel", "OracleNumericsError",
    "Decomp", "Problem", "Pair", "NewtonCfg", "SolverCfg", "Record", "Report",
    "sym", "gaussian_gram", "mean_embedding", "embedding_norm_sq", "assemble",
    "cholesky_psd", "sym_eig", "cg", "proj", "proj_psd", "cross_coeffs",
    "apply_proj_jacobian", "eliminator", "apply_eliminator", "phi", "phi_adj",
    "objective_grad", "objective", "residual_parts", "apply_jacobian",
    "middle_operator", "newton_direction", "theta_update", "eg_step", "solve",
    "solve_pure_eg", "ot_estimate", "evaluate_map", "iterate_once",
]


class OracleEigenError(RuntimeError):
    """linalg.py:17-18 EigenSolveError."""


class OracleIndefiniteKernel(RuntimeError):
    """linalg.py:21-22 IndefiniteKernelError."""


class OracleNumericsError(RuntimeError):
    """solver.py:28-33 SolverNumericsError (carries the partial trace)."""

    def __init__(self, msg, trace):
        super().__init__(msg)
        self.trace = trace


# --------------------------------------------------------------------- linalg

def sym(a: np.ndarray) -> np.ndarray:
    """linalg.py:25-27: (a + a.T)/2."""
    return 0.5 * (a + a.T)


@dataclass(frozen=True)
class Decomp:
    """linalg.py:30-49 SpectralDecomp: descending eigenvalues, k = #(σ > 0)."""

    vecs: np.ndarray
    vals: np.ndarray
    k: int

    @property
    def n(self) -> int:
        return self.vals.shape[0]


def sym_eig(z: np.ndarray) -> Decomp:
    """linalg.py:60-83: eigh of sym(z), stable descending order, strict σ>0 split."""
    zs = sym(np.asarray(z, dtype=float))
    try:
        w, v = np.linalg.eigh(zs)
    except np.linalg.LinAlgError as exc:  # pragma: no cover - LAPACK failure
        raise OracleEigenError(str(exc)) from exc
    order = np.argsort(-w, kind="stable")
    w = w[order]
    return Decomp(vecs=v[:, order], vals=w, k=int(np.count_nonzero(w > 0.0)))


def jitter_ladder(scale: float) -> list[float]:
    """linalg.py:86-105: 0, then 1e-10·s ... 1e-6·s by decades."""
    out = [0.0]
    lev = 1e-10
    while lev <= 1e-6 * (1 + 1e-12):
        out.append(lev * scale)
        lev *= 10.0
    return out


def cholesky_psd(k: np.ndarray) -> tuple[np.ndarray, float]:
    """linalg.py:91-114: upper Cholesky of sym(k) + jitter·I over the ladder."""
    ks = sym(np.asarray(k, dtype=float))
    n = ks.shape[0]
    for jit in jitter_ladder(np.trace(ks) / n):
        try:
            up = scipy.linalg.cholesky(ks + jit * np.eye(n), lower=False, check_finite=False)
        except scipy.linalg.LinAlgError:
            continue
        return up, jit
    raise OracleIndefiniteKernel("kernel matrix numerically indefinite")


def cg(apply: Callable[[np.ndarray], np.ndarray], b: np.ndarray, tol: float, max_iter: int):
    """linalg.py:117-162: plain CG from 0; recursive-residual stop; pAp<=0 break."""
    if max_iter < 1:
        raise ValueError("max_iter must be >= 1")
    b = np.asarray(b, dtype=float)
    x = np.zeros_like(b)
    r = b.copy()
    bn = float(np.linalg.norm(b))
    goal = tol * bn
    res = bn
    if res <= goal:
        return x, 0, res
    p = r.copy()
    rr = float(r @ r)
    it = 0
    for it in range(1, max_iter + 1):
        q = apply(p)
        pq = float(p @ q)
        if not np.isfinite(pq):
            raise FloatingPointError("non-finite curvature in conjugate gradient")
        if pq <= 0.0:
            it -= 1
            break
        a = rr / pq
        x += a * p
        r -= a * q
        res = float(np.linalg.norm(r))
        if not np.isfinite(res):
            raise FloatingPointError("non-finite residual in conjugate gradient")
        if res <= goal:
            return x, it, res
        rr2 = float(r @ r)
        p = r + (rr2 / rr) * p
        rr = rr2
    return x, it, res


# -------------------------------------------------------------------- kernels

def gaussian_gram(bw_sq: float, a: np.ndarray, b: np.ndarray | None = None) -> np.ndarray:
    """kernels.py:61-73: exp(-||a_i-b_j||^2/(2σ²)); square ⇒ sym, unit diagonal."""
    a = np.atleast_2d(np.asarray(a, dtype=float))
    square = b is None
    bb = a if square else np.atleast_2d(np.asarray(b, dtype=float))
    g = np.exp(-cdist(a, bb, metric="sqeuclidean") / (2.0 * bw_sq))
    if square:
        g = 0.5 * (g + g.T)
        np.fill_diagonal(g, 1.0)
    return g


def mean_embedding(bw_sq: float, samples: np.ndarray, queries: np.ndarray) -> np.ndarray:
    """kernels.py:83-87: column means of the (n × m) sample/query Gram."""
    return gaussian_gram(bw_sq, samples, queries).mean(axis=0)


def embedding_norm_sq(bw_sq: float, samples: np.ndarray) -> float:
    """kernels.py:90-94: mean of the square sample Gram."""
    return float(np.mean(gaussian_gram(bw_sq, samples)))


# -------------------------------------------------------------------- problem

@dataclass
class Problem:
    """problem.py:86-123 ProblemData (fields renamed: q, z, q_sq, r, l1, l2, embed)."""

    q: np.ndarray
    z: np.ndarray
    q_sq: float
    r: np.ndarray
    l1: float
    l2: float
    embed: np.ndarray | None = None
    xt: np.ndarray | None = None
    yt: np.ndarray | None = None
    bw_sq: float | None = None
    jitter: float = 0.0

    def __post_init__(self):
        self.q = sym(np.asarray(self.q, dtype=float))  # problem.py:112
        self.z = np.asarray(self.z, dtype=float)
        self.r = np.asarray(self.r, dtype=float)

    @property
    def n(self) -> int:
        return self.z.shape[0]


def assemble(xs, ys, xt, yt, l1, l2, bw_sq, bw_y=None, bw_xy=None) -> tuple[Problem, np.ndarray]:
    """problem.py:135-169 (+ build_kernel_specs :126-132: one bandwidth unless bw_y / bw_xy are given,
    i.e. spec_x, spec_y, spec_xy with their own bandwidth_sq).

    Returns the problem and the pair-kernel Gram K (for the EG stepsize rule).
    """
    if l1 <= 0.0 or l2 <= 0.0:
        raise ValueError("lambda1 and lambda2 must be positive")
    bw_x = bw_sq
    bw_y = bw_sq if bw_y is None else bw_y
    bw_xy = bw_sq if bw_xy is None else bw_xy
    q = gaussian_gram(bw_x, xt) + gaussian_gram(bw_y, yt)
    emb = mean_embedding(bw_x, xs, xt) + mean_embedding(bw_y, ys, yt)
    cost = np.sum((xt - yt) ** 2, axis=1)
    z = emb - l2 * cost
    q_sq = embedding_norm_sq(bw_x, xs) + embedding_norm_sq(bw_y, ys)
    kmat = gaussian_gram(bw_xy, np.hstack([xt, yt]))
    r, jit = cholesky_psd(kmat)
    return Problem(q=q, z=z, q_sq=q_sq, r=r, l1=l1, l2=l2, embed=emb, xt=xt, yt=yt,
                   bw_sq=bw_sq, jitter=jit), kmat


@dataclass
class Pair:
    """problem.py:45-83 IteratePair; norm is ||γ||₂ + ||X||_F (a sum)."""

    g: np.ndarray
    x: np.ndarray

    def norm(self) -> float:
        return float(np.linalg.norm(self.g) + np.linalg.norm(self.x))

    def dot(self, o: "Pair") -> float:
        return float(self.g @ o.g + np.sum(self.x * o.x))

    def copy(self) -> "Pair":
        return Pair(self.g.copy(), self.x.copy())

    def __add__(self, o):
        return Pair(self.g + o.g, self.x + o.x)

    def finite(self) -> bool:
        return bool(np.all(np.isfinite(self.g)) and np.all(np.isfinite(self.x)))


def phi(pd: Problem, xm: np.ndarray) -> np.ndarray:
    """problem.py:172-177: Φ(X)_i = r_i X r_iᵀ with r_i = row i of R."""
    return np.einsum("ij,ij->i", pd.r @ xm, pd.r)


def phi_adj(pd: Problem, g: np.ndarray) -> np.ndarray:
    """problem.py:180-185: Φ*(γ) = sym(Rᵀ diag(γ) R)."""
    return sym(pd.r.T @ (g[:, None] * pd.r))


def objective_grad(pd: Problem, g: np.ndarray) -> np.ndarray:
    """problem.py:188-189."""
    return (pd.q @ g - pd.z) / (2.0 * pd.l2)


def objective(pd: Problem, g: np.ndarray) -> float:
    """problem.py:192-196."""
    quad = float(g @ (pd.q @ g)) / (4.0 * pd.l2)
    lin = float(g @ pd.z) / (2.0 * pd.l2)
    return quad - lin + pd.q_sq / (4.0 * pd.l2)


def constraint_matrix(pd: Problem, g: np.ndarray) -> np.ndarray:
    """problem.py:199-201."""
    return phi_adj(pd, g) + pd.l1 * np.eye(pd.n)


# -------------------------------------------------------------------- psdcone

def proj(dc: Decomp) -> np.ndarray:
    """psdcone.py:52-59: sym(P_α diag(σ_α) P_αᵀ); zero if k = 0."""
    if dc.k == 0:
        return np.zeros((dc.n, dc.n))
    pa = dc.vecs[:, : dc.k]
    return sym((pa * dc.vals[: dc.k]) @ pa.T)


def proj_psd(z: np.ndarray) -> np.ndarray:
    """psdcone.py:62-64."""
    return proj(sym_eig(z))


def cross_coeffs(dc: Decomp) -> np.ndarray:
    """psdcone.py:67-80: η_ab = σ_a/(σ_a − σ_b), a ∈ α, b ∈ ᾱ."""
    pos = dc.vals[: dc.k]
    non = dc.vals[dc.k:]
    den = pos[:, None] - non[None, :]
    if den.size and not np.all(den > 0.0):
        raise AssertionError("eigenvalue gap between sign groups must be positive")
    return pos[:, None] / den if den.size else np.zeros((dc.k, dc.n - dc.k))


def _omega(dc: Decomp, eta: np.ndarray) -> np.ndarray:
    """psdcone.py:83-91 jacobian_coeff_matrix."""
    w = np.zeros((dc.n, dc.n))
    w[: dc.k, : dc.k] = 1.0
    w[: dc.k, dc.k:] = eta
    w[dc.k:, : dc.k] = eta.T
    return w


def apply_proj_jacobian(dc: Decomp, eta: np.ndarray, s: np.ndarray) -> np.ndarray:
    """psdcone.py:94-100: dense M(Z)[S] = P(Ω∘PᵀSP)Pᵀ (unsymmetrized)."""
    if s.shape != (dc.n, dc.n):
        raise ValueError("order mismatch")
    p = dc.vecs
    return p @ (_omega(dc, eta) * (p.T @ s @ p)) @ p.T


@dataclass(frozen=True)
class Elim:
    """psdcone.py:35-49 NewtonEliminator: ξ = η/(μ+1−η), path by k ≤ n−k."""

    dc: Decomp
    eta: np.ndarray
    mu: float
    xi: np.ndarray
    pos_path: bool


def eliminator(dc: Decomp, eta: np.ndarray, mu: float) -> Elim:
    """psdcone.py:103-110."""
    if mu <= 0.0:
        raise ValueError("regularization mu must be positive")
    xi = eta / (mu + 1.0 - eta)
    return Elim(dc, eta, mu, xi, dc.k <= dc.n - dc.k)


def apply_eliminator(op: Elim, s: np.ndarray) -> np.ndarray:
    """psdcone.py:124-151: 𝒯[S] along the cheap low-rank path."""
    dc = op.dc
    if s.shape != (dc.n, dc.n):
        raise ValueError("order mismatch")
    pa = dc.vecs[:, : dc.k]
    pn = dc.vecs[:, dc.k:]
    if op.pos_path:
        u = pa.T @ s
        g = pa @ (((u @ pa) / (2.0 * op.mu)) @ pa.T + (op.xi * (u @ pn)) @ pn.T)
        return g + g.T
    rem = 1.0 / op.mu - op.xi
    v = pn.T @ s
    h = pn @ (((v @ pn) / (2.0 * op.mu)) @ pn.T + (rem.T * (v @ pa)) @ pa.T)
    return s / op.mu - (h + h.T)


def eliminator_dense(op: Elim, s: np.ndarray) -> np.ndarray:
    """psdcone.py:113-121 (test_psdcone.py:_direct_eliminator): P(W∘PᵀSP)Pᵀ."""
    dc = op.dc
    w = np.zeros((dc.n, dc.n))
    w[: dc.k, : dc.k] = 1.0 / op.mu
    w[: dc.k, dc.k:] = op.xi
    w[dc.k:, : dc.k] = op.xi.T
    p = dc.vecs
    return p @ (w * (p.T @ s @ p)) @ p.T


# ----------------------------------------------------------- residual / Jacobian

def residual_parts(pd: Problem, w: Pair) -> tuple[Pair, Decomp]:
    """problem.py:204-214: r1 = ∇f − Φ(X); Z = sym(X) − (Φ*(γ)+λ₁I); r2 = X − Π(Z)."""
    r1 = objective_grad(pd, w.g) - phi(pd, w.x)
    zarg = sym(w.x) - constraint_matrix(pd, w.g)
    dc = sym_eig(zarg)
    return Pair(r1, w.x - proj(dc)), dc


def objective_grad_dir(pd: Problem, d: np.ndarray) -> np.ndarray:
    """problem.py:239-241."""
    return (pd.q @ d) / (2.0 * pd.l2)


def apply_jacobian(pd: Problem, dc: Decomp, eta: np.ndarray, mu: float, dw: Pair) -> Pair:
    """problem.py:222-236: regularized generalized Jacobian (J + μI) dw."""
    top = objective_grad_dir(pd, dw.g) + mu * dw.g - phi(pd, dw.x)
    bot = apply_proj_jacobian(dc, eta, phi_adj(pd, dw.g) - dw.x) + (1.0 + mu) * dw.x
    return Pair(top, bot)


# --------------------------------------------------------------------- newton

@dataclass(frozen=True)
class NewtonCfg:
    """newton.py:36-71 NewtonConfig (same defaults and validation)."""

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

    def __post_init__(self):
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
class Ctx:
    """newton.py:74-107 NewtonContext."""

    dc: Decomp
    eta: np.ndarray
    op: Elim
    mu: float
    theta: float


def newton_context(dc: Decomp, res_norm: float, theta: float) -> Ctx:
    """newton.py:95-107: μ = θ‖r‖."""
    if res_norm <= 0.0:
        raise ValueError("context requires a nonzero residual")
    mu = theta * res_norm
    eta = cross_coeffs(dc)
    return Ctx(dc, eta, eliminator(dc, eta, mu), mu, theta)


def middle_operator(pd: Problem, op: Elim, mu: float):
    """newton.py:116-128: v ↦ Qv/(2λ₂) + μv + Φ(𝒯[Φ*(v)])."""

    def apply(v):
        return objective_grad_dir(pd, v) + mu * v + phi(pd, apply_eliminator(op, phi_adj(pd, v)))

    return apply


@dataclass(frozen=True)
class Step:
    """newton.py:85-92 NewtonStep (+ attempts, not logged by the reference)."""

    dw: Pair
    cg_iters: int
    met: bool
    lhs: float
    rhs: float
    cg_ms: float
    attempts: int


def newton_direction(pd: Problem, r: Pair, ctx: Ctx, cfg: NewtonCfg) -> Step:
    """newton.py:144-195: Algorithm 1 with CG restarts and the Eq.(9) criterion."""
    op, mu = ctx.op, ctx.mu
    rn = r.norm()
    if rn <= 0.0:
        raise ValueError("direction requires a nonzero residual")
    filt = r.x + apply_eliminator(op, r.x)
    a1 = -r.g - phi(pd, filt) / (mu + 1.0)
    a2t = -filt / (mu + 1.0)
    A = middle_operator(pd, op, mu)
    rel = cfg.cg_tol if cfg.cg_tol is not None else cfg.tau * min(1.0, cfg.kappa * rn)
    a1n = float(np.linalg.norm(a1))
    sol = np.zeros_like(a1)
    total = 0
    met, lhs, rhs = False, np.inf, 0.0
    t0 = time.perf_counter()
    attempts = 0
    cg_ms = 0.0
    for att in range(cfg.cg_restarts + 1):
        attempts = att + 1
        b = a1 - A(sol) if att else a1
        bn = float(np.linalg.norm(b))
        if bn > 0.0 and a1n > 0.0:
            corr, it, _ = cg(A, b, rel * a1n / bn, cfg.cg_max)
            sol = sol + corr
            total += it
        cg_ms = (time.perf_counter() - t0) * 1e3
        dw = Pair(sol, a2t - apply_eliminator(op, phi_adj(pd, sol)))
        lhs = (apply_jacobian(pd, ctx.dc, ctx.eta, mu, dw) + r).norm()
        rhs = cfg.tau * min(1.0, cfg.kappa * rn * dw.norm())
        met = lhs <= rhs
        if met:
            break
        rel /= 10.0
    return Step(dw, total, met, lhs, rhs, cg_ms, attempts)


def theta_update(theta: float, rho: float, dw_sq: float, cfg: NewtonCfg) -> float:
    """newton.py:198-211: three-branch damping update, clipped."""
    if rho >= cfg.alpha2 * dw_sq:
        t = max(cfg.theta_min, cfg.beta0 * theta)
    elif rho >= cfg.alpha1 * dw_sq:
        t = cfg.beta1 * theta
    else:
        t = min(cfg.theta_max, cfg.beta2 * theta)
    return float(np.clip(t, cfg.theta_min, cfg.theta_max))


# ------------------------------------------------------------------------- eg

def eg_step(pd: Problem, v: Pair, s: float) -> Pair:
    """eg.py:27-41: two-stage projected extragradient; output X is PSD."""
    gv = objective_grad(pd, v.g) - phi(pd, v.x)
    gm = constraint_matrix(pd, v.g)
    gh = v.g - s * gv
    xh = proj_psd(v.x - s * gm)
    gv = objective_grad(pd, gh) - phi(pd, xh)
    gm = constraint_matrix(pd, gh)
    return Pair(v.g - s * gv, proj_psd(v.x - s * gm))


# --------------------------------------------------------------------- solver

@dataclass(frozen=True)
class SolverCfg:
    """solver.py:36-51 SolverConfig (eg → its stepsize)."""

    newton: NewtonCfg = field(default_factory=NewtonCfg)
    eg_stepsize: float = 0.01
    residual_tol: float = 0.005
    max_iter: int = 500
    safeguard_every: int = 1


@dataclass(frozen=True)
class Record:
    """solver.py:54-73 IterationRecord (+ n_pos, attempts for the GPU trace)."""

    iteration: int
    res_accepted: float
    res_ssn: float
    res_eg: float
    accepted: str
    theta: float
    mu: float
    cg_iters: int
    criterion_met: bool
    crit_lhs: float
    crit_rhs: float
    step_ms: float
    attempts: int = 0


@dataclass
class Report:
    """solver.py:89-101 SolverReport."""

    gamma: np.ndarray
    x: np.ndarray
    ot: float | None
    res: float
    termination: str
    trace: list
    total_ms: float


@dataclass
class State:
    """Loop state of solver.py:114-233 between two iterations."""

    w: Pair
    v: Pair
    r_w: Pair
    dc_w: Decomp
    res_w: float
    r_v: Pair | None
    dc_v: Decomp | None
    res_v: float
    theta: float


def _finite(res, pair, trace):
    """solver.py:109-111."""
    if not (np.isfinite(res) and pair.finite()):
        raise OracleNumericsError("non-finite residual in solver iterate", trace)


def initial_state(pd: Problem, cfg: SolverCfg) -> State:
    """solver.py:129-139."""
    w = Pair(np.zeros(pd.n), np.zeros((pd.n, pd.n)))
    r_w, dc = residual_parts(pd, w)
    res = r_w.norm()
    _finite(res, r_w, [])
    return State(w, w.copy(), r_w, dc, res, None, None, res, cfg.newton.theta0)


def iterate_once(pd: Problem, st: State, k: int, cfg: SolverCfg, trace=None,
                 on_iteration=None) -> tuple[State, Record, Step]:
    """One pass of the solver.py:142-222 loop body (also the lock-step replay unit)."""
    trace = [] if trace is None else trace
    t_it = time.perf_counter()
    v, r_v, dc_v, res_v = st.v, st.r_v, st.dc_v, st.res_v
    if k % cfg.safeguard_every == 0:
        v = eg_step(pd, v, cfg.eg_stepsize)
        r_v, dc_v = residual_parts(pd, v)
        res_v = r_v.norm()
        _finite(res_v, r_v, trace)
    ctx = newton_context(st.dc_w, st.res_w, st.theta)
    step = newton_direction(pd, st.r_w, ctx, cfg.newton)
    wt = st.w + step.dw
    r_t, dc_t = residual_parts(pd, wt)
    res_t = r_t.norm()
    _finite(res_t, r_t, trace)
    if on_iteration is not None:
        on_iteration(k, st.w, st.r_w, ctx.mu, st.theta, step.dw, step.met)
    rho = -r_t.dot(step.dw)
    th_next = theta_update(st.theta, rho, step.dw.norm() ** 2, cfg.newton)
    if res_t <= res_v:
        acc = "ssn"
        w, r_w, dc_w, res_w = wt, r_t, dc_t, res_t
    else:
        acc = "eg"
        w, r_w, dc_w, res_w = v.copy(), r_v, dc_v, res_v
    rec = Record(k, res_w, res_t, res_v, acc, st.theta, ctx.mu, step.cg_iters, step.met,
                 step.lhs, step.rhs, (time.perf_counter() - t_it) * 1e3, step.attempts)
    return State(w, v, r_w, dc_w, res_w, r_v, dc_v, res_v, th_next), rec, step


def solve(pd: Problem, cfg: SolverCfg | None = None, on_iteration=None) -> Report:
    """solver.py:114-233: Algorithm 2 from the zero pair."""
    cfg = cfg or SolverCfg()
    t0 = time.perf_counter()
    trace: list[Record] = []
    st = initial_state(pd, cfg)
    term = "converged" if st.res_w <= cfg.residual_tol else "max_iter"
    k = 0
    while term != "converged" and k < cfg.max_iter:
        st, rec, _ = iterate_once(pd, st, k, cfg, trace, on_iteration)
        trace.append(rec)
        k += 1
        if st.res_w <= cfg.residual_tol:
            term = "converged"
    ot = ot_estimate(pd, st.w.g) if pd.embed is not None else None
    return Report(st.w.g, st.w.x, ot, st.res_w, term, trace, (time.perf_counter() - t0) * 1e3)


def solve_pure_eg(pd: Problem, cfg: SolverCfg | None = None) -> Report:
    """solver.py:236-289: the extragradient-only comparator."""
    cfg = cfg or SolverCfg()
    t0 = time.perf_counter()
    trace: list[Record] = []
    v = Pair(np.zeros(pd.n), np.zeros((pd.n, pd.n)))
    r_v, _ = residual_parts(pd, v)
    res = r_v.norm()
    _finite(res, r_v, trace)
    term = "converged" if res <= cfg.residual_tol else "max_iter"
    k = 0
    while term != "converged" and k < cfg.max_iter:
        t_it = time.perf_counter()
        v = eg_step(pd, v, cfg.eg_stepsize)
        r_v, _ = residual_parts(pd, v)
        res = r_v.norm()
        _finite(res, r_v, trace)
        nan = float("nan")
        trace.append(Record(k, res, nan, res, "eg", nan, nan, 0, False, nan, nan,
                            (time.perf_counter() - t_it) * 1e3))
        k += 1
        if res <= cfg.residual_tol:
            term = "converged"
    ot = ot_estimate(pd, v.g) if pd.embed is not None else None
    return Report(v.g, v.x, ot, res, term, trace, (time.perf_counter() - t0) * 1e3)


def ot_estimate(pd: Problem, g: np.ndarray) -> float:
    """problem.py:244-251: (q² − γ̂·embed)/(2λ₂)."""
    if pd.embed is None:
        raise ValueError("instance carries no embedding sums")
    return (pd.q_sq - float(g @ pd.embed)) / (2.0 * pd.l2)


def evaluate_map(pd: Problem, xs: np.ndarray, g: np.ndarray, queries: np.ndarray):
    """problem.py:254-284: potential u(x) and map T(x) = x − ∇u(x)."""
    queries = np.atleast_2d(np.asarray(queries, dtype=float))
    tl = 2.0 * pd.l2
    sq = pd.bw_sq
    gs = gaussian_gram(sq, xs, queries)
    gf = gaussian_gram(sq, pd.xt, queries)
    emb = gs.mean(axis=0)
    wgt = g @ gf
    u = (emb - wgt) / tl
    ps = (gs.T @ xs) / xs.shape[0] - emb[:, None] * queries
    pf = gf.T @ (g[:, None] * pd.xt) - wgt[:, None] * queries
    return u, queries - (ps - pf) / (tl * sq)


def with_path(op: Elim, pos_path: bool) -> Elim:
    """Force an eliminator path (test_psdcone.py:_flip_path)."""
    return replace(op, pos_path=pos_path)
