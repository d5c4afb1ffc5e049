"""Dual instance, residual map and Jacobian (mirror of reference ``kot.problem``).

Reference: ``pkg/src/kot/problem.py``.  ``ProblemData`` keeps the
reference's host fields (NumPy arrays) and, lazily, a device-resident copy
(``kot_problem`` handle) that every operator and ``solve`` run against;
``assemble`` builds the instance on the GPU and keeps that handle.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from paper_2310_14087_b200 import _lib
from paper_2310_14087_b200.kernels import KernelSpec, SampleSet
from paper_2310_14087_b200.linalg import SpectralDecomp, symmetrize


@dataclass(frozen=True)
class FillingPoints:
    """Paired grid points at which the transport equality is sampled (problem.py:25-42)."""

    x_tilde: np.ndarray
    y_tilde: np.ndarray

    def __post_init__(self) -> None:
        x = np.atleast_2d(np.asarray(self.x_tilde, dtype=float))
        y = np.atleast_2d(np.asarray(self.y_tilde, dtype=float))
        if x.shape != y.shape or x.shape[0] < 1:
            raise ValueError("x_tilde and y_tilde must have equal shape (n, d), n >= 1")
        object.__setattr__(self, "x_tilde", x)
        object.__setattr__(self, "y_tilde", y)

    @property
    def count(self) -> int:
        return self.x_tilde.shape[0]


@dataclass
class IteratePair:
    """Solver state w = (gamma, X); pair norm ||γ||₂ + ||X||_F (problem.py:45-83)."""

    gamma: np.ndarray
    x_mat: np.ndarray

    def norm(self) -> float:
        return float(np.linalg.norm(self.gamma) + np.linalg.norm(self.x_mat))

    def dot(self, other: "IteratePair") -> float:
        return float(self.gamma @ other.gamma + np.sum(self.x_mat * other.x_mat))

    def copy(self) -> "IteratePair":
        return IteratePair(self.gamma.copy(), self.x_mat.copy())

    def __add__(self, other: "IteratePair") -> "IteratePair":
        return IteratePair(self.gamma + other.gamma, self.x_mat + other.x_mat)

    def __sub__(self, other: "IteratePair") -> "IteratePair":
        return IteratePair(self.gamma - other.gamma, self.x_mat - other.x_mat)

    def __mul__(self, c: float) -> "IteratePair":
        return IteratePair(c * self.gamma, c * self.x_mat)

    __rmul__ = __mul__

    def is_finite(self) -> bool:
        return bool(np.all(np.isfinite(self.gamma)) and np.all(np.isfinite(self.x_mat)))


def zero_pair(n: int) -> IteratePair:
    return IteratePair(np.zeros(n), np.zeros((n, n)))


class DeviceProblem:
    """Owns a ``kot_problem*`` (device-resident Q, z, R, embed + solver workspace)."""

    def __init__(self, handle: int, device: int):
        self.handle = C.c_void_p(handle)
        self.device = device

    def __del__(self):
        try:
            if self.handle:
                _lib.lib().kot_problem_destroy(self.handle)
                self.handle = C.c_void_p(0)
        except Exception:  # interpreter shutdown
            pass


@dataclass(eq=False)
class ProblemData:
    """Assembled dual instance (problem.py:86-123); R.T R = K + jitter I, rows of R are features."""

    q_mat: np.ndarray
    z: np.ndarray
    q_sq: float
    chol_upper: np.ndarray
    lambda1: float
    lambda2: float
    embed_sum: np.ndarray | None = None
    filling: FillingPoints | None = None
    spec_x: KernelSpec | None = None
    spec_y: KernelSpec | None = None
    spec_xy: KernelSpec | None = None
    jitter: float = 0.0
    # device-resident copy and pair Gram: never copied by dataclasses.replace (init=False), dropped
    # whenever a field they were built from is reassigned (__setattr__ below)
    _dev: DeviceProblem | None = field(default=None, init=False, repr=False, compare=False)
    _kmat: np.ndarray | None = field(default=None, init=False, repr=False, compare=False)

    # fields the uploaded instance is built from / the pair Gram depends on
    _DEVICE_FIELDS = frozenset({"q_mat", "z", "q_sq", "chol_upper", "lambda1", "lambda2", "embed_sum", "jitter"})
    _KMAT_FIELDS = frozenset({"filling", "spec_xy", "chol_upper"})

    def __setattr__(self, name, value):
        # Reassigning a data field invalidates the device copy (the reference ProblemData is a plain
        # mutable dataclass).  Arrays are uploaded as they are at the first GPU call: mutate them in
        # place only before that, or reassign the field (or call release_device()) afterwards.
        if name in ProblemData._DEVICE_FIELDS and "_dev" in self.__dict__:
            object.__setattr__(self, "_dev", None)
        if name in ProblemData._KMAT_FIELDS and "_kmat" in self.__dict__:
            object.__setattr__(self, "_kmat", None)
        object.__setattr__(self, name, value)

    def __post_init__(self) -> None:
        self.q_mat = symmetrize(np.asarray(self.q_mat, dtype=float))
        self.z = np.asarray(self.z, dtype=float)
        self.chol_upper = np.asarray(self.chol_upper, dtype=float)
        n = self.q_mat.shape[0]
        if self.z.shape != (n,) or self.chol_upper.shape != (n, n):
            raise ValueError("inconsistent instance dimensions")
        if self.lambda1 <= 0.0 or self.lambda2 <= 0.0:
            raise ValueError("regularization parameters must be positive")

    @property
    def n(self) -> int:
        return self.z.shape[0]

    def device_problem(self, device: int | None = None) -> DeviceProblem:
        """Upload (once) and return the device-resident copy of this instance."""
        dev = _lib.default_device() if device is None else device
        if self._dev is None or self._dev.device != dev:
            h = C.c_void_p(0)
            emb = None if self.embed_sum is None else _lib.f64(self.embed_sum)
            q, z, r = _lib.f64(self.q_mat), _lib.f64(self.z), _lib.f64(self.chol_upper)
            _lib.check(_lib.lib().kot_problem_create(
                _lib.ptr(q), _lib.ptr(z), float(self.q_sq), _lib.ptr(r), _lib.ptr(emb), self.n,
                float(self.lambda1), float(self.lambda2), float(self.jitter), dev, C.byref(h)))
            self._dev = DeviceProblem(h.value, dev)
        return self._dev

    def release_device(self) -> None:
        """Free the device-resident copy (its memory returns to the library's pool)."""
        self._dev = None

    def pair_gram(self) -> np.ndarray | None:
        """The pair-kernel Gram K (only for instances built by ``assemble``)."""
        return self._kmat


def build_kernel_specs(dim: int, bandwidth_sq: float) -> tuple[KernelSpec, KernelSpec, KernelSpec]:
    """One bandwidth, three kernels: marginals on R^d, pairs on R^{2d} (problem.py:126-132)."""
    return (KernelSpec(bandwidth_sq, dim), KernelSpec(bandwidth_sq, dim), KernelSpec(bandwidth_sq, 2 * dim))


def assemble(samples_mu: SampleSet, samples_nu: SampleSet, filling: FillingPoints, lambda1: float,
             lambda2: float, spec_x: KernelSpec, spec_y: KernelSpec, spec_xy: KernelSpec,
             device: int | None = None) -> ProblemData:
    """Build the dual instance on the GPU (problem.py:135-169)."""
    if lambda1 <= 0.0 or lambda2 <= 0.0:
        raise ValueError("lambda1 and lambda2 must be positive")
    if len(samples_mu) == 0 or len(samples_nu) == 0:
        raise ValueError("sample set is empty")
    xt, yt = _lib.f64(filling.x_tilde), _lib.f64(filling.y_tilde)
    l, d = xt.shape
    for spec, dim in ((spec_x, d), (spec_y, d), (spec_xy, 2 * d)):
        if spec.input_dim != dim:
            raise ValueError(f"kernel expects dimension {spec.input_dim}, got {dim}")
    xs, ys = _lib.f64(samples_mu.points), _lib.f64(samples_nu.points)
    if xs.shape[1] != d or ys.shape[1] != d:
        raise ValueError("sample dimension mismatch")
    dev = _lib.default_device() if device is None else device
    h = C.c_void_p(0)
    _lib.check(_lib.lib().kot_assemble(_lib.ptr(xs), xs.shape[0], _lib.ptr(ys), ys.shape[0], _lib.ptr(xt),
                                       _lib.ptr(yt), l, d, float(spec_x.bandwidth_sq), float(spec_y.bandwidth_sq),
                                       float(spec_xy.bandwidth_sq), float(lambda1), float(lambda2), dev,
                                       C.byref(h)))
    dp = DeviceProblem(h.value, dev)
    q, z, r, emb, kmat = np.empty((l, l)), np.empty(l), np.empty((l, l)), np.empty(l), np.empty((l, l))
    _lib.check(_lib.lib().kot_problem_download(dp.handle, _lib.ptr(q), _lib.ptr(z), _lib.ptr(r), _lib.ptr(emb),
                                               _lib.ptr(kmat)))
    qsq, jit = C.c_double(), C.c_double()
    _lib.check(_lib.lib().kot_problem_info(dp.handle, None, C.byref(qsq), C.byref(jit), None, None, None))
    # The device mirrors Q's triangle, so it is bitwise symmetric already: the instance is filled in
    # directly, without __post_init__'s symmetrisation pass over the ℓ × ℓ host array (its other checks
    # — shapes, positive λ — hold by construction).
    pd = object.__new__(ProblemData)
    for name, value in (("q_mat", q), ("z", z), ("q_sq", float(qsq.value)), ("chol_upper", r),
                        ("lambda1", lambda1), ("lambda2", lambda2), ("embed_sum", emb), ("filling", filling),
                        ("spec_x", spec_x), ("spec_y", spec_y), ("spec_xy", spec_xy), ("jitter", float(jit.value)),
                        ("_dev", dp), ("_kmat", kmat)):
        object.__setattr__(pd, name, value)
    return pd


def phi_forward(pd: ProblemData, x_mat) -> np.ndarray:
    """Φ(X)_i = r_i X r_iᵀ, r_i = row i of R (problem.py:172-177)."""
    x = _lib.f64(x_mat)
    if x.shape != (pd.n, pd.n):
        raise ValueError("matrix order mismatch")
    out = np.empty(pd.n)
    _lib.check(_lib.lib().kot_phi_forward(pd.device_problem().handle, _lib.ptr(x), _lib.ptr(out)))
    return out


def phi_adjoint(pd: ProblemData, gamma) -> np.ndarray:
    """Φ*(γ) = Rᵀ diag(γ) R, exactly symmetric (problem.py:180-185)."""
    g = _lib.f64(gamma)
    if g.shape != (pd.n,):
        raise ValueError("vector length mismatch")
    out = np.empty((pd.n, pd.n))
    _lib.check(_lib.lib().kot_phi_adjoint(pd.device_problem().handle, _lib.ptr(g), _lib.ptr(out)))
    return out


def objective(pd: ProblemData, gamma) -> float:
    """Dual quadratic objective value at γ (problem.py:192-196)."""
    g = _lib.f64(gamma, (pd.n,))
    out = C.c_double()
    _lib.check(_lib.lib().kot_objective(pd.device_problem().handle, _lib.ptr(g), C.byref(out)))
    return float(out.value)


def ot_estimate(pd: ProblemData, gamma_hat) -> float:
    """(q² − γ̂·embed)/(2λ₂) (problem.py:244-251)."""
    if pd.embed_sum is None:
        raise ValueError("instance carries no embedding sums; assemble() provides them")
    g = _lib.f64(gamma_hat, (pd.n,))
    out = C.c_double()
    _lib.check(_lib.lib().kot_ot_estimate(pd.device_problem().handle, _lib.ptr(g), C.byref(out)))
    return float(out.value)


def objective_grad(pd: ProblemData, gamma) -> np.ndarray:
    """(Qγ − z)/(2λ₂) (problem.py:188-189)."""
    g = _lib.f64(gamma, (pd.n,))
    out = np.empty(pd.n)
    _lib.check(_lib.lib().kot_objective_grad(pd.device_problem().handle, _lib.ptr(g), 0, _lib.ptr(out)))
    return out


def objective_grad_dir(pd: ProblemData, dgamma) -> np.ndarray:
    """Qd/(2λ₂) (problem.py:239-241)."""
    g = _lib.f64(dgamma, (pd.n,))
    out = np.empty(pd.n)
    _lib.check(_lib.lib().kot_objective_grad(pd.device_problem().handle, _lib.ptr(g), 1, _lib.ptr(out)))
    return out


def constraint_matrix(pd: ProblemData, gamma) -> np.ndarray:
    """Φ*(γ) + λ₁I, the matrix whose positive semidefiniteness the dual constrains (problem.py:199-201)."""
    g = _lib.f64(gamma, (pd.n,))
    out = np.empty((pd.n, pd.n))
    _lib.check(_lib.lib().kot_constraint_matrix(pd.device_problem().handle, _lib.ptr(g), _lib.ptr(out)))
    return out


def residual_parts(pd: ProblemData, w: IteratePair) -> tuple[IteratePair, SpectralDecomp]:
    """(r1, r2) and the eigendecomposition of Z = sym(X) − (Φ*(γ)+λ₁I) (problem.py:204-214)."""
    g, x = _lib.f64(w.gamma, (pd.n,)), _lib.f64(w.x_mat, (pd.n, pd.n))
    r1, r2, ev, vecs = np.empty(pd.n), np.empty((pd.n, pd.n)), np.empty(pd.n), np.empty((pd.n, pd.n))
    k, res = C.c_int(), C.c_double()
    _lib.check(_lib.lib().kot_residual_parts(pd.device_problem().handle, _lib.ptr(g), _lib.ptr(x), _lib.ptr(r1),
                                             _lib.ptr(r2), _lib.ptr(ev), C.byref(k), C.byref(res),
                                             _lib.ptr(vecs)))
    kk = int(k.value)
    return IteratePair(r1, r2), SpectralDecomp(eigvecs=vecs, eigvals=ev, pos_idx=np.arange(kk),
                                               nonpos_idx=np.arange(kk, pd.n))


def apply_jacobian(pd: ProblemData, coeffs, mu: float, dw: IteratePair) -> IteratePair:
    """Regularized generalized Jacobian (J + μI)dw at ``coeffs``' decomposition (problem.py:222-236):
    top = Qdγ/(2λ₂) + μdγ − Φ(dX), bottom = M[Φ*(dγ) − dX] + (1+μ)dX."""
    dc = coeffs.decomp
    dg, dx = _lib.f64(dw.gamma, (pd.n,)), _lib.f64(dw.x_mat, (pd.n, pd.n))
    top, bottom = np.empty(pd.n), np.empty((pd.n, pd.n))
    _lib.check(_lib.lib().kot_apply_jacobian(pd.device_problem().handle, _lib.ptr(_lib.f64(dc.eigvecs)),
                                             _lib.ptr(_lib.f64(dc.eigvals)), dc.n_pos, float(mu), _lib.ptr(dg),
                                             _lib.ptr(dx), _lib.ptr(top), _lib.ptr(bottom)))
    return IteratePair(top, bottom)


def evaluate_map(pd: ProblemData, samples_mu: SampleSet, gamma_hat, queries) -> tuple[np.ndarray, np.ndarray]:
    """Dual potential u and transport map T = id − ∇u at query points (problem.py:254-284), on the GPU."""
    if pd.filling is None or pd.spec_x is None:
        raise ValueError("instance carries no filling points / kernel specs")
    q = _lib.f64(np.atleast_2d(np.asarray(queries, dtype=float)))
    if q.shape[1] != pd.spec_x.input_dim:
        raise ValueError("query dimension mismatch")
    xs, xt = _lib.f64(samples_mu.points), _lib.f64(pd.filling.x_tilde)
    g = _lib.f64(gamma_hat, (pd.n,))
    m, d = q.shape
    u, t = np.empty(m), np.empty((m, d))
    dev = pd._dev.device if pd._dev is not None else _lib.default_device()
    _lib.check(_lib.lib().kot_evaluate_map(_lib.ptr(xs), xs.shape[0], _lib.ptr(xt), _lib.ptr(g), pd.n, _lib.ptr(q),
                                           m, d, float(pd.spec_x.bandwidth_sq), float(pd.lambda2), dev,
                                           _lib.ptr(u), _lib.ptr(t)))
    return u, t


def potential_and_map(pd: ProblemData, samples_mu: SampleSet, gamma_hat, query) -> tuple[float, np.ndarray]:
    """Single-point wrapper around :func:`evaluate_map` (problem.py:287-295)."""
    u, t = evaluate_map(pd, samples_mu, gamma_hat, np.atleast_2d(query))
    return float(u[0]), t[0]


def residual(pd: ProblemData, w: IteratePair) -> IteratePair:
    """Nonsmooth KKT residual (problem.py:217-219)."""
    return residual_parts(pd, w)[0]


__all__ = ["FillingPoints", "IteratePair", "ProblemData", "DeviceProblem", "SpectralDecomp", "zero_pair",
           "build_kernel_specs", "assemble", "phi_forward", "phi_adjoint", "objective", "objective_grad",
           "objective_grad_dir", "constraint_matrix", "ot_estimate", "residual_parts", "residual",
           "apply_jacobian", "evaluate_map", "potential_and_map"]
