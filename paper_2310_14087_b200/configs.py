"""Seeded synthetic workloads for the BASELINE.json configs.

The reference ships no benchmark data; BASELINE.json names five synthetic
configurations.  The draw order below is normative: the oracle, the GPU
solver and the bench consume the *same host arrays*.  Everything is
``numpy.random.default_rng(seed)`` in FP64.

Each builder returns a :class:`Workload` holding the samples, the filling
points and the scalar parameters that ``assemble`` takes
(reference ``pkg/src/kot/problem.py:135-144``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    xs: np.ndarray  # source samples (n, d)
    ys: np.ndarray  # target samples (n, d)
    xt: np.ndarray  # filling points, x part (l, d)
    yt: np.ndarray  # filling points, y part (l, d)
    bandwidth_sq: float
    lambda1: float
    lambda2: float

    @property
    def l(self) -> int:  # noqa: E743 - paper notation
        return self.xt.shape[0]

    @property
    def d(self) -> int:
        return self.xs.shape[1]


def _radial_clip(p: np.ndarray) -> np.ndarray:
    nrm = np.linalg.norm(p, axis=1, keepdims=True)
    return p / np.maximum(nrm, 1.0)


def config1(seed: int = 0) -> Workload:
    """d=2, n=l=100, N(0,0.1 I) -> N(0.3·1, 0.05 I) clipped to [-1,1]^2; sigma=0.5."""
    rng = np.random.default_rng(seed)
    n = l = 100
    d = 2
    xs = np.clip(rng.normal(0.0, np.sqrt(0.1), size=(n, d)), -1.0, 1.0)
    ys = np.clip(rng.normal(0.3, np.sqrt(0.05), size=(n, d)), -1.0, 1.0)
    f = rng.uniform(-1.0, 1.0, size=(l, 2 * d))
    return Workload("cfg1", xs, ys, f[:, :d].copy(), f[:, d:].copy(), 0.25, 1e-3, 1.0 / l)


def _two_component(rng: np.random.Generator, n: int, d: int, shift: float) -> np.ndarray:
    means = np.zeros((2, d))
    means[0, 0] = 0.3
    means[1, 0] = -0.3
    labels = rng.integers(0, 2, size=n)
    pts = means[labels] + 0.15 * rng.standard_normal((n, d)) + shift
    return np.clip(pts, -1.0, 1.0)


def config2(seed: int = 0, n: int = 500) -> Workload:
    """d=5, n=l=500, two-component mixtures (target shifted by 0.2·1); sigma=1."""
    rng = np.random.default_rng(seed)
    d = 5
    xs = _two_component(rng, n, d, 0.0)
    ys = _two_component(rng, n, d, 0.2)
    f = rng.uniform(-1.0, 1.0, size=(n, 2 * d))
    return Workload("cfg2", xs, ys, f[:, :d].copy(), f[:, d:].copy(), 1.0, 1e-3, 1.0 / n)


def _four_component(rng: np.random.Generator, n: int, d: int) -> np.ndarray:
    means = rng.uniform(-0.5, 0.5, size=(4, d))
    weights = rng.dirichlet(np.ones(4))
    labels = rng.choice(4, size=n, p=weights)
    pts = means[labels] + 0.1 * rng.standard_normal((n, d))
    return _radial_clip(pts)


def config3(seed: int = 0, n: int = 2000, sigma: float = 1.5) -> Workload:
    """d=10, n=l=2000, 4-component mixtures clipped to the unit ball; sigma=1.5 (headline)."""
    rng = np.random.default_rng(seed)
    d = 10
    xs = _four_component(rng, n, d)
    ys = _four_component(rng, n, d)
    f = rng.uniform(-1.0, 1.0, size=(n, 2 * d))
    return Workload(f"cfg3[n={n}]", xs, ys, f[:, :d].copy(), f[:, d:].copy(), sigma * sigma, 1e-4, 1.0 / n)


def config4(seed: int = 0, n: int = 8192) -> Workload:
    """d=64, n=l=8192 embedding-like data (rank-8 + noise, rotated target); sigma=1."""
    rng = np.random.default_rng(seed)
    d = 64
    g = rng.standard_normal((n, 8))
    w = rng.standard_normal((8, d))
    xs = g @ w + 0.05 * rng.standard_normal((n, d))
    xs /= np.linalg.norm(xs, axis=1, keepdims=True)
    qm, rm = np.linalg.qr(rng.standard_normal((d, d)))
    qm = qm * np.sign(np.diag(rm))[None, :]
    u = rng.standard_normal(d)
    u /= np.linalg.norm(u)
    ys = xs @ qm + 0.1 * u[None, :]
    a = rng.integers(0, n, size=n)
    b = rng.integers(0, n, size=n)
    xt = xs[a] + 0.05 * rng.standard_normal((n, d))
    yt = ys[b] + 0.05 * rng.standard_normal((n, d))
    return Workload("cfg4", xs, ys, xt, yt, 1.0, 1e-4, 1.0 / n)


CFG5_SIGMAS = (0.5, 1.0, 1.5, 2.0)


def config5_member(seed: int, n: int = 1000) -> Workload:
    """One member of the 512-problem batch: cfg3 family at n=l=1000, sigma by seed % 4."""
    sigma = CFG5_SIGMAS[seed % 4]
    w = config3(seed=seed, n=n, sigma=sigma)
    return Workload(f"cfg5[{seed}]", w.xs, w.ys, w.xt, w.yt, w.bandwidth_sq, w.lambda1, w.lambda2)


def eg_stepsize(q_mat: np.ndarray, k_mat: np.ndarray, lambda2: float, c: float = 0.5) -> float:
    """EG stepsize rule of SURVEY.md §8(d): c / (||Q||_F/(2 l2) + ||K||_F).

    The reference default (``EgConfig.stepsize=0.01``, ``pkg/src/kot/eg.py:20``)
    diverges at these configs; both sides must use this value.
    """
    return c / (np.linalg.norm(q_mat) / (2.0 * lambda2) + np.linalg.norm(k_mat))


PROFILES = {
    # SURVEY.md §8(d) solver profiles; identical on both sides.
    "paper": dict(),
    "tight": dict(alpha1=1e-8, alpha2=1e-4, cg_max=500),
}
