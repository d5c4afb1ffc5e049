"""Projected extragradient safeguard step (mirror of reference ``kot.eg``).

Reference: ``pkg/src/kot/eg.py``; the step runs on the device (two
eigensolves + PSD projections, csrc/ssn.cu eg_step).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from paper_2310_14087_b200 import _lib
from paper_2310_14087_b200.problem import IteratePair, ProblemData


@dataclass(frozen=True)
class EgConfig:
    """eg.py:18-24."""

    stepsize: float = 0.01

    def __post_init__(self) -> None:
        if self.stepsize <= 0.0:
            raise ValueError("stepsize must be positive")


def eg_step(pd: ProblemData, v: IteratePair, cfg: EgConfig) -> IteratePair:
    """Two-stage projected extragradient update; the output matrix is PSD (eg.py:34-41)."""
    g, x = _lib.f64(v.gamma, (pd.n,)), _lib.f64(v.x_mat, (pd.n, pd.n))
    go, xo = np.empty(pd.n), np.empty((pd.n, pd.n))
    _lib.check(_lib.lib().kot_eg_step(pd.device_problem().handle, _lib.ptr(g), _lib.ptr(x), float(cfg.stepsize),
                                      _lib.ptr(go), _lib.ptr(xo)))
    return IteratePair(go, xo)
