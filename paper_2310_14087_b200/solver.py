"""EG-safeguarded regularized SSN solve loop (mirror of reference ``kot.solver``).

Reference: ``pkg/src/kot/solver.py``.  The whole loop (Algorithm 2) runs in
libkotgpu on device-resident state; the report, trace and observer callback
have the reference's types and semantics.
"""

from __future__ import annotations

import ctypes as C
import logging
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from paper_2310_14087_b200 import _lib
from paper_2310_14087_b200._lib import SolverNumericsError  # noqa: F401
from paper_2310_14087_b200.eg import EgConfig
from paper_2310_14087_b200.newton import NewtonConfig, cfg_struct
from paper_2310_14087_b200.problem import IteratePair, ProblemData

log = logging.getLogger("kot.solver")

CONVERGED = "converged"
MAX_ITER = "max_iter"


@dataclass(frozen=True)
class SolverConfig:
    """solver.py:36-51."""

    newton: NewtonConfig = field(default_factory=NewtonConfig)
    eg: EgConfig = field(default_factory=EgConfig)
    residual_tol: float = 0.005
    max_iter: int = 500
    seed: int = 0
    safeguard_every: int = 1

    def __post_init__(self) -> None:
        if self.residual_tol <= 0.0:
            raise ValueError("residual_tol must be positive")
        if self.max_iter < 1:
            raise ValueError("max_iter must be >= 1")
        if self.safeguard_every < 1:
            raise ValueError("safeguard_every must be >= 1")

    def to_c(self) -> _lib.SolverCfgC:
        return cfg_struct(self.newton, self.eg.stepsize, self.residual_tol, self.max_iter, self.safeguard_every)


@dataclass(frozen=True)
class IterationRecord:
    """One row of the solve trace; times in milliseconds (solver.py:54-73) + n_pos, attempts."""

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
    eg_ms: float
    newton_ms: float
    cg_ms: float
    resid_ms: float
    step_ms: float
    n_pos: int = -1
    attempts: int = 0


@dataclass(frozen=True)
class IterationProbe:
    """Raw per-iteration objects handed to an observer callback (solver.py:76-86)."""

    iteration: int
    w: IteratePair
    r: IteratePair
    mu: float
    theta: float
    dw: IteratePair
    criterion_met: bool


@dataclass
class SolverReport:
    """solver.py:89-101."""

    gamma_hat: np.ndarray
    x_hat: np.ndarray
    ot_estimate: float | None
    residual_norm: float
    termination: str
    trace: list[IterationRecord]
    total_ms: float

    @property
    def iterations(self) -> int:
        return len(self.trace)


def _record(r: _lib.IterRecordC) -> IterationRecord:
    return IterationRecord(r.iteration, r.res_accepted, r.res_ssn, r.res_eg, "ssn" if r.accepted_ssn else "eg",
                           r.theta, r.mu, r.cg_iters, bool(r.criterion_met), r.crit_lhs, r.crit_rhs, r.eg_ms,
                           r.newton_ms, r.cg_ms, r.resid_ms, r.step_ms, r.n_pos, r.attempts)


def _run(pd: ProblemData, cfg: SolverConfig, on_iteration, pure_eg: bool, want_x: bool = True) -> SolverReport:
    n = pd.n
    dp = pd.device_problem()
    c = cfg.to_c()
    gamma = np.empty(n)
    x = np.empty((n, n)) if want_x else None
    trace = (_lib.IterRecordC * cfg.max_iter)()
    rep = _lib.ReportC()
    if pure_eg:
        st = _lib.lib().kot_solve_pure_eg(dp.handle, C.byref(c), _lib.ptr(gamma), _lib.ptr(x), trace,
                                          cfg.max_iter, C.byref(rep))
    else:
        cb = _lib.IterCB(0)
        raised: list[BaseException] = []
        if on_iteration is not None:
            def _cb(user, k, wg, wx, rg, rx, mu, theta, dg, dx, met):
                def vec(p):
                    return np.ctypeslib.as_array(p, shape=(n,)).copy()

                def mat(p):
                    return np.ctypeslib.as_array(p, shape=(n, n)).copy()

                try:
                    on_iteration(IterationProbe(k, IteratePair(vec(wg), mat(wx)), IteratePair(vec(rg), mat(rx)),
                                                float(mu), float(theta), IteratePair(vec(dg), mat(dx)), bool(met)))
                except BaseException as e:  # noqa: BLE001 — re-raised below, as the reference propagates it
                    raised.append(e)
                    return 1
                return 0
            cb = _lib.IterCB(_cb)
        st = _lib.lib().kot_solve(dp.handle, C.byref(c), cb, None, _lib.ptr(gamma), _lib.ptr(x), trace,
                                  cfg.max_iter, C.byref(rep))
        if raised:  # the observer's exception ends the solve (reference solver.py:170-181)
            raise raised[0]
    recs = [_record(trace[i]) for i in range(min(rep.iterations, cfg.max_iter))]
    _lib.check(st, recs)
    for r in recs:
        log.debug("iter %d accepted=%s res=%.3e (ssn %.3e, eg %.3e) theta=%.2e cg=%d", r.iteration, r.accepted,
                  r.res_accepted, r.res_ssn, r.res_eg, r.theta, r.cg_iters)
    ot = float(rep.ot_estimate) if pd.embed_sum is not None else None
    return SolverReport(gamma_hat=gamma, x_hat=x, ot_estimate=ot, residual_norm=float(rep.residual_norm),
                        termination=CONVERGED if rep.converged else MAX_ITER, trace=recs, total_ms=rep.total_ms)


def solve(pd: ProblemData, cfg: SolverConfig | None = None,
          on_iteration: Callable[[IterationProbe], None] | None = None) -> SolverReport:
    """Run the safeguarded Newton loop from the zero pair on the GPU (solver.py:114-233)."""
    return _run(pd, cfg or SolverConfig(), on_iteration, False)


def solve_pure_eg(pd: ProblemData, cfg: SolverConfig | None = None) -> SolverReport:
    """Baseline: the extragradient step alone to the residual tolerance (solver.py:236-289)."""
    return _run(pd, cfg or SolverConfig(), None, True)


def iterate(pd: ProblemData, cfg: SolverConfig, w: IteratePair, v: IteratePair, theta: float, k: int):
    """One loop body from (w, v, θ) at iteration k — the lock-step replay unit."""
    n = pd.n
    c = cfg.to_c()
    wg, wx, vg, vx = (np.empty(n), np.empty((n, n)), np.empty(n), np.empty((n, n)))
    th = C.c_double()
    rec = _lib.IterRecordC()
    _lib.check(_lib.lib().kot_iterate(pd.device_problem().handle, C.byref(c), _lib.ptr(_lib.f64(w.gamma)),
                                      _lib.ptr(_lib.f64(w.x_mat)), _lib.ptr(_lib.f64(v.gamma)),
                                      _lib.ptr(_lib.f64(v.x_mat)), float(theta), int(k), _lib.ptr(wg),
                                      _lib.ptr(wx), _lib.ptr(vg), _lib.ptr(vx), C.byref(th), C.byref(rec)))
    return IteratePair(wg, wx), IteratePair(vg, vx), float(th.value), _record(rec)


class Session:
    """A solve driven in chunks on device-resident state (used by bench.py).

    ``step(k)`` runs k loop bodies of Algorithm 2 continuing the same trajectory;
    ``stream`` is the CUDA stream every kernel of this problem is launched on.
    """

    def __init__(self, pd: ProblemData, cfg: SolverConfig):
        self.pd = pd
        self.cfg = cfg
        self._dp = pd.device_problem()
        self._c = cfg.to_c()
        h = C.c_void_p(0)
        _lib.check(_lib.lib().kot_session_begin(self._dp.handle, C.byref(self._c), C.byref(h)))
        self._h = h
        self.records: list[IterationRecord] = []

    @property
    def stream(self) -> int:
        return int(_lib.lib().kot_problem_stream(self._dp.handle) or 0)

    def step(self, iters: int) -> int:
        recs = (_lib.IterRecordC * max(iters, 1))()
        done = C.c_int(0)
        _lib.check(_lib.lib().kot_session_step(self._h, int(iters), recs, C.byref(done)))
        self.records.extend(_record(recs[i]) for i in range(done.value))
        return int(done.value)

    def result(self, want_x: bool = False) -> SolverReport:
        n = self.pd.n
        gamma = np.empty(n)
        x = np.empty((n, n)) if want_x else None
        rep = _lib.ReportC()
        _lib.check(_lib.lib().kot_session_result(self._h, _lib.ptr(gamma), _lib.ptr(x), C.byref(rep)))
        ot = float(rep.ot_estimate) if self.pd.embed_sum is not None else None
        return SolverReport(gamma, x, ot, float(rep.residual_norm), CONVERGED if rep.converged else MAX_ITER,
                            list(self.records), float("nan"))

    def state(self):
        """(w, v, θ) between two iterations (host copies)."""
        n = self.pd.n
        wg, wx, vg, vx = np.empty(n), np.empty((n, n)), np.empty(n), np.empty((n, n))
        th = C.c_double()
        _lib.check(_lib.lib().kot_session_state(self._h, _lib.ptr(wg), _lib.ptr(wx), _lib.ptr(vg), _lib.ptr(vx),
                                                C.byref(th)))
        return IteratePair(wg, wx), IteratePair(vg, vx), float(th.value)

    def close(self):
        if self._h:
            _lib.lib().kot_session_end(self._h)
            self._h = C.c_void_p(0)
        self._dp = None  # the instance's device problem may be released from here on

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
