"""ctypes binding of libkotgpu (C ABI in include/kotgpu.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
``-gencode arch=compute_100a,code=sm_100a``).  There is no CPU fallback: if
the library is missing every call raises, and on a machine without a B200 the
calls fail with the CUDA error the runtime reports.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KOT_LIB_PATH") or os.path.join(_HERE, "libkotgpu.so")  # override: diagnostics

dptr = C.POINTER(C.c_double)
iptr = C.POINTER(C.c_int)


class SolverCfgC(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "tau", "kappa", "alpha1", "alpha2", "beta0", "beta1", "beta2", "theta_min", "theta_max", "theta0")] + [
        ("cg_max", C.c_int), ("cg_restarts", C.c_int), ("cg_tol", C.c_double), ("has_cg_tol", C.c_int),
        ("eg_stepsize", C.c_double), ("residual_tol", C.c_double), ("max_iter", C.c_int),
        ("safeguard_every", C.c_int)]


class IterRecordC(C.Structure):
    _fields_ = [("iteration", C.c_int), ("res_accepted", C.c_double), ("res_ssn", C.c_double),
                ("res_eg", C.c_double), ("accepted_ssn", C.c_int), ("theta", C.c_double), ("mu", C.c_double),
                ("cg_iters", C.c_int), ("criterion_met", C.c_int), ("crit_lhs", C.c_double),
                ("crit_rhs", C.c_double), ("eg_ms", C.c_double), ("newton_ms", C.c_double),
                ("cg_ms", C.c_double), ("resid_ms", C.c_double), ("step_ms", C.c_double),
                ("n_pos", C.c_int), ("attempts", C.c_int)]


class ReportC(C.Structure):
    _fields_ = [("converged", C.c_int), ("iterations", C.c_int), ("residual_norm", C.c_double),
                ("ot_estimate", C.c_double), ("total_ms", C.c_double)]


class ProfEntryC(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("calls", C.c_longlong), ("ms", C.c_double), ("flops", C.c_double),
                ("bytes", C.c_double)]


MatvecFn = C.CFUNCTYPE(C.c_int, C.c_void_p, dptr, dptr)

CommFn = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, dptr, C.c_long, C.c_long, C.c_int, C.c_int)

IterCB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, dptr, dptr, dptr, dptr, C.c_double, C.c_double, dptr, dptr,
                     C.c_int)

# name -> (restype, argtypes)
_SIGS = {
    "kot_last_error": (C.c_char_p, []),
    "kot_launch_count": (C.c_longlong, []),
    "kot_problem_create": (C.c_int, [dptr, dptr, C.c_double, dptr, dptr, C.c_int, C.c_double, C.c_double,
                                     C.c_double, C.c_int, C.POINTER(C.c_void_p)]),
    "kot_assemble": (C.c_int, [dptr, C.c_int, dptr, C.c_int, dptr, dptr, C.c_int, C.c_int, C.c_double, C.c_double,
                               C.c_double, C.c_double, C.c_double, C.c_int, C.POINTER(C.c_void_p)]),
    "kot_problem_info": (C.c_int, [C.c_void_p, iptr, dptr, dptr, dptr, dptr, iptr]),
    "kot_problem_download": (C.c_int, [C.c_void_p, dptr, dptr, dptr, dptr, dptr]),
    "kot_problem_destroy": (None, [C.c_void_p]),
    "kot_solve": (C.c_int, [C.c_void_p, C.POINTER(SolverCfgC), IterCB, C.c_void_p, dptr, dptr,
                            C.POINTER(IterRecordC), C.c_int, C.POINTER(ReportC)]),
    "kot_solve_pure_eg": (C.c_int, [C.c_void_p, C.POINTER(SolverCfgC), dptr, dptr, C.POINTER(IterRecordC),
                                    C.c_int, C.POINTER(ReportC)]),
    "kot_iterate": (C.c_int, [C.c_void_p, C.POINTER(SolverCfgC), dptr, dptr, dptr, dptr, C.c_double, C.c_int,
                              dptr, dptr, dptr, dptr, dptr, C.POINTER(IterRecordC)]),
    "kot_session_begin": (C.c_int, [C.c_void_p, C.POINTER(SolverCfgC), C.POINTER(C.c_void_p)]),
    "kot_session_step": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(IterRecordC), iptr]),
    "kot_session_result": (C.c_int, [C.c_void_p, dptr, dptr, C.POINTER(ReportC)]),
    "kot_session_end": (None, [C.c_void_p]),
    "kot_session_state": (C.c_int, [C.c_void_p, dptr, dptr, dptr, dptr, dptr]),
    "kot_problem_stream": (C.c_void_p, [C.c_void_p]),
    "kot_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "kot_problem_shard": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int, C.c_int]),
    "kot_problem_shard_host": (C.c_int, [C.c_void_p, CommFn, C.c_void_p, C.c_int, C.c_int]),
    "kot_problem_shard_info": (C.c_int, [C.c_void_p, iptr, iptr, iptr, iptr]),
    "kot_profile_enable": (C.c_int, [C.c_int]),
    "kot_profile_read": (C.c_int, [C.POINTER(ProfEntryC), C.c_int]),
    "kot_debug_eig_stages": (C.c_int, [C.c_int]),
    "kot_debug_cg_batch": (C.c_int, [C.c_int]),
    "kot_debug_eg_parallel": (C.c_int, [C.c_int]),
    "kot_debug_gemm_tma": (C.c_int, [C.c_int]),
    "kot_set_panel_grid_cap": (C.c_int, [C.c_int]),
    "kot_reserve": (C.c_int, [C.c_int, C.c_ulonglong]),
    "kot_debug_sytrd_timing": (C.c_int, [C.c_int, C.POINTER(C.c_ulonglong)]),
    "kot_debug_tail_timing": (C.c_int, [C.c_int, C.POINTER(C.c_ulonglong)]),
    "kot_debug_mid_timing": (C.c_int, [C.c_int, C.POINTER(C.c_ulonglong)]),
    "kot_debug_trd_mid": (C.c_int, [C.c_int, C.c_int]),
    "kot_debug_trd_mid_head": (C.c_int, [C.c_int]),
    "kot_debug_mid_trace": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_longlong)]),
    "kot_debug_mid_capacity": (C.c_int, [C.c_int, C.c_long]),
    "kot_debug_gate_selftest": (C.c_int, [C.c_int, C.c_int]),
    "kot_gram": (C.c_int, [dptr, C.c_int, C.c_int, C.c_double, C.c_int, dptr]),
    "kot_cholesky_psd": (C.c_int, [dptr, C.c_int, C.c_int, dptr, dptr]),
    "kot_sym_eig": (C.c_int, [dptr, C.c_int, C.c_int, dptr, dptr, iptr]),
    "kot_proj_psd": (C.c_int, [dptr, C.c_int, C.c_int, dptr]),
    "kot_spectral_apply": (C.c_int, [dptr, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, dptr, dptr]),
    "kot_phi_forward": (C.c_int, [C.c_void_p, dptr, dptr]),
    "kot_phi_adjoint": (C.c_int, [C.c_void_p, dptr, dptr]),
    "kot_residual_parts": (C.c_int, [C.c_void_p, dptr, dptr, dptr, dptr, dptr, iptr, dptr, dptr]),
    "kot_objective_grad": (C.c_int, [C.c_void_p, dptr, C.c_int, dptr]),
    "kot_constraint_matrix": (C.c_int, [C.c_void_p, dptr, dptr]),
    "kot_gram_rect": (C.c_int, [dptr, C.c_int, dptr, C.c_int, C.c_int, C.c_double, C.c_int, dptr]),
    "kot_mean_embedding": (C.c_int, [dptr, C.c_int, dptr, C.c_int, C.c_int, C.c_double, C.c_int, dptr]),
    "kot_sobol_points": (C.c_int, [C.POINTER(C.c_ulonglong), C.c_int, C.c_int, C.c_long, C.c_int, dptr, dptr,
                                   C.c_int, dptr]),
    "kot_embedding_norm_sq": (C.c_int, [dptr, C.c_int, C.c_int, C.c_double, C.c_int, dptr]),
    "kot_spectral_apply_decomp": (C.c_int, [dptr, dptr, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                            dptr, dptr]),
    "kot_apply_jacobian": (C.c_int, [C.c_void_p, dptr, dptr, C.c_int, C.c_double, dptr, dptr, dptr, dptr]),
    "kot_cg_solve": (C.c_int, [MatvecFn, C.c_void_p, dptr, C.c_int, C.c_double, C.c_int, C.c_int, dptr, iptr,
                               dptr]),
    "kot_cg_solve_middle": (C.c_int, [C.c_void_p, dptr, dptr, C.c_int, C.c_double, dptr, C.c_double, C.c_int,
                                      dptr, iptr, dptr]),
    "kot_middle_operator_decomp": (C.c_int, [C.c_void_p, dptr, dptr, C.c_int, C.c_double, dptr, dptr]),
    "kot_newton_direction_decomp": (C.c_int, [C.c_void_p, C.POINTER(SolverCfgC), dptr, dptr, dptr, dptr, C.c_int,
                                              C.c_double, dptr, dptr, iptr, iptr, dptr, dptr]),
    "kot_middle_operator": (C.c_int, [C.c_void_p, dptr, dptr, C.c_double, dptr, C.c_int, dptr, dptr]),
    "kot_newton_direction": (C.c_int, [C.c_void_p, C.POINTER(SolverCfgC), dptr, dptr, C.c_double, dptr, dptr,
                                       iptr, iptr, dptr, dptr]),
    "kot_eg_step": (C.c_int, [C.c_void_p, dptr, dptr, C.c_double, dptr, dptr]),
    "kot_objective": (C.c_int, [C.c_void_p, dptr, dptr]),
    "kot_evaluate_map": (C.c_int, [dptr, C.c_int, dptr, dptr, C.c_int, dptr, C.c_int, C.c_int, C.c_double,
                                   C.c_double, C.c_int, dptr, dptr]),
    "kot_ot_estimate": (C.c_int, [C.c_void_p, dptr, dptr]),
}

_lib = None


class LibraryMissing(ImportError):
    pass


def lib():
    """Load libkotgpu.so (built in-tree); raise loudly if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(
                f"{LIB_PATH} not found: build the CUDA library first "
                "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGS)


# ---------------------------------------------------------------- errors

class EigenSolveError(RuntimeError):
    """linalg.py:17-18."""


class IndefiniteKernelError(RuntimeError):
    """linalg.py:21-22."""


class SolverNumericsError(RuntimeError):
    """solver.py:28-33: carries the trace up to the failure."""

    def __init__(self, message, trace):
        super().__init__(message)
        self.trace = trace


class CudaError(RuntimeError):
    pass


class CallbackError(RuntimeError):
    """Status 8: the on_iteration callback failed (the shim re-raises the observer's own exception)."""


def check(status: int, trace=None):
    if status == 0:
        return
    msg = lib().kot_last_error().decode(errors="replace")
    if status == 1:
        raise ValueError(msg)
    if status == 2:
        raise IndefiniteKernelError(msg)
    if status == 3:
        raise EigenSolveError(msg)
    if status == 4:
        raise SolverNumericsError(msg, trace if trace is not None else [])
    if status == 5:
        raise FloatingPointError(msg)
    if status == 7:
        raise AssertionError(msg)
    if status == 8:
        raise CallbackError(msg)
    raise CudaError(msg)


# --------------------------------------------------------------- helpers

def f64(a, shape=None) -> np.ndarray:
    out = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if shape is not None and out.shape != tuple(shape):
        raise ValueError(f"expected shape {tuple(shape)}, got {out.shape}")
    return out


def ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(dptr)


def default_device() -> int:
    return int(os.environ.get("KOT_DEVICE", os.environ.get("LOCAL_RANK", "0")))


def reserve_device_memory(nbytes: int, device: int | None = None) -> None:
    """Process set-up of a long-running service: grow the library's device memory pool by ``nbytes``
    once (kot_reserve).  The first solve of a process otherwise pays the driver's mapping of the pool."""
    check(lib().kot_reserve(default_device() if device is None else device, int(nbytes)))


def launch_count() -> int:
    return int(lib().kot_launch_count())


def profile_enable(on: bool = True, mode: int = 1) -> None:
    """mode 1: every library scope; mode 2: only the roofline scopes (sytrd panels, Q2, 1/16 of the
    GEMM launches) — cheap enough to leave on inside a timed region."""
    lib().kot_profile_enable(mode if on else 0)


def profile_read() -> dict:
    buf = (ProfEntryC * 64)()
    n = lib().kot_profile_read(buf, 64)
    return {buf[i].name.decode(): dict(calls=int(buf[i].calls), ms=float(buf[i].ms), flops=float(buf[i].flops),
                                        bytes=float(buf[i].bytes))
            for i in range(n)}
