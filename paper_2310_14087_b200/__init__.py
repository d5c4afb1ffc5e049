"""B200-native semismooth-Newton solver for kernel-based optimal transport.

Drop-in for the reference package ``kot`` (arXiv 2310.14087): the same
public names (``pkg/src/kot/__init__.py:9-34``), backed by hand-written
sm_100a FP64 kernels in ``libkotgpu.so`` (C ABI: ``include/kotgpu.h``).
"""

from paper_2310_14087_b200.eg import EgConfig
from paper_2310_14087_b200.kernels import KernelSpec, SampleSet
from paper_2310_14087_b200.newton import NewtonConfig
from paper_2310_14087_b200.problem import (FillingPoints, IteratePair, ProblemData, assemble, build_kernel_specs,
                                           objective, ot_estimate)
from paper_2310_14087_b200.solver import SolverConfig, SolverReport, solve, solve_pure_eg
from paper_2310_14087_b200.datagen import MixtureSpec, sample_mixture, sobol_points
from paper_2310_14087_b200._lib import reserve_device_memory  # extension: pool set-up of a service process

__version__ = "0.1.0"

__all__ = [
    "KernelSpec", "SampleSet", "FillingPoints", "IteratePair", "ProblemData", "assemble", "build_kernel_specs",
    "SolverConfig", "SolverReport", "solve", "solve_pure_eg", "NewtonConfig", "EgConfig", "objective",
    "ot_estimate", "MixtureSpec", "sample_mixture", "sobol_points", "reserve_device_memory",
]
