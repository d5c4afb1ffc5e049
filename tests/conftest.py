import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI library)")
    config.addinivalue_line("markers", "slow: long-running oracle case")


@pytest.fixture(scope="session")
def cfg1():
    return dict(np.load(os.path.join(GOLDEN, "cfg1.npz")))


@pytest.fixture(scope="session")
def small():
    return dict(np.load(os.path.join(GOLDEN, "small.npz")))


def random_symmetric(rng, n, scale=1.0):
    """Same draws as the reference fixture pkg/tests/conftest.py:50-52."""
    a = scale * rng.standard_normal((n, n))
    return 0.5 * (a + a.T)


def symmetric_with_signs(rng, n, n_pos, gap=0.1):
    """Same draws as the reference fixture pkg/tests/conftest.py:55-63."""
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    pos = 0.5 + gap * np.arange(n_pos) + rng.uniform(0, 0.05, size=n_pos)
    neg = -0.5 - gap * np.arange(n - n_pos) - rng.uniform(0, 0.05, size=n - n_pos)
    return (q * np.concatenate([pos, neg])) @ q.T


def random_problem_arrays(seed, n=5, q_reg=0.5, feat_reg=0.5, z_scale=2.0, lambda1=0.5, lambda2=0.4):
    """Same draws as pkg/tests/conftest.py:9-31; returns plain arrays."""
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, n))
    q = a @ a.T / n + q_reg * np.eye(n)
    b = rng.standard_normal((n, n))
    r_up = np.linalg.cholesky(b @ b.T / n + feat_reg * np.eye(n)).T
    z = z_scale * rng.standard_normal(n)
    q_sq = float(rng.uniform(0.0, 1.0))
    return dict(q=q, z=z, q_sq=q_sq, r=r_up, l1=lambda1, l2=lambda2)
