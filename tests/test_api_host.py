"""Host-side pieces of the public surface (CPU only): datagen against the reference's golden draws,
the oracle pinned to the reference's outputs for the API fixtures (tests/golden/api.npz), and the
psdcone dataclass views and validation that need no GPU."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import kot_port as O


@pytest.fixture(scope="module")
def api():
    return dict(np.load(os.path.join(GOLDEN, "api.npz")))


def test_datagen_matches_reference_draws(api):
    """Mixture draws (host: the reference's NumPy streams); the Sobol half runs on the GPU
    (test_gpu_api.py::test_sobol_points_on_device)."""
    import paper_2310_14087_b200 as K
    from paper_2310_14087_b200 import datagen as D
    np.testing.assert_array_equal(K.sample_mixture(D.default_mixture(3, 4, 7), 50).points, api["mix_points"])
    v, bits = D._direction_numbers(5)  # the device kernel's table: XOR rule reproduces the reference
    for i, row in enumerate(api["sobol_nat"]):
        idx, x = i + 4, np.zeros(5, dtype=np.uint64)
        for b in range(bits):
            if (idx >> b) & 1:
                x ^= v[:, b]
        np.testing.assert_array_equal(x.astype(float) / 2.0 ** bits, row)


def test_datagen_validation_mirrors_reference():
    from paper_2310_14087_b200 import datagen as D
    with pytest.raises(ValueError):
        D.MixtureSpec(2, (D.MixtureComponent(0.5, (0.0, 0.0), 0.1),), 0)  # weights do not sum to 1
    with pytest.raises(ValueError):
        D.sobol_points(5, 10)  # odd dimension
    with pytest.raises(ValueError):
        D.sobol_natural(65, 0, 4)
    with pytest.raises(ValueError):
        D.sample_mixture(D.default_mixture(2, 2, 0), 0)


def test_oracle_kernels_and_bandwidths(api, cfg1):
    a, b, bw = api["k_a"], api["k_b"], float(api["k_bw"])
    np.testing.assert_allclose(O.gaussian_gram(bw, a, b), api["k_rect"], rtol=1e-15, atol=0)
    np.testing.assert_allclose(O.gaussian_gram(bw, a), api["k_square"], rtol=1e-15, atol=0)
    np.testing.assert_allclose(O.mean_embedding(bw, a, b), api["k_mean"], rtol=1e-15)
    assert O.embedding_norm_sq(bw, a) == pytest.approx(float(api["k_norm"]), rel=1e-15)
    pd, _ = O.assemble(cfg1["xs"], cfg1["ys"], cfg1["xt"], cfg1["yt"], float(cfg1["l1"]), float(cfg1["l2"]),
                       0.25, 0.4, 0.6)
    np.testing.assert_allclose(pd.q, api["bw3_q"], rtol=1e-15, atol=1e-15)
    np.testing.assert_allclose(pd.z, api["bw3_z"], rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(pd.r, api["bw3_r"], rtol=1e-13, atol=1e-14)
    assert pd.q_sq == pytest.approx(float(api["bw3_q_sq"]), rel=1e-15)


def test_oracle_jacobian_criterion_cg_and_pure_eg(api, cfg1):
    pd = O.Problem(q=cfg1["q"], z=cfg1["z"], q_sq=float(cfg1["q_sq"]), r=cfg1["r"], l1=float(cfg1["l1"]),
                   l2=float(cfg1["l2"]), embed=cfg1["embed"])
    r, dc = O.residual_parts(pd, O.Pair(cfg1["op_g"], cfg1["op_x"]))
    ctx = O.newton_context(dc, r.norm(), float(cfg1["op_theta"]))
    dw = O.Pair(cfg1["op_dir_dg"], cfg1["op_dir_dx"])
    jd = O.apply_jacobian(pd, dc, ctx.eta, ctx.mu, dw)
    np.testing.assert_allclose(jd.g, api["jac_top"], rtol=0, atol=1e-11 * np.abs(api["jac_top"]).max())
    np.testing.assert_allclose(jd.x, api["jac_bottom"], rtol=0, atol=1e-11 * np.abs(api["jac_bottom"]).max())
    assert (jd + r).norm() == pytest.approx(float(api["crit_lhs"]), rel=1e-10)
    assert float(api["crit_lhs"]) == pytest.approx(float(cfg1["op_dir_lhs"]), rel=1e-12)
    np.testing.assert_allclose(O.objective_grad(pd, cfg1["op_g"]), api["grad"], rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(O.objective_grad_dir(pd, cfg1["op_v"]), api["grad_dir"], rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(O.constraint_matrix(pd, cfg1["op_g"]), api["cmat"], rtol=1e-13, atol=1e-13)
    x, it, res = O.cg(lambda v: api["cg_a"] @ v, api["cg_b"], 1e-10, 200)
    assert it == int(api["cg_iters"])
    np.testing.assert_allclose(x, api["cg_x"], rtol=1e-12)
    x, it, _ = O.cg(O.middle_operator(pd, ctx.op, ctx.mu), cfg1["op_v"], 1e-12, 500)
    assert abs(it - int(api["cgm_iters"])) <= 2
    np.testing.assert_allclose(x, api["cgm_x"], rtol=0, atol=1e-9 * np.abs(api["cgm_x"]).max())
    rep = O.solve_pure_eg(pd, O.SolverCfg(eg_stepsize=float(cfg1["eg_stepsize"]), residual_tol=1e-12, max_iter=30))
    np.testing.assert_allclose([t.res_accepted for t in rep.trace], api["peg_res"], rtol=1e-10)
    np.testing.assert_allclose(rep.gamma, api["peg_gamma"], rtol=0, atol=1e-10 * np.abs(api["peg_gamma"]).max())


def test_psdcone_dataclasses_and_path_rule(small):
    """proj_jacobian_coeffs / make_eliminator: the host views equal the oracle's coefficients, the path
    rule is the reference's (POS_BLOCK iff k ≤ ℓ − k), μ ≤ 0 raises (psdcone.py:67-110)."""
    from paper_2310_14087_b200 import psdcone as C
    from paper_2310_14087_b200.linalg import SpectralDecomp
    for n_pos in (0, 1, 3, 5, 6):
        z = small[f"sign{n_pos}_z"]
        dco = O.sym_eig(z)
        dc = SpectralDecomp(eigvecs=dco.vecs, eigvals=dco.vals, pos_idx=np.arange(dco.k),
                            nonpos_idx=np.arange(dco.k, 6))
        coeffs = C.proj_jacobian_coeffs(dc)
        np.testing.assert_allclose(coeffs.cross, O.cross_coeffs(dco), rtol=1e-15)
        op = C.make_eliminator(coeffs, 0.7)
        assert op.path == (C.POS_BLOCK if n_pos <= 6 - n_pos else C.NONPOS_COMPLEMENT)
        np.testing.assert_allclose(op.cross_scaled, O.eliminator(dco, O.cross_coeffs(dco), 0.7).xi, rtol=1e-15)
        w = C.eliminator_coeff_matrix(op)
        assert w.shape == (6, 6) and np.allclose(w[:n_pos, :n_pos], 1 / 0.7)
        with pytest.raises(ValueError):
            C.make_eliminator(coeffs, 0.0)


def test_problem_data_cache_follows_field_updates():
    """dataclasses.replace never carries the device copy; reassigning a data field drops it."""
    import dataclasses

    from paper_2310_14087_b200.problem import ProblemData
    pd = ProblemData(q_mat=np.eye(2), z=np.ones(2), q_sq=1.0, chol_upper=np.eye(2), lambda1=1.0, lambda2=1.0)
    object.__setattr__(pd, "_dev", "device copy")
    object.__setattr__(pd, "_kmat", "K")
    assert dataclasses.replace(pd, lambda1=2.0)._dev is None
    pd.lambda1 = 3.0
    assert pd._dev is None and pd._kmat == "K"
    object.__setattr__(pd, "_dev", "device copy")
    pd.chol_upper = np.eye(2)
    assert pd._dev is None and pd._kmat is None
