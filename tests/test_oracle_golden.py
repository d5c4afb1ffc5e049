"""Pin the CPU oracle (oracle/kot_port.py) to the unmodified reference.

Golden vectors come from tests/golden/make_golden.py (reference `kot` imported
from /root/reference in the build container).  CPU only.
"""

import numpy as np
import pytest

from oracle import kot_port as O
from paper_2310_14087_b200 import configs


def _pd(d, p=""):
    return O.Problem(q=d[p + "q"], z=d[p + "z"], q_sq=float(d[p + "q_sq"]), r=d[p + "r"],
                     l1=float(d[p + "l1"]), l2=float(d[p + "l2"]), embed=d.get(p + "embed"))


def test_cfg1_workload_reproduces_fixture_inputs(cfg1):
    wl = configs.config1()
    for k in ("xs", "ys", "xt", "yt"):
        np.testing.assert_array_equal(getattr(wl, k), cfg1[k])


def test_assemble_matches_reference(cfg1):
    pd, kmat = O.assemble(cfg1["xs"], cfg1["ys"], cfg1["xt"], cfg1["yt"], float(cfg1["l1"]),
                          float(cfg1["l2"]), float(cfg1["bw_sq"]))
    np.testing.assert_allclose(pd.q, cfg1["q"], rtol=1e-15, atol=1e-15)
    np.testing.assert_allclose(pd.z, cfg1["z"], rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(pd.r, cfg1["r"], rtol=1e-14, atol=1e-14)
    np.testing.assert_allclose(pd.embed, cfg1["embed"], rtol=1e-14)
    assert pd.q_sq == pytest.approx(float(cfg1["q_sq"]), rel=1e-15)
    assert pd.jitter == float(cfg1["jitter"]) == 0.0
    np.testing.assert_allclose(kmat, cfg1["kmat"], rtol=1e-15)
    assert configs.eg_stepsize(pd.q, kmat, pd.l2) == pytest.approx(float(cfg1["eg_stepsize"]), rel=1e-14)


def test_per_op_values(cfg1):
    pd = _pd(cfg1)
    g, x = cfg1["op_g"], cfg1["op_x"]
    np.testing.assert_allclose(O.phi(pd, x), cfg1["op_phi"], rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(O.phi_adj(pd, g), cfg1["op_phi_adj"], rtol=1e-13, atol=1e-13)
    r, dc = O.residual_parts(pd, O.Pair(g, x))
    np.testing.assert_allclose(r.g, cfg1["op_r1"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(r.x, cfg1["op_r2"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(dc.vals, cfg1["op_eigvals"], rtol=1e-12, atol=1e-12)
    assert dc.k == int(cfg1["op_npos"])
    ctx = O.newton_context(dc, r.norm(), float(cfg1["op_theta"]))
    assert ctx.mu == pytest.approx(float(cfg1["op_mu"]), rel=1e-13)
    mid = O.middle_operator(pd, ctx.op, ctx.mu)(cfg1["op_v"])
    np.testing.assert_allclose(mid, cfg1["op_middle"], rtol=1e-10, atol=1e-10 * np.abs(mid).max())
    el = O.apply_eliminator(ctx.op, cfg1["op_s"])
    np.testing.assert_allclose(el, cfg1["op_elim"], rtol=0, atol=1e-10 * np.abs(el).max())
    mz = O.apply_proj_jacobian(dc, ctx.eta, cfg1["op_s"])
    np.testing.assert_allclose(mz, cfg1["op_mz"], rtol=0, atol=1e-10 * np.abs(mz).max())
    assert O.objective(pd, g) == pytest.approx(float(cfg1["op_objective"]), rel=1e-12)
    st = O.newton_direction(pd, r, ctx, O.NewtonCfg())
    assert st.cg_iters == int(cfg1["op_dir_cg"])
    assert st.met == bool(cfg1["op_dir_met"])
    np.testing.assert_allclose(st.dw.g, cfg1["op_dir_dg"], rtol=1e-8, atol=1e-8 * np.abs(st.dw.g).max())
    ve = O.eg_step(pd, O.Pair(g, cfg1["op_eg_in_x"]), float(cfg1["eg_stepsize"]))
    np.testing.assert_allclose(ve.g, cfg1["op_eg_g"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(ve.x, cfg1["op_eg_x"], rtol=0, atol=1e-11 * np.abs(ve.x).max())


def test_paper_profile_trace_40_iterations(cfg1):
    pd = _pd(cfg1)
    cfg = O.SolverCfg(newton=O.NewtonCfg(), eg_stepsize=float(cfg1["eg_stepsize"]),
                      residual_tol=1e-12, max_iter=40)
    rep = O.solve(pd, cfg)
    res = np.array([t.res_accepted for t in rep.trace])
    # same BLAS here as at generation time: the traces agree to rounding (chaotic
    # beyond ~1e-6 only under perturbation)
    np.testing.assert_allclose(res, cfg1["paper_res_accepted"], rtol=1e-6)
    assert [t.cg_iters for t in rep.trace] == list(cfg1["paper_cg_iters"])
    assert [t.accepted == "ssn" for t in rep.trace] == list(cfg1["paper_accepted_ssn"])


@pytest.mark.slow
def test_tight_profile_end_state(cfg1):
    pd = _pd(cfg1)
    cfg = O.SolverCfg(newton=O.NewtonCfg(alpha1=1e-8, alpha2=1e-4, cg_max=500),
                      eg_stepsize=float(cfg1["eg_stepsize"]), residual_tol=1e-10, max_iter=1000)
    rep = O.solve(pd, cfg)
    assert abs(len(rep.trace) - int(cfg1["tight_iters"])) <= 2
    np.testing.assert_allclose(rep.gamma, cfg1["tight_gamma"], rtol=1e-6, atol=1e-9)
    assert O.objective(pd, rep.gamma) == pytest.approx(float(cfg1["tight_objective"]), rel=1e-8)
    assert rep.ot == pytest.approx(float(cfg1["tight_ot"]), rel=1e-8)


def test_evaluate_map(cfg1):
    pd = _pd(cfg1)
    pd.xt, pd.bw_sq = cfg1["xt"], float(cfg1["bw_sq"])
    u, t = O.evaluate_map(pd, cfg1["xs"], cfg1["tight_gamma"], cfg1["map_queries"])
    np.testing.assert_allclose(u, cfg1["map_u"], rtol=1e-12)
    np.testing.assert_allclose(t, cfg1["map_t"], rtol=1e-12)


@pytest.mark.parametrize("name", ["interior", "active"])
def test_scalar_kkt_fixtures(small, name):
    z = 1.0 if name == "interior" else -4.0
    pd = O.Problem(q=[[2.0]], z=[z], q_sq=0.0, r=[[1.0]], l1=1.0, l2=0.5)
    rep = O.solve(pd, O.SolverCfg(residual_tol=1e-12, max_iter=100))
    assert len(rep.trace) == int(small[f"scalar_{name}_iters"])
    np.testing.assert_allclose(rep.gamma, small[f"scalar_{name}_gamma"], rtol=1e-14)
    np.testing.assert_allclose(rep.x, small[f"scalar_{name}_x"], rtol=1e-14, atol=1e-15)
    expect_g, expect_x = (0.5, 0.0) if name == "interior" else (-1.0, 2.0)
    assert rep.gamma[0] == pytest.approx(expect_g, abs=1e-10)
    assert rep.x[0, 0] == pytest.approx(expect_x, abs=1e-10)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_random_problem_solves(small, seed):
    p = f"rand{seed}_"
    pd = _pd(small, p)
    rep = O.solve(pd, O.SolverCfg(residual_tol=1e-10, max_iter=200))
    assert len(rep.trace) == int(small[p + "iters"])
    np.testing.assert_allclose(rep.gamma, small[p + "gamma"], rtol=1e-9, atol=1e-10)


@pytest.mark.parametrize("n_pos", [0, 1, 3, 5, 6])
def test_sign_fixtures(small, n_pos):
    p = f"sign{n_pos}_"
    dc = O.sym_eig(small[p + "z"])
    np.testing.assert_allclose(dc.vals, small[p + "eigvals"], atol=1e-14)
    np.testing.assert_allclose(O.proj(dc), small[p + "proj"], atol=1e-14)
    eta = O.cross_coeffs(dc)
    np.testing.assert_allclose(O.apply_proj_jacobian(dc, eta, small[p + "s"]), small[p + "mz"], atol=1e-13)
    for mu in (0.03, 1.0, 17.0):
        op = O.eliminator(dc, eta, mu)
        np.testing.assert_allclose(O.apply_eliminator(op, small[p + "s"]), small[f"{p}elim_{mu}"],
                                   atol=1e-12 * max(1.0, np.abs(small[f"{p}elim_{mu}"]).max()))


def test_cholesky_rank_deficient_fixture(small):
    r, jit = O.cholesky_psd(small["chol_rankdef_in"])
    assert jit == float(small["chol_rankdef_jitter"]) > 0
    np.testing.assert_allclose(r, small["chol_rankdef_r"], rtol=1e-12, atol=1e-12)
