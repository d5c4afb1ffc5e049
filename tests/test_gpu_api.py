"""GPU parity for the rest of the drop-in surface (through the C ABI) against reference outputs
(tests/golden/api.npz, tests/golden/cfg1.npz): rectangular Grams, mean embeddings, embedding norms,
distinct-bandwidth assembly, objective gradients, the psdcone decomposition API, apply_jacobian and
the Eq.(9) criterion values, cg_solve (host callable and device middle operator), the reference-
signature Newton direction, solve_pure_eg, and the observer / cache semantics of ADVICE r1."""

import dataclasses
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import kot_port as O

pytestmark = pytest.mark.gpu

K = pytest.importorskip("paper_2310_14087_b200")
from paper_2310_14087_b200 import kernels as GK  # noqa: E402
from paper_2310_14087_b200 import linalg as GL  # noqa: E402
from paper_2310_14087_b200 import newton as GN  # noqa: E402
from paper_2310_14087_b200 import problem as GP  # noqa: E402
from paper_2310_14087_b200 import psdcone as GC  # noqa: E402
from paper_2310_14087_b200.eg import EgConfig  # noqa: E402


@pytest.fixture(scope="module")
def api():
    return dict(np.load(os.path.join(GOLDEN, "api.npz")))


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def gpu_pd(d, p=""):
    return GP.ProblemData(q_mat=d[p + "q"], z=d[p + "z"], q_sq=float(d[p + "q_sq"]), chol_upper=d[p + "r"],
                          lambda1=float(d[p + "l1"]), lambda2=float(d[p + "l2"]), embed_sum=d.get(p + "embed"))


def test_kernels_module(api):
    spec = K.KernelSpec(float(api["k_bw"]), 3)
    a, b = api["k_a"], api["k_b"]
    assert rel(GK.gram_matrix(spec, a, b), api["k_rect"]) <= 1e-15
    sq = GK.gram_matrix(spec, a)
    assert rel(sq, api["k_square"]) <= 1e-15 and np.array_equal(sq, sq.T)
    assert rel(GK.mean_embedding(spec, K.SampleSet(a), b), api["k_mean"]) <= 1e-15
    assert GK.mean_embedding_at(spec, K.SampleSet(a), b[3]) == pytest.approx(float(api["k_mean_at"]), rel=1e-15)
    assert GK.embedding_norm_sq(spec, K.SampleSet(a)) == pytest.approx(float(api["k_norm"]), rel=1e-14)
    assert GK.kernel_eval(spec, a[0], b[0]) == pytest.approx(float(api["k_eval"]), rel=1e-15)
    with pytest.raises(ValueError):
        GK.gram_matrix(spec, a, b[:, :2])
    with pytest.raises(ValueError):
        GK.mean_embedding(spec, K.SampleSet(np.zeros((0, 3))), b)


def test_assemble_distinct_bandwidths(api, cfg1):
    sx, sy, sxy = K.KernelSpec(0.25, 2), K.KernelSpec(0.4, 2), K.KernelSpec(0.6, 4)
    pd = K.assemble(K.SampleSet(cfg1["xs"]), K.SampleSet(cfg1["ys"]), K.FillingPoints(cfg1["xt"], cfg1["yt"]),
                    float(cfg1["l1"]), float(cfg1["l2"]), sx, sy, sxy)
    assert rel(pd.q_mat, api["bw3_q"]) <= 1e-15
    assert rel(pd.z, api["bw3_z"]) <= 1e-14
    assert rel(pd.embed_sum, api["bw3_embed"]) <= 1e-14
    assert pd.q_sq == pytest.approx(float(api["bw3_q_sq"]), rel=1e-14)
    assert rel(pd.chol_upper, api["bw3_r"]) <= 1e-13


def test_objective_gradients_and_constraint_matrix(api, cfg1):
    pd = gpu_pd(cfg1)
    assert rel(GP.objective_grad(pd, cfg1["op_g"]), api["grad"]) <= 1e-12  # (Qγ − z): cancellation
    assert rel(GP.objective_grad_dir(pd, cfg1["op_v"]), api["grad_dir"]) <= 1e-13
    c = GP.constraint_matrix(pd, cfg1["op_g"])
    assert rel(c, api["cmat"]) <= 1e-13 and np.array_equal(c, c.T)


def _ctx(pd, cfg1):
    r, dc = GP.residual_parts(pd, GP.IteratePair(cfg1["op_g"], cfg1["op_x"]))
    return r, dc, GN.newton_context(dc, r.norm(), float(cfg1["op_theta"]))


def test_psdcone_decomposition_api(cfg1):
    """proj_from_decomp / apply_eliminator(make_eliminator(...)) / apply_proj_jacobian(coeffs, s) with the
    reference signatures, at a decomposition computed on the device (residual_parts returns it)."""
    pd = gpu_pd(cfg1)
    r, dc, ctx = _ctx(pd, cfg1)
    assert dc.n_pos == int(cfg1["op_npos"])
    p = dc.eigvecs
    assert np.linalg.norm(p.T @ p - np.eye(pd.n)) <= 1e-12 * pd.n
    assert ctx.mu == pytest.approx(float(cfg1["op_mu"]), rel=1e-12)
    assert rel(GC.proj_from_decomp(dc), cfg1["op_proj"]) <= 1e-12
    assert rel(GC.apply_eliminator(ctx.eliminator, cfg1["op_s"]), cfg1["op_elim"]) <= 1e-11
    for path in (GC.POS_BLOCK, GC.NONPOS_COMPLEMENT):  # both routes give the same operator
        op = dataclasses.replace(ctx.eliminator, path=path)
        assert rel(GC.apply_eliminator(op, cfg1["op_s"]), cfg1["op_elim"]) <= 1e-11
    assert rel(GC.apply_proj_jacobian(ctx.coeffs, cfg1["op_s"]), cfg1["op_mz"]) <= 1e-11


def test_apply_jacobian_and_criterion_values(api, cfg1):
    """Row a21: (J+μI)dw (problem.py:222-236) and the Eq.(9) values lhs = ‖(J+μI)dw + r‖,
    rhs = τ·min(1, κ‖r‖‖dw‖) (newton.py:131-141) against the reference, for the reference's dw."""
    pd = gpu_pd(cfg1)
    r, dc, ctx = _ctx(pd, cfg1)
    dw = GP.IteratePair(cfg1["op_dir_dg"], cfg1["op_dir_dx"])
    jd = GP.apply_jacobian(pd, ctx.coeffs, ctx.mu, dw)
    assert rel(jd.gamma, api["jac_top"]) <= 1e-11
    assert rel(jd.x_mat, api["jac_bottom"]) <= 1e-11
    lhs = (jd + r).norm()
    assert lhs == pytest.approx(float(api["crit_lhs"]), rel=1e-9)
    cfg = GN.NewtonConfig()
    assert cfg.tau * min(1.0, cfg.kappa * r.norm() * dw.norm()) == pytest.approx(float(api["crit_rhs"]), rel=1e-12)


def test_newton_direction_reference_signature(api, cfg1):
    """newton_direction(pd, r, ctx, cfg) with converged CG: direction ≤1e-8, crit_rhs ≤1e-8, and the
    reported lhs is the norm of (J+μI)dw + r recomputed from the returned dw."""
    pd = gpu_pd(cfg1)
    r, dc, ctx = _ctx(pd, cfg1)
    cfg = GN.NewtonConfig(cg_tol=1e-13, cg_max=3000, cg_restarts=0)
    st = GN.newton_direction(pd, r, ctx, cfg)
    assert rel(st.dw.gamma, api["dirc_dg"]) <= 1e-8
    assert rel(st.dw.x_mat, api["dirc_dx"]) <= 1e-8
    assert st.crit_rhs == pytest.approx(float(api["dirc_rhs"]), rel=1e-8)
    lhs = (GP.apply_jacobian(pd, ctx.coeffs, ctx.mu, st.dw) + r).norm()
    assert st.crit_lhs == pytest.approx(lhs, rel=1e-6, abs=1e-12 * r.norm())
    # paper profile: lhs is the capped CG's residual, pinned to 100× the oracle's own 1-ulp spread
    st = GN.newton_direction(pd, r, ctx, GN.NewtonConfig())
    assert st.cg_iters == int(cfg1["op_dir_cg"]) and st.criterion_met == bool(cfg1["op_dir_met"])
    spread = 0.0
    for seed in (1, 2):
        rng = np.random.default_rng(seed)
        rp = cfg1["r"] * (1.0 + rng.choice([-1.0, 1.0], cfg1["r"].shape) * 2.2e-16)
        po = O.Problem(q=cfg1["q"], z=cfg1["z"], q_sq=float(cfg1["q_sq"]), r=rp, l1=float(cfg1["l1"]),
                       l2=float(cfg1["l2"]))
        ro, dco = O.residual_parts(po, O.Pair(cfg1["op_g"], cfg1["op_x"]))
        so = O.newton_direction(po, ro, O.newton_context(dco, ro.norm(), float(cfg1["op_theta"])), O.NewtonCfg())
        spread = max(spread, abs(so.lhs / float(cfg1["op_dir_lhs"]) - 1.0))
    assert st.crit_lhs == pytest.approx(float(cfg1["op_dir_lhs"]), rel=max(1e-8, 100 * spread))


def test_cg_solve_host_callable_and_device_operator(api, cfg1):
    """linalg.cg_solve (linalg.py:117-162): an arbitrary callable (CG algebra on the device, matvec on the
    host) and the device middle operator (newton.middle_operator → fused device CG)."""
    a = api["cg_a"]
    x, it, res = GL.cg_solve(lambda v: a @ v, api["cg_b"], 1e-10, 200)
    # the stopping test sits on a knife edge at the last step (device reductions vs NumPy's): ±1 step
    assert abs(it - int(api["cg_iters"])) <= 1
    assert rel(x, api["cg_x"]) <= 1e-9
    assert res <= 1e-10 * np.linalg.norm(api["cg_b"])
    pd = gpu_pd(cfg1)
    _, _, ctx = _ctx(pd, cfg1)
    op = GN.middle_operator(pd, ctx.eliminator, ctx.mu)
    mv = op(cfg1["op_v"])
    assert rel(mv, cfg1["op_middle"]) <= 1e-11
    x, it, res = GL.cg_solve(op, cfg1["op_v"], 1e-12, 500)
    assert abs(it - int(api["cgm_iters"])) <= 2
    assert rel(x, api["cgm_x"]) <= 1e-9

    def boom(v):
        raise KeyError("observer")
    with pytest.raises(KeyError):
        GL.cg_solve(boom, api["cg_b"], 1e-10, 10)
    with pytest.raises(ValueError):
        GL.cg_solve(lambda v: a @ v, api["cg_b"], 1e-10, 0)
    with pytest.raises(FloatingPointError):
        GL.cg_solve(lambda v: np.full_like(v, np.nan), api["cg_b"], 1e-10, 10)


def test_solve_pure_eg_matches_reference(api, cfg1):
    """Row f2: solve_pure_eg (solver.py:236-289) — no CG, so the trajectory is determined to eigensolver
    accuracy over 30 EG steps."""
    pd = gpu_pd(cfg1)
    rep = K.solve_pure_eg(pd, K.SolverConfig(eg=EgConfig(float(cfg1["eg_stepsize"])), residual_tol=1e-12,
                                             max_iter=30))
    assert rep.iterations == int(api["peg_iters"]) and rep.termination == "max_iter"
    res = np.array([t.res_accepted for t in rep.trace])
    assert np.max(np.abs(res / api["peg_res"] - 1.0)) <= 1e-9
    assert all(t.accepted == "eg" for t in rep.trace)
    assert rel(rep.gamma_hat, api["peg_gamma"]) <= 1e-9
    assert rel(rep.x_hat, api["peg_x"]) <= 1e-9
    assert rep.ot_estimate == pytest.approx(O.ot_estimate(O.Problem(
        q=cfg1["q"], z=cfg1["z"], q_sq=float(cfg1["q_sq"]), r=cfg1["r"], l1=float(cfg1["l1"]), l2=float(cfg1["l2"]),
        embed=cfg1["embed"]), api["peg_gamma"]), rel=1e-9)


def test_observer_exception_ends_the_solve(cfg1):
    """an exception raised by on_iteration propagates out of solve() and stops it
    (reference solver.py:170-181), it is not swallowed by the ctypes trampoline."""
    pd = gpu_pd(cfg1)
    seen = []

    def observer(probe):
        seen.append(probe.iteration)
        if probe.iteration == 2:
            raise RuntimeError("stop here")
    with pytest.raises(RuntimeError, match="stop here"):
        K.solve(pd, K.SolverConfig(eg=EgConfig(float(cfg1["eg_stepsize"])), residual_tol=1e-12, max_iter=10),
                on_iteration=observer)
    assert seen == [0, 1, 2]
    # the problem stays usable
    rep = K.solve(pd, K.SolverConfig(eg=EgConfig(float(cfg1["eg_stepsize"])), residual_tol=1e-12, max_iter=2))
    assert rep.iterations == 2


def test_replaced_problem_data_is_reuploaded(cfg1):
    """dataclasses.replace(pd, lambda1=…) and field reassignment must not reuse the old device
    instance."""
    pd = gpu_pd(cfg1)
    g = cfg1["op_g"]
    o1 = GP.objective(pd, g)
    pd2 = dataclasses.replace(pd, lambda2=2.0 * pd.lambda2)
    po = O.Problem(q=cfg1["q"], z=cfg1["z"], q_sq=float(cfg1["q_sq"]), r=cfg1["r"], l1=float(cfg1["l1"]),
                   l2=2.0 * float(cfg1["l2"]))
    assert GP.objective(pd2, g) == pytest.approx(O.objective(po, g), rel=1e-13)
    pd.lambda2 = 2.0 * pd.lambda2
    assert GP.objective(pd, g) == pytest.approx(O.objective(po, g), rel=1e-13)
    assert o1 != GP.objective(pd, g)


def test_sobol_points_on_device(api):
    """Row f4: natural-order Sobol filling points generated on the GPU equal the reference's
    (datagen.py:77-132: SciPy's Gray-code stream re-indexed), bit for bit."""
    from paper_2310_14087_b200 import datagen as D
    fp = K.sobol_points(6, 37, -1.0, 1.0)
    assert np.array_equal(fp.x_tilde, api["sobol_xt"]) and np.array_equal(fp.y_tilde, api["sobol_yt"])
    assert np.array_equal(D.sobol_natural(5, 3, 20), api["sobol_nat"])
    s = D.SobolStream(5, 3)
    assert np.array_equal(np.vstack([s.take(7), s.take(13)]), api["sobol_nat"])
    with pytest.raises(ValueError):
        K.sobol_points(5, 10)


def test_reserve_device_memory_grows_the_pool_once():
    """kot_reserve: process set-up of a service; a second call of the same size is
    served from the pool, and solves afterwards are unaffected."""
    import time
    import paper_2310_14087_b200 as K2
    K2.reserve_device_memory(256 << 20)
    t0 = time.perf_counter()
    K2.reserve_device_memory(256 << 20)
    assert time.perf_counter() - t0 < 0.5
    with pytest.raises(Exception):
        K2.reserve_device_memory(1 << 50)  # more than the device has: reported, not fatal
    z = np.diag([2.0, -1.0, 0.5])
    assert np.allclose(np.sort(GL.sym_eig(z).eigvals), [-1.0, 0.5, 2.0])
