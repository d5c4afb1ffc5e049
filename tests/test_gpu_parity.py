"""GPU parity: libkotgpu (through the C ABI) vs the CPU oracle and reference golden vectors.

Tolerances follow SURVEY.md §8(c) P1/P2/P3: ~1e-13 relative for Gram/Φ/Φ*,
≤1e-11 for eigen-derived operators, ≤1e-9 for one lock-step replay
iteration, objective ≤1e-8 / potentials ≤1e-6 at tol 1e-10.
"""

import numpy as np
import pytest

from conftest import random_problem_arrays, random_symmetric, symmetric_with_signs
from oracle import kot_port as O

pytestmark = pytest.mark.gpu

K = pytest.importorskip("paper_2310_14087_b200")
from paper_2310_14087_b200 import linalg as GL  # noqa: E402
from paper_2310_14087_b200 import newton as GN  # noqa: E402
from paper_2310_14087_b200 import problem as GP  # noqa: E402
from paper_2310_14087_b200 import psdcone as GC  # noqa: E402
from paper_2310_14087_b200 import solver as GS  # noqa: E402
from paper_2310_14087_b200.eg import EgConfig, eg_step  # noqa: E402


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def gpu_pd(d, p=""):
    return GP.ProblemData(q_mat=d[p + "q"], z=d[p + "z"], q_sq=float(d[p + "q_sq"]), chol_upper=d[p + "r"],
                          lambda1=float(d[p + "l1"]), lambda2=float(d[p + "l2"]), embed_sum=d.get(p + "embed"))


def oracle_pd(d, p=""):
    return O.Problem(q=d[p + "q"], z=d[p + "z"], q_sq=float(d[p + "q_sq"]), r=d[p + "r"], l1=float(d[p + "l1"]),
                     l2=float(d[p + "l2"]), embed=d.get(p + "embed"))


# ------------------------------------------------------------------ eigen

@pytest.mark.parametrize("n", [1, 2, 3, 5, 17, 31, 32, 33, 64, 65, 100, 129, 257, 500])
def test_sym_eig_random(n):
    rng = np.random.default_rng(n)
    z = random_symmetric(rng, n)
    dc = GL.sym_eig(z)
    ref = np.sort(np.linalg.eigvalsh(z))[::-1]
    nz = np.linalg.norm(z)
    assert np.max(np.abs(dc.eigvals - ref)) <= 1e-13 * max(nz, 1.0)
    p = dc.eigvecs
    assert np.linalg.norm(p.T @ p - np.eye(n)) <= 1e-13 * n
    assert np.linalg.norm((p * dc.eigvals) @ p.T - z) <= 1e-13 * max(nz, 1.0) * np.sqrt(n)
    assert dc.n_pos == int(np.count_nonzero(ref > 0))


@pytest.mark.parametrize("n,kind", [(40, "clustered"), (200, "clustered"), (300, "lowrank"), (128, "diag"),
                                    (96, "scaled"), (1000, "signs")])
def test_sym_eig_structured(n, kind):
    rng = np.random.default_rng(7)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    if kind == "clustered":
        vals = np.repeat([3.0, 1e-3, -1e-3, -2.0], n // 4)
        vals = np.concatenate([vals, np.zeros(n - vals.size)])
    elif kind == "lowrank":
        vals = np.zeros(n)
        vals[:5] = [5, 4, 3, 2, 1]
        vals[-3:] = -1e-4
    elif kind == "diag":
        z = np.diag(np.linspace(-1, 1, n))
        vals = None
    elif kind == "scaled":
        vals = np.logspace(-8, 8, n) * np.where(np.arange(n) % 2, 1, -1)
    else:
        z = symmetric_with_signs(rng, n, n // 3)
        vals = None
    if vals is not None:
        z = (q * vals) @ q.T
        z = 0.5 * (z + z.T)
    dc = GL.sym_eig(z)
    ref = np.sort(np.linalg.eigvalsh(z))[::-1]
    nz = np.linalg.norm(z, 2)
    assert np.max(np.abs(dc.eigvals - ref)) <= 1e-12 * nz
    p = dc.eigvecs
    assert np.linalg.norm(p.T @ p - np.eye(n)) <= 1e-12 * n
    assert np.linalg.norm((p * dc.eigvals) @ p.T - z) <= 1e-12 * nz * n


@pytest.mark.parametrize("scale", [1e-8, 1.0, 1e8])
def test_sym_eig_scale_invariant(scale):
    """A nearly diagonal matrix with a few positive eigenvalues (the first EG argument of a config-5
    member has this shape at norm ~1e-8): D&C deflation is relative to the tridiagonal's norm, as in
    dstedc, so the decomposition and the PSD projection are accurate at any scale."""
    n = 600
    rng = np.random.default_rng(11)
    base = np.diag(-1.0 - rng.random(n))
    base[:12, :12] += np.diag(1.2 + rng.random(12))
    e = rng.standard_normal((n, n)) * 1e-6
    z = scale * (base + 0.5 * (e + e.T))
    dc = GL.sym_eig(z)
    nz = np.linalg.norm(z, 2)
    ref = np.sort(np.linalg.eigvalsh(z))[::-1]
    assert np.max(np.abs(dc.eigvals - ref)) <= 1e-13 * nz
    p = dc.eigvecs
    assert np.max(np.abs((p * dc.eigvals) @ p.T - z)) <= 1e-13 * nz
    proj = GC.proj_psd(z)
    assert rel(proj, O.proj_psd(z)) <= 1e-12


def test_sym_eig_kats():
    # test_linalg.py:13-44
    d = GL.sym_eig(np.diag([2.0, -1.0]))
    assert np.allclose(np.abs(d.eigvecs), np.eye(2)) and np.allclose(d.eigvals, [2.0, -1.0])
    assert d.pos_idx.tolist() == [0] and d.nonpos_idx.tolist() == [1]
    d = GL.sym_eig(np.eye(3))
    assert np.allclose(d.eigvals, 1.0) and d.pos_idx.tolist() == [0, 1, 2] and d.nonpos_idx.size == 0
    d = GL.sym_eig(np.diag([0.0, 1.0, -2.0]))
    assert d.eigvals.tolist() == [1.0, 0.0, -2.0]
    assert d.pos_idx.tolist() == [0] and d.nonpos_idx.tolist() == [1, 2]


# ---------------------------------------------------------------- Cholesky

def test_cholesky_kats(small, cfg1):
    f = GL.cholesky_psd(np.eye(2))
    assert np.allclose(f.upper, np.eye(2)) and f.jitter_applied == 0.0
    f = GL.cholesky_psd(np.array([[4.0, 2.0], [2.0, 2.0]]))
    assert np.allclose(f.upper, [[2.0, 1.0], [0.0, 1.0]])
    f = GL.cholesky_psd(small["chol_rankdef_in"])
    assert f.jitter_applied == float(small["chol_rankdef_jitter"]) > 0
    tgt = small["chol_rankdef_in"] + f.jitter_applied * np.eye(3)
    assert np.linalg.norm(f.upper.T @ f.upper - tgt) <= 1e-8 * np.linalg.norm(tgt)
    with pytest.raises(GL.IndefiniteKernelError):
        GL.cholesky_psd(np.diag([1.0, -1.0]))
    f = GL.cholesky_psd(cfg1["kmat"])
    assert f.jitter_applied == 0.0
    assert rel(f.upper, cfg1["r"]) <= 1e-13
    assert np.all(np.tril(f.upper, -1) == 0.0)


@pytest.mark.parametrize("n", [130, 700])
def test_cholesky_large(n):
    rng = np.random.default_rng(n)
    pts = rng.uniform(-1, 1, (n, 6))
    k = O.gaussian_gram(1.0, pts)
    up, jit = O.cholesky_psd(k)
    f = GL.cholesky_psd(k)
    assert f.jitter_applied == jit
    assert rel(f.upper, up) <= 1e-11


# -------------------------------------------------------------- assembly

def test_gram_matches_oracle():
    rng = np.random.default_rng(3)
    pts = rng.uniform(-1, 1, (77, 5))
    g = K.kernels.gram_matrix(K.KernelSpec(0.7, 5), pts)
    assert np.array_equal(g, g.T) and np.all(np.diag(g) == 1.0)
    assert rel(g, O.gaussian_gram(0.7, pts)) <= 1e-15


def test_assemble_cfg1(cfg1):
    sx, sy, sxy = K.build_kernel_specs(2, float(cfg1["bw_sq"]))
    pd = K.assemble(K.SampleSet(cfg1["xs"]), K.SampleSet(cfg1["ys"]), K.FillingPoints(cfg1["xt"], cfg1["yt"]),
                    float(cfg1["l1"]), float(cfg1["l2"]), sx, sy, sxy)
    assert rel(pd.q_mat, cfg1["q"]) <= 1e-15
    assert rel(pd.z, cfg1["z"]) <= 1e-14
    assert rel(pd.embed_sum, cfg1["embed"]) <= 1e-14
    assert pd.q_sq == pytest.approx(float(cfg1["q_sq"]), rel=1e-14)
    assert pd.jitter == 0.0
    assert rel(pd.chol_upper, cfg1["r"]) <= 1e-13
    assert rel(pd.pair_gram(), cfg1["kmat"]) <= 1e-15
    # assemble() skips ProblemData.__post_init__'s symmetrisation pass: the device result is exactly
    # symmetric, so the reference's 0.5 (Q + Qᵀ) (problem.py:86-123) would return it unchanged
    assert np.array_equal(pd.q_mat, pd.q_mat.T)
    import dataclasses
    pd2 = dataclasses.replace(pd, lambda1=2.0 * pd.lambda1)  # a regular instance again
    assert np.array_equal(pd2.q_mat, pd.q_mat) and pd2._dev is None and pd2.lambda1 == 2.0 * pd.lambda1


# ------------------------------------------------------------ operators

def test_phi_and_adjoint(cfg1):
    pd = gpu_pd(cfg1)
    g, x = cfg1["op_g"], cfg1["op_x"]
    assert rel(GP.phi_forward(pd, x), cfg1["op_phi"]) <= 1e-13
    pa = GP.phi_adjoint(pd, g)
    assert np.array_equal(pa, pa.T)
    assert rel(pa, cfg1["op_phi_adj"]) <= 1e-13
    # adjointness <Φ(X), γ> = <X, Φ*(γ)>
    rng = np.random.default_rng(0)
    xr = random_symmetric(rng, pd.n)
    gr = rng.standard_normal(pd.n)
    lhs = GP.phi_forward(pd, xr) @ gr
    rhs = np.sum(xr * GP.phi_adjoint(pd, gr))
    assert abs(lhs - rhs) <= 1e-13 * abs(rhs)


def test_residual_parts(cfg1):
    pd = gpu_pd(cfg1)
    r, info = GP.residual_parts(pd, GP.IteratePair(cfg1["op_g"], cfg1["op_x"]))
    assert rel(r.gamma, cfg1["op_r1"]) <= 1e-12
    assert rel(r.x_mat, cfg1["op_r2"]) <= 1e-11
    assert np.array_equal(r.x_mat, r.x_mat.T)
    assert np.max(np.abs(info.eigvals - cfg1["op_eigvals"])) <= 1e-12 * np.abs(cfg1["op_eigvals"]).max()
    assert info.n_pos == int(cfg1["op_npos"])


@pytest.mark.parametrize("n_pos", [0, 1, 3, 5, 6])
def test_spectral_operators_sign_fixtures(small, n_pos):
    p = f"sign{n_pos}_"
    z, s = small[p + "z"], small[p + "s"]
    assert np.max(np.abs(GC.proj_psd(z) - small[p + "proj"])) <= 1e-13
    assert np.max(np.abs(GC.apply_proj_jacobian_at(z, s) - small[p + "mz"])) <= 1e-13
    for mu in (0.03, 1.0, 17.0):
        ref = small[f"{p}elim_{mu}"]
        for path in (None, GC.POS_BLOCK, GC.NONPOS_COMPLEMENT):
            out = GC.apply_eliminator_at(z, s, mu, path)
            assert np.linalg.norm(out - ref) <= 1e-12 * max(np.linalg.norm(ref), 1.0)


def test_eliminator_and_jacobian_cfg1(cfg1):
    pd_o = oracle_pd(cfg1)
    zarg = O.sym(cfg1["op_x"]) - O.constraint_matrix(pd_o, cfg1["op_g"])
    s, mu = cfg1["op_s"], float(cfg1["op_mu"])
    el = GC.apply_eliminator_at(zarg, s, mu)
    assert rel(el, cfg1["op_elim"]) <= 1e-11
    mz = GC.apply_proj_jacobian_at(zarg, s)
    assert rel(mz, cfg1["op_mz"]) <= 1e-11


@pytest.mark.parametrize("form", ["reduced", "blocked", "direct"])
def test_middle_operator(cfg1, form):
    pd = gpu_pd(cfg1)
    out, mu = GN.middle_operator_at(pd, GP.IteratePair(cfg1["op_g"], cfg1["op_x"]), float(cfg1["op_theta"]),
                                    cfg1["op_v"], form=form)
    assert mu == pytest.approx(float(cfg1["op_mu"]), rel=1e-12)
    assert rel(out, cfg1["op_middle"]) <= 1e-11


@pytest.mark.parametrize("form", ["reduced", "blocked"])
@pytest.mark.parametrize("shift", [-5.0, 0.0, 5.0, -1e3, 1e3])
def test_middle_operator_both_paths(cfg1, shift, form):
    """Reduced (B = R·P) vs oracle at states whose spectrum is mostly negative, mixed, mostly
    positive, all negative (k = 0), all positive (k = ℓ): exercises the POS and NONPOS
    (G2 = (RRᵀ)∘(RRᵀ)) branches of both structure-reduced layouts."""
    pd = gpu_pd(cfg1)
    po = oracle_pd(cfg1)
    rng = np.random.default_rng(5)
    x = cfg1["op_x"] + shift * np.eye(pd.n) * np.abs(np.diag(cfg1["op_x"])).mean()
    g = cfg1["op_g"]
    v = rng.standard_normal(pd.n)
    out, mu = GN.middle_operator_at(pd, GP.IteratePair(g, x), 0.7, v, form=form)
    r, dc = O.residual_parts(po, O.Pair(g, x))
    ctx = O.newton_context(dc, r.norm(), 0.7)
    ref = O.middle_operator(po, ctx.op, ctx.mu)(v)
    assert mu == pytest.approx(ctx.mu, rel=1e-12)
    assert rel(out, ref) <= 1e-11, (dc.k, rel(out, ref))


def _perturbed_oracle_pd(d, seed, p="", eps=2.2e-16):
    """Oracle problem with R perturbed by ±eps relative (default 1 ulp: the oracle's own rounding spread)."""
    rng = np.random.default_rng(seed)
    r = d[p + "r"] * (1.0 + rng.choice([-1.0, 1.0], d[p + "r"].shape) * eps)
    return O.Problem(q=d[p + "q"], z=d[p + "z"], q_sq=float(d[p + "q_sq"]), r=r, l1=float(d[p + "l1"]),
                     l2=float(d[p + "l2"]), embed=d.get(p + "embed"))


def test_newton_direction(cfg1):
    """Default profile: CG stops at the 20×(1+2) cap, so the direction is only determined up to the
    oracle's own sensitivity (measured ≈2.3e-5 relative under a 1-ulp perturbation of R; the
    solver's structure-reduced matvec differs from the reference form by ~1e-13, i.e. a larger
    perturbation than 1 ulp): tolerance 100× the ulp spread.  The converged-CG test below is the
    accuracy check (≤1e-8)."""
    pd = gpu_pd(cfg1)
    w = GP.IteratePair(cfg1["op_g"], cfg1["op_x"])
    st = GN.newton_direction_at(pd, w, float(cfg1["op_theta"]), GN.NewtonConfig())
    spread = 0.0
    for seed in (1, 2):
        po = _perturbed_oracle_pd(cfg1, seed)
        r, dc = O.residual_parts(po, O.Pair(cfg1["op_g"], cfg1["op_x"]))
        so = O.newton_direction(po, r, O.newton_context(dc, r.norm(), float(cfg1["op_theta"])), O.NewtonCfg())
        spread = max(spread, rel(so.dw.g, cfg1["op_dir_dg"]))
    assert st.cg_iters == int(cfg1["op_dir_cg"])
    assert st.criterion_met == bool(cfg1["op_dir_met"])
    assert rel(st.dw.gamma, cfg1["op_dir_dg"]) <= max(1e-9, 100 * spread)
    assert rel(st.dw.x_mat, cfg1["op_dir_dx"]) <= max(1e-9, 100 * spread)
    assert np.array_equal(st.dw.x_mat, st.dw.x_mat.T)


def test_newton_direction_converged_cg(cfg1):
    """With CG driven to 1e-13 the direction is well determined: GPU vs oracle ≤ 1e-9 (Lemma-1 regime)."""
    pd = gpu_pd(cfg1)
    po = oracle_pd(cfg1)
    cfg = GN.NewtonConfig(cg_tol=1e-13, cg_max=3000, cg_restarts=0)
    w = GP.IteratePair(cfg1["op_g"], cfg1["op_x"])
    st = GN.newton_direction_at(pd, w, float(cfg1["op_theta"]), cfg)
    r, dc = O.residual_parts(po, O.Pair(cfg1["op_g"], cfg1["op_x"]))
    so = O.newton_direction(po, r, O.newton_context(dc, r.norm(), float(cfg1["op_theta"])),
                            O.NewtonCfg(cg_tol=1e-13, cg_max=3000, cg_restarts=0))
    assert rel(st.dw.gamma, so.dw.g) <= 1e-8
    assert rel(st.dw.x_mat, so.dw.x) <= 1e-8


def test_eg_step(cfg1):
    pd = gpu_pd(cfg1)
    v = eg_step(pd, GP.IteratePair(cfg1["op_g"], cfg1["op_eg_in_x"]), EgConfig(float(cfg1["eg_stepsize"])))
    assert rel(v.gamma, cfg1["op_eg_g"]) <= 1e-12
    assert rel(v.x_mat, cfg1["op_eg_x"]) <= 1e-11
    assert np.array_equal(v.x_mat, v.x_mat.T)


@pytest.mark.parametrize("n,shift", [(1000, 0.0), (1000, -0.3), (700, 0.2)])
def test_eg_step_large(n, shift):
    """EG step at orders where the α-only back-transform (σ > 0 eigenvectors only, column count read
    on the device) runs its Vᵀ·P products split-K: the partial layout must follow the static column
    bound and the reduction must skip the uncomputed columns (regression: garbage projections)."""
    d = random_problem_arrays(11, n=n)
    rng = np.random.default_rng(n)
    x = random_symmetric(rng, n) / np.sqrt(n) + shift * np.eye(n)
    g = rng.standard_normal(n)
    pd = GP.ProblemData(q_mat=d["q"], z=d["z"], q_sq=d["q_sq"], chol_upper=d["r"], lambda1=d["l1"],
                        lambda2=d["l2"])
    po = O.Problem(q=d["q"], z=d["z"], q_sq=d["q_sq"], r=d["r"], l1=d["l1"], l2=d["l2"])
    s = 0.05
    for _ in range(2):  # second call: workspaces hold the first call's values
        v = eg_step(pd, GP.IteratePair(g, x), EgConfig(s))
    ref = O.eg_step(po, O.Pair(g, x), s)
    assert rel(v.gamma, ref.g) <= 1e-12
    assert rel(v.x_mat, ref.x) <= 1e-11


def test_objective_and_ot(cfg1):
    pd = gpu_pd(cfg1)
    assert GP.objective(pd, cfg1["op_g"]) == pytest.approx(float(cfg1["op_objective"]), rel=1e-13)
    assert GP.ot_estimate(pd, cfg1["tight_gamma"]) == pytest.approx(float(cfg1["tight_ot"]), rel=1e-12)


# ------------------------------------------------------------------ solve

@pytest.mark.parametrize("name", ["interior", "active"])
def test_scalar_kkt_fixtures(small, name):
    z = 1.0 if name == "interior" else -4.0
    pd = GP.ProblemData(q_mat=[[2.0]], z=[z], q_sq=0.0, chol_upper=[[1.0]], lambda1=1.0, lambda2=0.5)
    rep = K.solve(pd, K.SolverConfig(residual_tol=1e-12, max_iter=100))
    assert rep.termination == "converged"
    assert rep.iterations == int(small[f"scalar_{name}_iters"])
    eg, ex = (0.5, 0.0) if name == "interior" else (-1.0, 2.0)
    assert rep.gamma_hat[0] == pytest.approx(eg, abs=1e-10)
    assert rep.x_hat[0, 0] == pytest.approx(ex, abs=1e-10)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_random_problem_solves(small, seed):
    p = f"rand{seed}_"
    pd = gpu_pd(small, p)
    rep = K.solve(pd, K.SolverConfig(residual_tol=1e-10, max_iter=200))
    ref_iters = int(small[p + "iters"])
    if ref_iters < 200:  # the reference converges: same end point
        assert rep.termination == "converged"
        assert abs(rep.iterations - ref_iters) <= 2
        assert rel(rep.gamma_hat, small[p + "gamma"]) <= 1e-8
    else:  # the reference stalls at max_iter (seed 2: ‖R‖≈9.4e-3); so must we, at the same level
        assert rep.termination == "max_iter"
        assert rep.residual_norm == pytest.approx(float(small[p + "res"]), rel=0.05)


def _cfg5_like(seed, n):
    rng = np.random.default_rng(seed)
    xs = np.clip(rng.normal(0.0, 0.3, (n, 3)), -1, 1)
    ys = np.clip(rng.normal(0.2, 0.3, (n, 3)), -1, 1)
    f = rng.uniform(-1, 1, (n, 6))
    sx, sy, sxy = K.build_kernel_specs(3, 1.0)
    return K.assemble(K.SampleSet(xs), K.SampleSet(ys), K.FillingPoints(f[:, :3], f[:, 3:]), 1e-3, 1.0 / n,
                      sx, sy, sxy)


def test_pooled_problem_reuse_is_exact():
    """Released device problems are pooled and reused by the next instance of the same order (all
    workspace, contexts and EG-pipeline buffers): a solve on a reused problem must be bit-identical
    to one on a problem whose workspace held another instance's data."""
    cfg = K.SolverConfig(residual_tol=1e-12, max_iter=6)
    pa = _cfg5_like(1, 300)
    K.solve(pa, cfg)
    pa.release_device()               # → pool
    pb = _cfg5_like(2, 300)           # reuses pa's workspace (stale data everywhere)
    rb = K.solve(pb, cfg)
    pb.release_device()
    pc = _cfg5_like(2, 300)           # same instance again, on pb's workspace
    rc = K.solve(pc, cfg)
    assert np.array_equal(rb.gamma_hat, rc.gamma_hat)
    assert [r.res_accepted for r in rb.trace] == [r.res_accepted for r in rc.trace]
    assert np.array_equal(pb.chol_upper, pc.chol_upper) and np.array_equal(pb.q_mat, pc.q_mat)


def test_repeated_solves_do_not_grow_device_memory():
    """The EG pipeline's buffers are allocated once per problem, not once per solve."""
    torch = pytest.importorskip("torch")
    pd = _cfg5_like(3, 400)
    cfg = K.SolverConfig(residual_tol=1e-12, max_iter=3)
    K.solve(pd, cfg)
    K.solve(pd, cfg)
    free0, _ = torch.cuda.mem_get_info()
    for _ in range(4):
        K.solve(pd, cfg)
    free1, _ = torch.cuda.mem_get_info()
    assert free0 - free1 < 64 * 2 ** 20, (free0 - free1) / 2 ** 20


def test_solve_report_serialises_exactly(cfg1, tmp_path):
    """A real solve's report and trace survive the JSON / CSV formats bit-exactly (§8(f) item 3)."""
    from paper_2310_14087_b200 import report as RP
    rep = K.solve(gpu_pd(cfg1), K.SolverConfig(eg=EgConfig(float(cfg1["eg_stepsize"])), residual_tol=1e-12,
                                              max_iter=5))
    RP.write_report_json(rep, str(tmp_path / "r.json"), include_x=True)
    RP.write_trace_csv(rep.trace, str(tmp_path / "t.csv"))
    back = RP.read_report_json(str(tmp_path / "r.json"))
    assert np.array_equal(back.gamma_hat, rep.gamma_hat) and np.array_equal(back.x_hat, rep.x_hat)
    assert back.trace == rep.trace == RP.read_trace_csv(str(tmp_path / "t.csv"))


@pytest.mark.parametrize("hook,values", [("kot_debug_cg_batch", (1, 4, 7)), ("kot_debug_eg_parallel", (0, 1))])
def test_schedule_variants_are_bit_identical(hook, values):
    """Batched CG stopping (device-side test, B iterations per host check) and the parallel EG
    projections only change the schedule: the solve must be bit-identical for every setting."""
    from paper_2310_14087_b200 import _lib
    f = getattr(_lib.lib(), hook)
    pd = _cfg5_like(7, 700)
    step = 0.5 / (np.linalg.norm(pd.q_mat) / (2 * pd.lambda2) + np.linalg.norm(pd.pair_gram()))
    cfg = K.SolverConfig(eg=EgConfig(step), residual_tol=1e-12, max_iter=6)
    reps = []
    try:
        for v in values:
            f(v)
            reps.append(K.solve(pd, cfg))
    finally:
        f(values[-1] if hook == "kot_debug_eg_parallel" else 4)
    for r in reps[1:]:
        assert np.array_equal(r.gamma_hat, reps[0].gamma_hat) and np.array_equal(r.x_hat, reps[0].x_hat)
        assert [(t.res_accepted, t.res_eg, t.cg_iters) for t in r.trace] == \
               [(t.res_accepted, t.res_eg, t.cg_iters) for t in reps[0].trace]


def test_lockstep_replay_cfg1(cfg1):
    """one GPU iteration from each saved oracle state.

    The oracle is run from the same state on ±1e-13-relative perturbations of R (4 seeds) — the
    size by which the GPU's arithmetic differs from the reference (its structure-reduced matvec
    agrees with the reference form to ~1e-13).  The GPU's CG count must be one the oracle ensemble
    produces (Eq.(9) knife edges flip the restart count: measured at state 5); when the ensemble
    agrees and the GPU matches the reference, the next w must agree to max(1e-9, 10× ensemble
    spread).  v (no CG) is checked at 1e-9 everywhere."""
    pd = gpu_pd(cfg1)
    cfg = K.SolverConfig(eg=EgConfig(float(cfg1["eg_stepsize"])), residual_tol=1e-12, max_iter=40)
    ocfg = O.SolverCfg(eg_stepsize=float(cfg1["eg_stepsize"]), residual_tol=1e-12, max_iter=40)
    matched = 0
    for i in cfg1["replay_iters"]:
        if f"rp{i}_next_wg" not in cfg1:
            continue
        w = GP.IteratePair(cfg1[f"rp{i}_wg"], cfg1[f"rp{i}_wx"])
        v = GP.IteratePair(cfg1[f"rp{i}_vg"], cfg1[f"rp{i}_vx"])
        spread, cg_set = 0.0, {int(cfg1["paper_cg_iters"][i])}
        for seed in (11, 12, 13, 14):
            po = _perturbed_oracle_pd(cfg1, seed, eps=1e-13)
            ow = O.Pair(w.gamma.copy(), w.x_mat.copy())
            r_w, dc_w = O.residual_parts(po, ow)
            st0 = O.State(ow, O.Pair(v.gamma.copy(), v.x_mat.copy()), r_w, dc_w, r_w.norm(), None, None,
                          r_w.norm(), float(cfg1[f"rp{i}_theta"]))
            ost, orec, _ = O.iterate_once(po, st0, int(i), ocfg)
            cg_set.add(orec.cg_iters)
            if orec.cg_iters == int(cfg1["paper_cg_iters"][i]):
                spread = max(spread, rel(ost.w.g, cfg1[f"rp{i}_next_wg"]), rel(ost.w.x, cfg1[f"rp{i}_next_wx"]))
        w2, v2, th2, rec = GS.iterate(pd, cfg, w, v, float(cfg1[f"rp{i}_theta"]), int(i))
        if rec.cg_iters not in cg_set:
            # Rare rounding events in the capped second CG attempt flip Eq.(9) (measured: the oracle
            # itself gives lhs 0.44 instead of 0.32 for one of six 1e-13 seeds at state 2, the GPU
            # 0.61 for one eigensolver variant): the GPU run must then be the outlier of its own
            # ±1e-14 ensemble, i.e. most perturbed GPU runs land in the oracle's set.
            rng = np.random.default_rng(i)
            hits = 0
            for _ in range(3):
                xp = w.x_mat * (1.0 + 1e-14 * rng.standard_normal(w.x_mat.shape))
                wp = GP.IteratePair(w.gamma, 0.5 * (xp + xp.T))
                hits += GS.iterate(pd, cfg, wp, v, float(cfg1[f"rp{i}_theta"]), int(i))[3].cg_iters in cg_set
            assert hits >= 2, (i, rec.cg_iters, cg_set, hits)
            continue
        # the EG step has no CG: v is determined to eigensolver accuracy
        assert rel(v2.gamma, cfg1[f"rp{i}_next_vg"]) <= 1e-9, i
        assert rel(v2.x_mat, cfg1[f"rp{i}_next_vx"]) <= 1e-9, i
        if rec.cg_iters != int(cfg1["paper_cg_iters"][i]):
            continue
        # capped CG (default profile): one iteration's w is only determined to the CG's rounding
        # sensitivity; bounded loosely here — the converged-CG replay below is the tight check
        tol = max(2e-3, 10 * spread)
        assert rec.accepted == ("ssn" if cfg1["paper_accepted_ssn"][i] else "eg"), i
        assert th2 == pytest.approx(float(cfg1[f"rp{i}_next_theta"]), rel=1e-12), i
        assert rel(w2.gamma, cfg1[f"rp{i}_next_wg"]) <= tol, (i, tol)
        assert rel(w2.x_mat, cfg1[f"rp{i}_next_wx"]) <= tol, (i, tol)
        matched += 1
    assert matched >= 3


def test_lockstep_replay_converged_cg(cfg1):
    """Replay with the Newton system solved to 1e-14 on both sides (cg_tol, no restarts): one full
    iteration (EG step, residuals, Newton step, θ rule, acceptance) must agree to 1e-8."""
    pd = gpu_pd(cfg1)
    newton = K.NewtonConfig(cg_tol=1e-14, cg_max=3000, cg_restarts=0)
    cfg = K.SolverConfig(newton=newton, eg=EgConfig(float(cfg1["eg_stepsize"])), residual_tol=1e-12, max_iter=40)
    ocfg = O.SolverCfg(newton=O.NewtonCfg(cg_tol=1e-14, cg_max=3000, cg_restarts=0),
                       eg_stepsize=float(cfg1["eg_stepsize"]), residual_tol=1e-12, max_iter=40)
    po = oracle_pd(cfg1)
    for i in (0, 2, 10, 20):
        w = GP.IteratePair(cfg1[f"rp{i}_wg"], cfg1[f"rp{i}_wx"])
        v = GP.IteratePair(cfg1[f"rp{i}_vg"], cfg1[f"rp{i}_vx"])
        theta = float(cfg1[f"rp{i}_theta"])
        ow = O.Pair(w.gamma.copy(), w.x_mat.copy())
        r_w, dc_w = O.residual_parts(po, ow)
        st0 = O.State(ow, O.Pair(v.gamma.copy(), v.x_mat.copy()), r_w, dc_w, r_w.norm(), None, None, r_w.norm(),
                      theta)
        ost, orec, _ = O.iterate_once(po, st0, i, ocfg)
        w2, v2, th2, rec = GS.iterate(pd, cfg, w, v, theta, i)
        assert rec.accepted == orec.accepted and th2 == pytest.approx(ost.theta, rel=1e-12), i
        assert rel(w2.gamma, ost.w.g) <= 1e-8, i
        assert rel(w2.x_mat, ost.w.x) <= 1e-8, i
        assert rel(v2.x_mat, ost.v.x) <= 1e-9, i


def test_paper_profile_first_iterations(cfg1):
    pd = gpu_pd(cfg1)
    cfg = K.SolverConfig(eg=EgConfig(float(cfg1["eg_stepsize"])), residual_tol=1e-12, max_iter=40)
    rep = K.solve(pd, cfg)
    res = np.array([t.res_accepted for t in rep.trace])
    ref = cfg1["paper_res_accepted"]
    # chaotic at ulp level: tight agreement only on the first iterations
    assert np.allclose(res[:2], ref[:2], rtol=1e-8)
    # beyond that only the envelope is reproducible (oracle vs itself under ±2 ulp: >1e-2 by iter 4-88)
    assert np.all(np.abs(np.log(res / ref)) <= np.log(3.0))
    assert rep.iterations == 40


def test_tight_profile_end_state(cfg1):
    """tol 1e-10 end state vs the reference."""
    pd = gpu_pd(cfg1)
    cfg = K.SolverConfig(newton=K.NewtonConfig(alpha1=1e-8, alpha2=1e-4, cg_max=500),
                         eg=EgConfig(float(cfg1["eg_stepsize"])), residual_tol=1e-10, max_iter=1000)
    rep = K.solve(pd, cfg)
    assert rep.termination == "converged"
    ref_iters = int(cfg1["tight_iters"])
    # The tight-profile trajectory is chaotic: under ±1-ulp perturbations of R the
    # GPU takes 399-508 iterations and the oracle itself spreads similarly, with
    # rare long excursions; the iteration count is therefore only checked within a 2× band, while
    # the END STATE at tol 1e-10 is checked tightly.
    assert ref_iters / 2 <= rep.iterations <= 2 * ref_iters
    obj = O.objective(oracle_pd(cfg1), rep.gamma_hat)
    assert obj == pytest.approx(float(cfg1["tight_objective"]), rel=1e-8)
    assert rel(rep.gamma_hat, cfg1["tight_gamma"]) <= 1e-6
    assert rep.ot_estimate == pytest.approx(float(cfg1["tight_ot"]), rel=1e-8)


def test_evaluate_map(cfg1):
    """§8(f) next #1: potentials / Monge map at query points vs the reference (problem.py:254-284)."""
    sx, sy, sxy = K.build_kernel_specs(2, float(cfg1["bw_sq"]))
    pd = gpu_pd(cfg1)
    pd.filling = K.FillingPoints(cfg1["xt"], cfg1["yt"])
    pd.spec_x = sx
    u, t = GP.evaluate_map(pd, K.SampleSet(cfg1["xs"]), cfg1["tight_gamma"], cfg1["map_queries"])
    assert rel(u, cfg1["map_u"]) <= 1e-12
    assert rel(t, cfg1["map_t"]) <= 1e-12
    u1, t1 = GP.potential_and_map(pd, K.SampleSet(cfg1["xs"]), cfg1["tight_gamma"], cfg1["map_queries"][0])
    assert u1 == pytest.approx(float(cfg1["map_u"][0]), rel=1e-12)


# ------------------------------------------------ row-sharded CG matvec (config 4)

@pytest.mark.parametrize("world", [2, 3, 7])
@pytest.mark.parametrize("shift", [-5.0, 5.0])
@pytest.mark.parametrize("form", ["reduced", "blocked"])
def test_row_sharded_middle_operator(cfg1, world, shift, form):
    """The sharded decompositions of the structure-reduced matvec (rowshard.py), every rank's share
    computed in turn on one device (the single-GPU hook of kot_problem_shard), vs the oracle, for the
    POS and NONPOS branches and shares that do not align with the GEMM tiles: "reduced" = the split
    H form (mixed-block columns + folded H/Q rows per rank, partial vectors summed), "blocked" = the
    legacy row-block layout (partial T̃ summed)."""
    from paper_2310_14087_b200 import rowshard
    pd = gpu_pd(cfg1)
    po = oracle_pd(cfg1)
    rowshard.emulate_shards(pd, world)
    rng = np.random.default_rng(11)
    x = cfg1["op_x"] + shift * np.eye(pd.n) * np.abs(np.diag(cfg1["op_x"])).mean()
    g = cfg1["op_g"]
    v = rng.standard_normal(pd.n)
    out, mu = GN.middle_operator_at(pd, GP.IteratePair(g, x), 0.7, v, form=form)
    r, dc = O.residual_parts(po, O.Pair(g, x))
    ctx = O.newton_context(dc, r.norm(), 0.7)
    ref = O.middle_operator(po, ctx.op, ctx.mu)(v)
    assert rel(out, ref) <= 1e-11, (world, dc.k, rel(out, ref))


@pytest.mark.parametrize("world", [2, 8])
def test_row_sharded_matches_unsharded_large(world):
    """ℓ = 700 (several 64-row tiles per block, ragged last block): sharded = unsharded to 1e-12."""
    from paper_2310_14087_b200 import configs, rowshard
    wl = configs.config3(n=700)
    sx, sy, sxy = K.build_kernel_specs(wl.d, wl.bandwidth_sq)
    pd = K.assemble(K.SampleSet(wl.xs), K.SampleSet(wl.ys), K.FillingPoints(wl.xt, wl.yt), wl.lambda1,
                    wl.lambda2, sx, sy, sxy)
    rng = np.random.default_rng(3)
    for shift in (-0.2, 0.2):
        x = random_symmetric(rng, pd.n, 1.0 / pd.n) + shift * np.eye(pd.n) / pd.n
        w = GP.IteratePair(rng.standard_normal(pd.n) * 1e-2, x)
        v = rng.standard_normal(pd.n)
        rowshard.emulate_shards(pd, 1)
        ref, _ = GN.middle_operator_at(pd, w, 0.3, v)
        rowshard.emulate_shards(pd, world)
        out, _ = GN.middle_operator_at(pd, w, 0.3, v)
        assert rel(out, ref) <= 1e-12, (world, shift, rel(out, ref))


def test_row_sharded_iteration_replay(cfg1):
    """One full converged-CG iteration through the sharded matvec agrees with the oracle to 1e-8."""
    from paper_2310_14087_b200 import rowshard
    pd = gpu_pd(cfg1)
    rowshard.emulate_shards(pd, 3)
    newton = K.NewtonConfig(cg_tol=1e-14, cg_max=3000, cg_restarts=0)
    cfg = K.SolverConfig(newton=newton, eg=EgConfig(float(cfg1["eg_stepsize"])), residual_tol=1e-12, max_iter=40)
    ocfg = O.SolverCfg(newton=O.NewtonCfg(cg_tol=1e-14, cg_max=3000, cg_restarts=0),
                       eg_stepsize=float(cfg1["eg_stepsize"]), residual_tol=1e-12, max_iter=40)
    po = oracle_pd(cfg1)
    for i in (0, 10):
        w = GP.IteratePair(cfg1[f"rp{i}_wg"], cfg1[f"rp{i}_wx"])
        v = GP.IteratePair(cfg1[f"rp{i}_vg"], cfg1[f"rp{i}_vx"])
        theta = float(cfg1[f"rp{i}_theta"])
        ow = O.Pair(w.gamma.copy(), w.x_mat.copy())
        r_w, dc_w = O.residual_parts(po, ow)
        st0 = O.State(ow, O.Pair(v.gamma.copy(), v.x_mat.copy()), r_w, dc_w, r_w.norm(), None, None, r_w.norm(),
                      theta)
        ost, orec, _ = O.iterate_once(po, st0, i, ocfg)
        w2, v2, th2, rec = GS.iterate(pd, cfg, w, v, theta, i)
        assert rec.accepted == orec.accepted, i
        assert rel(w2.gamma, ost.w.g) <= 1e-8, i
        assert rel(w2.x_mat, ost.w.x) <= 1e-8, i


# ------------------------------------------- grid-resident sytrd mid kernel (sytrd_mid.cuh)

@pytest.fixture
def mid_everywhere():
    """Force the grid-resident mid kernel for every order (default: latency-critical eigensolves with a
    trailing block larger than the cluster tail's)."""
    from paper_2310_14087_b200 import _lib
    f = _lib.lib().kot_debug_trd_mid
    yield f
    f(1, 0)


def _check_decomposition(z, tol=1e-12):
    n = z.shape[0]
    dc = GL.sym_eig(z)
    ref = np.sort(np.linalg.eigvalsh(z))[::-1]
    nz = max(np.abs(ref).max(), 1e-300)
    p = dc.eigvecs
    assert np.max(np.abs(dc.eigvals - ref)) <= tol * nz * max(1.0, n / 100)
    assert np.max(np.abs(p.T @ p - np.eye(n))) <= tol * max(1.0, n / 100)
    assert np.max(np.abs((p * dc.eigvals) @ p.T - z)) <= tol * nz * max(1.0, n / 100)
    return dc


@pytest.mark.parametrize("tail", [0, 200, 640])
@pytest.mark.parametrize("n", [3, 4, 33, 148, 149, 257, 641, 999, 1000])
def test_mid_kernel_sym_eig(mid_everywhere, n, tail):
    """Every column through the mid kernel (tail = 0) or handed over to the cluster tail for the last
    `tail` columns; odd and even orders (padding column), fewer rows than CTAs, one row triple."""
    mid_everywhere(2, tail)
    rng = np.random.default_rng(1000 * tail + n)
    _check_decomposition(random_symmetric(rng, n))


@pytest.mark.parametrize("n", [1500, 1776, 1777, 2000])
def test_mid_kernel_large_orders(mid_everywhere, n):
    """Orders around the resident-block capacity (1776 on 148 SMs): panels first, then the mid kernel."""
    mid_everywhere(1, 0)
    rng = np.random.default_rng(n)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    vals = np.concatenate([np.linspace(1, 100, n // 2), -np.linspace(1e-4, 1, n - n // 2)])
    z = (q * vals) @ q.T
    _check_decomposition(0.5 * (z + z.T))


@pytest.mark.parametrize("n", [1500, 2000, 2300])
def test_mid_kernel_head_launch(mid_everywhere, n):
    """The solver's schedule beside an EG pipeline, forced for a standalone eigensolve: panels, a head
    launch on every SM that hands its block over, then the launch on 96 SMs."""
    from paper_2310_14087_b200 import _lib
    mid_everywhere(1, 0)
    head = _lib.lib().kot_debug_trd_mid_head
    head(2)
    try:
        rng = np.random.default_rng(n + 1)
        _check_decomposition(random_symmetric(rng, n))
    finally:
        head(1)


def test_mid_kernel_identity_reflectors(mid_everywhere):
    """Columns with H = I (τ = 0): a diagonal matrix, and a block matrix mixing both kinds of column."""
    mid_everywhere(2, 0)
    rng = np.random.default_rng(5)
    _check_decomposition(np.diag(rng.standard_normal(700)))
    b = np.zeros((800, 800))
    x = rng.standard_normal((400, 400))
    b[:400, :400] = (x + x.T) / 2
    b[600:, 600:] = np.eye(200) * 3.0
    _check_decomposition(b)


@pytest.mark.parametrize("scale", [1e-145, 1e-8, 1e8, 1e150])
def test_mid_kernel_scales(mid_everywhere, scale):
    """dlarfg from the sum of squares (hardware rsqrt / reciprocal seeds + Newton steps) and its dlapy2
    branch for sums of squares near over/underflow (below 1e-145 the divide-and-conquer stage itself
    loses accuracy to underflow, with or without this kernel)."""
    mid_everywhere(2, 0)
    rng = np.random.default_rng(9)
    _check_decomposition(scale * random_symmetric(rng, 300), tol=1e-11 if scale < 1e-100 else 1e-12)


def test_mid_kernel_is_deterministic(mid_everywhere):
    """The tagged-sector exchange never delivers a torn or stale payload: repeated eigensolves of the
    same matrix are bit-identical (every CTA derives the same scalars from the same gathered vectors)."""
    mid_everywhere(1, 0)
    rng = np.random.default_rng(21)
    z = random_symmetric(rng, 1400)
    first = GL.sym_eig(z)
    for _ in range(20):
        again = GL.sym_eig(z)
        assert np.array_equal(first.eigvals, again.eigvals)
        assert np.array_equal(first.eigvecs, again.eigvecs)


# ------------------------------------------- two-stage tridiagonalisation (eig2.cu)

def _tridiag(z, stages):
    import ctypes as C
    from paper_2310_14087_b200 import _lib
    n = z.shape[0]
    L = _lib.lib()
    f = L.kot_debug_tridiag
    f.argtypes = [_lib.dptr, C.c_int, C.c_int, C.c_int, _lib.dptr, _lib.dptr]
    d, e = np.empty(n), np.empty(max(n - 1, 1))
    zz = _lib.f64(z)
    _lib.check(f(_lib.ptr(zz), n, _lib.default_device(), stages, _lib.ptr(d), _lib.ptr(e)))
    return d, e[:n - 1]


@pytest.mark.parametrize("n", [3, 4, 17, 18, 33, 64, 100, 257, 700, 1100])
@pytest.mark.parametrize("stages", [1, 2])
def test_tridiagonal_form_preserves_spectrum(n, stages):
    """sy2sb + sb2st (band width 16, clusters) and the one-stage sytrd: same spectrum as the input."""
    rng = np.random.default_rng(n)
    z = random_symmetric(rng, n)
    d, e = _tridiag(z, stages)
    t = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
    ref = np.linalg.eigvalsh(z)
    got = np.linalg.eigvalsh(t)
    assert np.max(np.abs(got - ref)) <= 1e-12 * np.abs(ref).max() * max(1.0, n / 100), (n, stages)


@pytest.fixture
def two_stage():
    from paper_2310_14087_b200 import _lib
    f = _lib.lib().kot_debug_eig_stages
    f(2)
    yield
    f(0)


@pytest.mark.parametrize("n", [64, 65, 300, 1100])
def test_two_stage_sym_eig(two_stage, n):
    """Full eigendecomposition through the two-stage reduction (+ Q2, Q1 back-transforms)."""
    rng = np.random.default_rng(100 + n)
    z = random_symmetric(rng, n)
    dc = GL.sym_eig(z)
    ref = np.sort(np.linalg.eigvalsh(z))[::-1]
    scale = np.abs(ref).max()
    assert np.max(np.abs(dc.eigvals - ref)) <= 1e-13 * scale * max(1.0, n / 100)
    p = dc.eigvecs
    assert np.linalg.norm(p.T @ p - np.eye(n)) <= 1e-12 * n
    assert np.linalg.norm(p @ np.diag(dc.eigvals) @ p.T - z) <= 1e-13 * scale * n


def test_two_stage_residual_and_middle_operator(two_stage, cfg1):
    pd = gpu_pd(cfg1)
    po = oracle_pd(cfg1)
    w = GP.IteratePair(cfg1["op_g"], cfg1["op_x"])
    out, mu = GN.middle_operator_at(pd, w, float(cfg1["op_theta"]), cfg1["op_v"])
    assert rel(out, cfg1["op_middle"]) <= 1e-11
    r, dc = O.residual_parts(po, O.Pair(cfg1["op_g"], cfg1["op_x"]))
    rg, _ = GP.residual_parts(pd, w)
    assert rel(rg.gamma, r.g) <= 1e-11 and rel(rg.x_mat, r.x) <= 1e-11


def test_sym_eig_default_two_stage_order():
    """ℓ ≥ 3000 uses the two-stage reduction by default: full decomposition accuracy at ℓ = 3001."""
    n = 3001
    rng = np.random.default_rng(7)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    vals = np.concatenate([np.linspace(1, 50, n // 2), -np.logspace(-6, 0, n - n // 2)])
    z = (q * vals) @ q.T
    z = 0.5 * (z + z.T)
    dc = GL.sym_eig(z)
    ref = np.sort(vals)[::-1]
    assert np.max(np.abs(dc.eigvals - ref)) <= 2e-12 * np.abs(ref).max()
    p = dc.eigvecs
    assert np.linalg.norm(p.T @ p - np.eye(n)) <= 1e-10
    assert np.linalg.norm((p * dc.eigvals) @ p.T - z) / np.linalg.norm(z) <= 1e-13
    assert dc.pos_idx.size == n // 2


def test_two_stage_iteration_replay_converged_cg(two_stage, cfg1):
    """One full SSN iteration (EG step, residuals, converged-CG Newton step, acceptance) with every
    eigensolve going through the two-stage reduction agrees with the oracle to 1e-8."""
    pd = gpu_pd(cfg1)
    newton = K.NewtonConfig(cg_tol=1e-14, cg_max=3000, cg_restarts=0)
    cfg = K.SolverConfig(newton=newton, eg=EgConfig(float(cfg1["eg_stepsize"])), residual_tol=1e-12, max_iter=40)
    ocfg = O.SolverCfg(newton=O.NewtonCfg(cg_tol=1e-14, cg_max=3000, cg_restarts=0),
                       eg_stepsize=float(cfg1["eg_stepsize"]), residual_tol=1e-12, max_iter=40)
    po = oracle_pd(cfg1)
    for i in (0, 10, 20):
        w = GP.IteratePair(cfg1[f"rp{i}_wg"], cfg1[f"rp{i}_wx"])
        v = GP.IteratePair(cfg1[f"rp{i}_vg"], cfg1[f"rp{i}_vx"])
        theta = float(cfg1[f"rp{i}_theta"])
        ow = O.Pair(w.gamma.copy(), w.x_mat.copy())
        r_w, dc_w = O.residual_parts(po, ow)
        st0 = O.State(ow, O.Pair(v.gamma.copy(), v.x_mat.copy()), r_w, dc_w, r_w.norm(), None, None, r_w.norm(),
                      theta)
        ost, orec, _ = O.iterate_once(po, st0, i, ocfg)
        w2, v2, th2, rec = GS.iterate(pd, cfg, w, v, theta, i)
        assert rec.accepted == orec.accepted and th2 == pytest.approx(ost.theta, rel=1e-12), i
        assert rel(w2.gamma, ost.w.g) <= 1e-8, i
        assert rel(w2.x_mat, ost.w.x) <= 1e-8, i
        assert rel(v2.x_mat, ost.v.x) <= 1e-9, i


@pytest.mark.parametrize("n", [700, 701])
def test_gemm_cores_agree(n):
    """The TMA-staged DMMA core (default) and the cp.async core compute the same products: Φ* is
    bit-identical (same k order per element), Φ's fused row-dot sums the tile's columns in the TMA
    fragment order (≤1e-15), and a short solve agrees (odd orders fall back to the cp.async core)."""
    from paper_2310_14087_b200 import _lib
    f = _lib.lib().kot_debug_gemm_tma
    d = random_problem_arrays(5, n=n)
    pd = GP.ProblemData(q_mat=d["q"], z=d["z"], q_sq=d["q_sq"], chol_upper=d["r"], lambda1=d["l1"], lambda2=d["l2"])
    rng = np.random.default_rng(n)
    g = rng.standard_normal(n)
    x = random_symmetric(rng, n)
    cfg = K.SolverConfig(eg=EgConfig(0.05), residual_tol=1e-12, max_iter=3)
    out = []
    try:
        for mode in (0, 1):
            f(mode)
            out.append((GP.phi_adjoint(pd, g), GP.phi_forward(pd, x), K.solve(pd, cfg)))
    finally:
        f(1)
    (a0, p0, r0), (a1, p1, r1) = out
    assert np.array_equal(a0, a1) and rel(p1, p0) <= 1e-15
    assert rel(r1.gamma_hat, r0.gamma_hat) <= 1e-10
    assert [t.cg_iters for t in r1.trace] == [t.cg_iters for t in r0.trace]
