"""Generate golden fixtures from the UNMODIFIED reference ``kot`` package.

Run in the build container (the only place ``/root/reference`` exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``kot`` from ``/root/reference/pkg/src`` (read-only, nothing is
copied) and writes small ``.npz`` files next to this script.  The fixtures
pin the oracle (``oracle/kot_port.py``) and are the parity targets of the
GPU tests; the GPU box never reads ``/root/reference``.

Inputs are the seeded synthetic config-1 workload of SURVEY.md §8(d)
(``paper_2310_14087_b200/configs.py``) and the reference's own test fixtures
(``pkg/tests/conftest.py:9-63``: random_problem, scalar_interior,
scalar_active, symmetric_with_signs).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import kot  # noqa: E402
from kot import linalg as klin  # noqa: E402
from kot import newton as knew  # noqa: E402
from kot import problem as kprob  # noqa: E402
from kot import psdcone as kpsd  # noqa: E402
from kot import eg as keg  # noqa: E402
from kot import solver as ksol  # noqa: E402

from paper_2310_14087_b200 import configs  # noqa: E402


def _pd_arrays(pd, prefix=""):
    out = {
        prefix + "q": pd.q_mat, prefix + "z": pd.z, prefix + "q_sq": np.float64(pd.q_sq),
        prefix + "r": pd.chol_upper, prefix + "l1": np.float64(pd.lambda1),
        prefix + "l2": np.float64(pd.lambda2), prefix + "jitter": np.float64(pd.jitter),
    }
    if pd.embed_sum is not None:
        out[prefix + "embed"] = pd.embed_sum
    return out


def _trace_arrays(trace, prefix):
    return {
        prefix + "res_accepted": np.array([t.res_accepted for t in trace]),
        prefix + "res_ssn": np.array([t.res_ssn for t in trace]),
        prefix + "res_eg": np.array([t.res_eg for t in trace]),
        prefix + "accepted_ssn": np.array([t.accepted == "ssn" for t in trace]),
        prefix + "theta": np.array([t.theta for t in trace]),
        prefix + "mu": np.array([t.mu for t in trace]),
        prefix + "cg_iters": np.array([t.cg_iters for t in trace]),
        prefix + "criterion_met": np.array([t.criterion_met for t in trace]),
        prefix + "crit_lhs": np.array([t.crit_lhs for t in trace]),
        prefix + "crit_rhs": np.array([t.crit_rhs for t in trace]),
    }


def random_problem(seed, n=5, q_reg=0.5, feat_reg=0.5, z_scale=2.0, lambda1=0.5, lambda2=0.4):
    """Same draws as pkg/tests/conftest.py:9-31 (kept here so the fixture is self-describing)."""
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, n))
    q = a @ a.T / n + q_reg * np.eye(n)
    b = rng.standard_normal((n, n))
    r_up = np.linalg.cholesky(b @ b.T / n + feat_reg * np.eye(n)).T
    return kprob.ProblemData(q_mat=q, z=z_scale * rng.standard_normal(n),
                             q_sq=float(rng.uniform(0.0, 1.0)), chol_upper=r_up,
                             lambda1=lambda1, lambda2=lambda2)


def symmetric_with_signs(rng, n, n_pos, gap=0.1):
    """pkg/tests/conftest.py:55-63."""
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    pos = 0.5 + gap * np.arange(n_pos) + rng.uniform(0, 0.05, size=n_pos)
    neg = -0.5 - gap * np.arange(n - n_pos) - rng.uniform(0, 0.05, size=n - n_pos)
    return (q * np.concatenate([pos, neg])) @ q.T


def gen_cfg1():
    wl = configs.config1()
    sx, sy, sxy = kprob.build_kernel_specs(wl.d, wl.bandwidth_sq)
    pd = kprob.assemble(kot.SampleSet(wl.xs, "mu"), kot.SampleSet(wl.ys, "nu"),
                        kprob.FillingPoints(wl.xt, wl.yt), wl.lambda1, wl.lambda2, sx, sy, sxy)
    kmat = kot.kernels.gram_matrix(sxy, np.hstack([wl.xt, wl.yt]))
    step = configs.eg_stepsize(pd.q_mat, kmat, pd.lambda2)
    out = {"xs": wl.xs, "ys": wl.ys, "xt": wl.xt, "yt": wl.yt, "bw_sq": np.float64(wl.bandwidth_sq),
           "kmat": kmat, "eg_stepsize": np.float64(step)}
    out.update(_pd_arrays(pd))

    # ---- paper profile: 40 iterations, capture iterates for lock-step replay
    probes = []
    cfg = ksol.SolverConfig(newton=knew.NewtonConfig(), eg=keg.EgConfig(stepsize=step),
                            residual_tol=1e-12, max_iter=40)
    # capture (w, v, theta) before each iteration by wrapping eg_step (v enters eg_step)
    vs = []
    orig_eg = ksol.eg_step

    def spy(pd_, v_, c_):
        vs.append((v_.gamma.copy(), v_.x_mat.copy()))
        return orig_eg(pd_, v_, c_)

    ksol.eg_step = spy
    try:
        rep = ksol.solve(pd, cfg, on_iteration=lambda p: probes.append(
            (p.w.gamma.copy(), p.w.x_mat.copy(), p.theta, p.mu, p.r.gamma.copy(), p.r.x_mat.copy(),
             p.dw.gamma.copy(), p.dw.x_mat.copy())))
    finally:
        ksol.eg_step = orig_eg
    out.update(_trace_arrays(rep.trace, "paper_"))
    keep = [0, 1, 2, 5, 10, 20, 39]
    out["replay_iters"] = np.array(keep)
    for i in keep:
        g, x, th, mu, r1, r2, dg, dx = probes[i]
        out[f"rp{i}_wg"], out[f"rp{i}_wx"], out[f"rp{i}_theta"] = g, x, np.float64(th)
        out[f"rp{i}_vg"], out[f"rp{i}_vx"] = vs[i]
        out[f"rp{i}_mu"], out[f"rp{i}_r1"], out[f"rp{i}_r2"] = np.float64(mu), r1, r2
        out[f"rp{i}_dg"], out[f"rp{i}_dx"] = dg, dx
        # next-iteration state for the replay comparison
        if i + 1 < len(probes):
            out[f"rp{i}_next_wg"], out[f"rp{i}_next_wx"] = probes[i + 1][0], probes[i + 1][1]
            out[f"rp{i}_next_theta"] = np.float64(probes[i + 1][2])
            out[f"rp{i}_next_vg"], out[f"rp{i}_next_vx"] = vs[i + 1]

    # ---- per-op values at replay state 10 (a generic interior iterate)
    g, x = probes[10][0], probes[10][1]
    w = kprob.IteratePair(g, x)
    r, dc = kprob.residual_parts(pd, w)
    ctx = knew.newton_context(dc, r.norm(), probes[10][2])
    rng = np.random.default_rng(1234)
    vvec = rng.standard_normal(pd.n)
    smat = rng.standard_normal((pd.n, pd.n))
    smat = 0.5 * (smat + smat.T)
    out.update({
        "op_g": g, "op_x": x, "op_theta": np.float64(probes[10][2]),
        "op_phi": kprob.phi_forward(pd, x), "op_phi_adj": kprob.phi_adjoint(pd, g),
        "op_r1": r.gamma, "op_r2": r.x_mat, "op_eigvals": dc.eigvals, "op_npos": np.int64(dc.n_pos),
        "op_proj": kpsd.proj_from_decomp(dc), "op_mu": np.float64(ctx.mu),
        "op_v": vvec, "op_s": smat,
        "op_middle": knew.middle_operator(pd, ctx.eliminator, ctx.mu)(vvec),
        "op_elim": kpsd.apply_eliminator(ctx.eliminator, smat),
        "op_mz": kpsd.apply_proj_jacobian(ctx.coeffs, smat),
        "op_objective": np.float64(kprob.objective(pd, g)),
    })
    st = knew.newton_direction(pd, r, ctx, knew.NewtonConfig())
    out.update({"op_dir_dg": st.dw.gamma, "op_dir_dx": st.dw.x_mat, "op_dir_cg": np.int64(st.cg_iters),
                "op_dir_met": np.bool_(st.criterion_met), "op_dir_lhs": np.float64(st.crit_lhs)})
    ve = keg.eg_step(pd, kprob.IteratePair(g, kpsd.proj_psd(x)), keg.EgConfig(stepsize=step))
    out.update({"op_eg_in_x": kpsd.proj_psd(x), "op_eg_g": ve.gamma, "op_eg_x": ve.x_mat})

    # ---- tight profile to 1e-10 (end-state parity target)
    cfg_t = ksol.SolverConfig(newton=knew.NewtonConfig(alpha1=1e-8, alpha2=1e-4, cg_max=500),
                              eg=keg.EgConfig(stepsize=step), residual_tol=1e-10, max_iter=1000)
    rep_t = ksol.solve(pd, cfg_t)
    out.update({"tight_gamma": rep_t.gamma_hat, "tight_res": np.float64(rep_t.residual_norm),
                "tight_iters": np.int64(rep_t.iterations), "tight_ot": np.float64(rep_t.ot_estimate),
                "tight_objective": np.float64(kprob.objective(pd, rep_t.gamma_hat))})
    out.update(_trace_arrays(rep_t.trace, "tight_"))
    q = np.stack([wl.xs[:8, 0] * 0.9, wl.xs[:8, 1] * 0.9], axis=1)
    u, tmap = kprob.evaluate_map(pd, kot.SampleSet(wl.xs), rep_t.gamma_hat, q)
    out.update({"map_queries": q, "map_u": u, "map_t": tmap})
    # first iteration at which tol 1e-6 is hit, for the ±2 comparison
    hit = np.nonzero(np.array([t.res_accepted for t in rep_t.trace]) <= 1e-6)[0]
    out["tight_first_1e6"] = np.int64(hit[0] + 1 if hit.size else -1)
    np.savez_compressed(os.path.join(HERE, "cfg1.npz"), **out)
    print("cfg1: paper res@40", rep.trace[-1].res_accepted, "tight iters", rep_t.iterations,
          "first<=1e-6", out["tight_first_1e6"])


def gen_small():
    """Reference test-suite fixtures + KATs (pkg/tests/*) with reference outputs."""
    out = {}
    # scalar KKT fixtures (conftest.py:34-47)
    for name, z in (("interior", 1.0), ("active", -4.0)):
        pd = kprob.ProblemData(q_mat=[[2.0]], z=[z], q_sq=0.0, chol_upper=[[1.0]], lambda1=1.0, lambda2=0.5)
        rep = ksol.solve(pd, ksol.SolverConfig(residual_tol=1e-12, max_iter=100))
        out[f"scalar_{name}_gamma"] = rep.gamma_hat
        out[f"scalar_{name}_x"] = rep.x_hat
        out[f"scalar_{name}_iters"] = np.int64(rep.iterations)
        out[f"scalar_{name}_res"] = np.float64(rep.residual_norm)
    # random_problem instances: short solves + Newton direction vs dense Lemma-1 check
    for seed, n in ((0, 5), (1, 8), (2, 12)):
        pd = random_problem(seed, n=n)
        rep = ksol.solve(pd, ksol.SolverConfig(residual_tol=1e-10, max_iter=200))
        p = f"rand{seed}_"
        out.update(_pd_arrays(pd, p))
        out[p + "gamma"] = rep.gamma_hat
        out[p + "x"] = rep.x_hat
        out[p + "iters"] = np.int64(rep.iterations)
        out[p + "res"] = np.float64(rep.residual_norm)
        out.update(_trace_arrays(rep.trace, p + "tr_"))
    # eigen / eliminator inputs with controlled sign counts (test_psdcone.py:160-179)
    for n_pos in (0, 1, 3, 5, 6):
        rng = np.random.default_rng(100 + n_pos)
        zz = symmetric_with_signs(rng, 6, n_pos) if 0 < n_pos < 6 else (np.eye(6) if n_pos == 6 else -np.eye(6))
        s = rng.standard_normal((6, 6))
        s = 0.5 * (s + s.T)
        dc = klin.sym_eig(zz)
        c = kpsd.proj_jacobian_coeffs(dc)
        out[f"sign{n_pos}_z"] = zz
        out[f"sign{n_pos}_s"] = s
        out[f"sign{n_pos}_eigvals"] = dc.eigvals
        out[f"sign{n_pos}_proj"] = kpsd.proj_from_decomp(dc)
        out[f"sign{n_pos}_mz"] = kpsd.apply_proj_jacobian(c, s)
        for mu in (0.03, 1.0, 17.0):
            out[f"sign{n_pos}_elim_{mu}"] = kpsd.apply_eliminator(kpsd.make_eliminator(c, mu), s)
    # Cholesky KATs (test_linalg.py:47-78)
    v = np.array([[1.0, 2.0, 3.0], [1.0, 2.0, 3.0], [0.5, 0.1, -1.0]])
    f = klin.cholesky_psd(v @ v.T)
    out["chol_rankdef_in"] = v @ v.T
    out["chol_rankdef_r"] = f.upper
    out["chol_rankdef_jitter"] = np.float64(f.jitter_applied)
    np.savez_compressed(os.path.join(HERE, "small.npz"), **out)
    print("small fixtures written")


def gen_api():
    """Reference outputs for the rest of the public surface (kernels, datagen, psdcone decomposition
    API, apply_jacobian / criterion values, cg_solve, solve_pure_eg, distinct-bandwidth assemble)."""
    from kot import datagen as kdat
    from kot import kernels as kker
    out = {}
    # datagen (host input generation, datagen.py:49-132)
    out["mix_points"] = kot.sample_mixture(kdat.default_mixture(3, 4, 7), 50).points
    fp = kot.sobol_points(6, 37, -1.0, 1.0)
    out["sobol_xt"], out["sobol_yt"] = fp.x_tilde, fp.y_tilde
    out["sobol_nat"] = kdat.sobol_natural(5, 3, 20)
    # kernels (kernels.py:54-94)
    rng = np.random.default_rng(99)
    a, b = rng.uniform(-1, 1, (40, 3)), rng.uniform(-1, 1, (25, 3))
    spec = kker.KernelSpec(0.3, 3)
    out.update({"k_a": a, "k_b": b, "k_bw": np.float64(0.3), "k_rect": kker.gram_matrix(spec, a, b),
                "k_square": kker.gram_matrix(spec, a),
                "k_mean": kker.mean_embedding(spec, kot.SampleSet(a), b),
                "k_mean_at": np.float64(kker.mean_embedding_at(spec, kot.SampleSet(a), b[3])),
                "k_norm": np.float64(kker.embedding_norm_sq(spec, kot.SampleSet(a))),
                "k_eval": np.float64(kker.kernel_eval(spec, a[0], b[0]))})
    # assemble with three different bandwidths (problem.py:135-169)
    wl = configs.config1()
    sx, sy, sxy = kker.KernelSpec(0.25, 2), kker.KernelSpec(0.4, 2), kker.KernelSpec(0.6, 4)
    pd3 = kprob.assemble(kot.SampleSet(wl.xs), kot.SampleSet(wl.ys), kprob.FillingPoints(wl.xt, wl.yt),
                         wl.lambda1, wl.lambda2, sx, sy, sxy)
    out.update(_pd_arrays(pd3, "bw3_"))
    # operators at cfg1's replay state 10 through the decomposition API
    sx, sy, sxy = kprob.build_kernel_specs(wl.d, wl.bandwidth_sq)
    pd = kprob.assemble(kot.SampleSet(wl.xs), kot.SampleSet(wl.ys), kprob.FillingPoints(wl.xt, wl.yt),
                        wl.lambda1, wl.lambda2, sx, sy, sxy)
    cfg1 = dict(np.load(os.path.join(HERE, "cfg1.npz")))
    w = kprob.IteratePair(cfg1["op_g"], cfg1["op_x"])
    r, dc = kprob.residual_parts(pd, w)
    ctx = knew.newton_context(dc, r.norm(), float(cfg1["op_theta"]))
    dw = kprob.IteratePair(cfg1["op_dir_dg"], cfg1["op_dir_dx"])
    jd = kprob.apply_jacobian(pd, ctx.coeffs, ctx.mu, dw)
    out.update({"jac_top": jd.gamma, "jac_bottom": jd.x_mat,
                "crit_lhs": np.float64((jd + r).norm()),
                "crit_rhs": np.float64(0.5 * min(1.0, 0.1 * r.norm() * dw.norm())),
                "grad": kprob.objective_grad(pd, cfg1["op_g"]),
                "grad_dir": kprob.objective_grad_dir(pd, cfg1["op_v"]),
                "cmat": kprob.constraint_matrix(pd, cfg1["op_g"])})
    st = knew.newton_direction(pd, r, ctx, knew.NewtonConfig(cg_tol=1e-13, cg_max=3000, cg_restarts=0))
    out.update({"dirc_dg": st.dw.gamma, "dirc_dx": st.dw.x_mat, "dirc_rhs": np.float64(st.crit_rhs)})
    # cg_solve (linalg.py:117-162): the middle operator and a plain SPD matrix
    x, it, res = klin.cg_solve(knew.middle_operator(pd, ctx.eliminator, ctx.mu), cfg1["op_v"], 1e-12, 500)
    out.update({"cgm_x": x, "cgm_iters": np.int64(it), "cgm_res": np.float64(res)})
    m = rng.standard_normal((30, 30))
    spd = m @ m.T / 30 + 0.1 * np.eye(30)
    rhs = rng.standard_normal(30)
    x, it, res = klin.cg_solve(lambda v: spd @ v, rhs, 1e-10, 200)
    out.update({"cg_a": spd, "cg_b": rhs, "cg_x": x, "cg_iters": np.int64(it), "cg_res": np.float64(res)})
    # solve_pure_eg (solver.py:236-289)
    step = float(cfg1["eg_stepsize"])
    rep = ksol.solve_pure_eg(pd, ksol.SolverConfig(eg=keg.EgConfig(stepsize=step), residual_tol=1e-12, max_iter=30))
    out.update({"peg_gamma": rep.gamma_hat, "peg_x": rep.x_hat, "peg_iters": np.int64(rep.iterations),
                "peg_res": np.array([t.res_accepted for t in rep.trace])})
    np.savez_compressed(os.path.join(HERE, "api.npz"), **out)
    print("api fixtures written")


if __name__ == "__main__":
    which = sys.argv[1:] or ["small", "cfg1", "api"]
    if "small" in which:
        gen_small()
    if "cfg1" in which:
        gen_cfg1()
    if "api" in which:
        gen_api()
