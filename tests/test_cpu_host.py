"""CPU-only tests: the C-ABI library loads and exports the header's symbols, host-side logic
(configs, validation, damping rule, batch sharding/packing) and the multi-process gather
path (gloo, world_size 2).  No CUDA compute runs here."""

import os
import re
import socket

import numpy as np
import pytest

from oracle import kot_port as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ---------------------------------------------------------------- ABI

def header_functions():
    src = open(os.path.join(ROOT, "include", "kotgpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(kot_[a-z0-9_]+)\s*\(", src))
    names -= {"kot_iter_cb"}
    return sorted(names)


def test_library_exports_every_declared_symbol():
    from paper_2310_14087_b200 import _lib
    lib = _lib.lib()
    declared = header_functions()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(lib, name), name
    # every declared entry point is bound with a signature by the Python layer (debug hooks excepted)
    bound = set(_lib.exported_symbols())
    missing = [n for n in declared if n not in bound]
    assert not missing, missing


def test_debug_hook_exported():
    from paper_2310_14087_b200 import _lib
    assert hasattr(_lib.lib(), "kot_debug_sytrd_timing")


def test_mid_kernel_capacity_rule():
    """Order of the trailing block the grid-resident sytrd kernel keeps in shared memory: (rows + 4
    vectors) × 8 B per CTA, at most 18 rows per CTA (csrc/sytrd_mid.cuh: mid_capacity; host-only hook)."""
    from paper_2310_14087_b200 import _lib
    f = _lib.lib().kot_debug_mid_capacity
    smem = 228352  # 227 KB opt-in maximum minus the kernel's 4 KB of static shared memory
    assert f(148, smem) == 1776 and f(96, smem) == 1440  # ℓ = 2000 alone / beside an EG pipeline
    for g in (1, 16, 52, 96, 148):
        m0 = f(g, smem)
        rpc, ld = -(-m0 // g), m0 + (m0 & 1)
        assert rpc <= 18 and (rpc + 4) * ld * 8 <= smem
        m1 = m0 + 1  # one more column does not fit
        rpc1, ld1 = -(-m1 // g), m1 + (m1 & 1)
        assert rpc1 > 18 or (rpc1 + 4) * ld1 * 8 > smem or m1 > 2048
    assert [f(g, smem) for g in (16, 24, 52, 96, 148)] == sorted(f(g, smem) for g in (16, 24, 52, 96, 148))
    assert f(148, 0) == 0 and f(0, smem) == -1


@pytest.mark.timeout(120)
def test_cooperative_gate_exclusive_windows():
    """The gate that admits cooperative eigensolver grids (csrc/eig.cu: CoopGate), host logic only: three
    background panel loops that yield between panels and one foreground thread opening exclusive
    windows (the mid kernel's launch protocol).  No background panel may be in flight inside a window,
    nobody deadlocks, and the slot accounting returns to zero."""
    from paper_2310_14087_b200 import _lib
    windows = _lib.lib().kot_debug_gate_selftest(3, 400)
    assert windows > 10, windows


def test_ctypes_struct_layouts_match_c(tmp_path):
    """Compile a probe against include/kotgpu.h with gcc and compare sizes/offsets with ctypes."""
    import ctypes as C
    import shutil
    import subprocess
    from paper_2310_14087_b200 import _lib
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    src = tmp_path / "probe.c"
    src.write_text(
        f'#include "{ROOT}/include/kotgpu.h"\n#include <stdio.h>\n#include <stddef.h>\n'
        'int main(){printf("%zu %zu %zu %zu %zu %zu %zu %zu\\n", sizeof(kot_solver_cfg),'
        ' offsetof(kot_solver_cfg, cg_tol), offsetof(kot_solver_cfg, eg_stepsize),'
        ' offsetof(kot_solver_cfg, safeguard_every), sizeof(kot_iter_record),'
        ' offsetof(kot_iter_record, step_ms), sizeof(kot_report), sizeof(kot_prof_entry));return 0;}\n')
    exe = tmp_path / "probe"
    subprocess.run(["gcc", str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    want = [C.sizeof(_lib.SolverCfgC), _lib.SolverCfgC.cg_tol.offset, _lib.SolverCfgC.eg_stepsize.offset,
            _lib.SolverCfgC.safeguard_every.offset, C.sizeof(_lib.IterRecordC), _lib.IterRecordC.step_ms.offset,
            C.sizeof(_lib.ReportC), C.sizeof(_lib.ProfEntryC)]
    assert got == want


def test_no_cpu_fallback_without_gpu():
    """The product path fails loudly when no GPU is present (no silent NumPy fallback)."""
    import paper_2310_14087_b200 as K
    from paper_2310_14087_b200 import _lib
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(_lib.CudaError):
        K.linalg.sym_eig(np.eye(3))
    pd = K.ProblemData(q_mat=[[2.0]], z=[1.0], q_sq=0.0, chol_upper=[[1.0]], lambda1=1.0, lambda2=0.5)
    with pytest.raises(_lib.CudaError):
        K.solve(pd)


# ------------------------------------------------------- host-side API

def test_dataclass_validation_mirrors_reference():
    import paper_2310_14087_b200 as K
    with pytest.raises(ValueError):
        K.KernelSpec(0.0, 2)
    with pytest.raises(ValueError):
        K.KernelSpec(1.0, 2, family="laplace")
    with pytest.raises(ValueError):
        K.SampleSet(np.ones(3))
    with pytest.raises(ValueError):
        K.SampleSet(np.array([[np.nan, 1.0]]))
    with pytest.raises(ValueError):
        K.FillingPoints(np.ones((3, 2)), np.ones((2, 2)))
    with pytest.raises(ValueError):
        K.ProblemData(q_mat=np.eye(2), z=np.zeros(3), q_sq=0.0, chol_upper=np.eye(2), lambda1=1.0, lambda2=1.0)
    with pytest.raises(ValueError):
        K.ProblemData(q_mat=np.eye(2), z=np.zeros(2), q_sq=0.0, chol_upper=np.eye(2), lambda1=0.0, lambda2=1.0)
    for bad in (dict(tau=1.0), dict(alpha1=2.0, alpha2=1.0), dict(beta0=1.5), dict(theta_min=0.0), dict(cg_max=0)):
        with pytest.raises(ValueError):
            K.NewtonConfig(**bad)
    with pytest.raises(ValueError):
        K.EgConfig(stepsize=0.0)
    for bad in (dict(residual_tol=0.0), dict(max_iter=0), dict(safeguard_every=0)):
        with pytest.raises(ValueError):
            K.SolverConfig(**bad)
    # q_mat is symmetrised on construction (problem.py:112)
    pd = K.ProblemData(q_mat=[[1.0, 2.0], [0.0, 1.0]], z=[0.0, 0.0], q_sq=0.0, chol_upper=np.eye(2),
                       lambda1=1.0, lambda2=1.0)
    assert np.array_equal(pd.q_mat, [[1.0, 1.0], [1.0, 1.0]])


def test_iterate_pair_algebra():
    from paper_2310_14087_b200.problem import IteratePair, zero_pair
    a = IteratePair(np.array([3.0, 4.0]), np.array([[0.0, 0.0], [0.0, 12.0]]))
    assert a.norm() == pytest.approx(5.0 + 12.0)  # problem.py:56-57: a sum of norms
    assert a.dot(a) == pytest.approx(25.0 + 144.0)
    b = zero_pair(2)
    assert (a + b).norm() == a.norm() and (2 * a).norm() == 2 * a.norm()
    assert a.is_finite() and not IteratePair(np.array([np.inf]), np.zeros((1, 1))).is_finite()


def test_theta_update_matches_oracle():
    from paper_2310_14087_b200 import newton
    rng = np.random.default_rng(0)
    cfg_g = newton.NewtonConfig()
    cfg_o = O.NewtonCfg()
    for _ in range(500):
        theta = float(np.exp(rng.uniform(-12, 12)))
        rho = float(rng.normal() * 10 ** rng.uniform(-8, 2))
        dw2 = float(10 ** rng.uniform(-6, 4))
        assert newton.theta_update(theta, rho, dw2, cfg_g) == O.theta_update(theta, rho, dw2, cfg_o)


def test_solver_cfg_struct_roundtrip():
    import paper_2310_14087_b200 as K
    c = K.SolverConfig(newton=K.NewtonConfig(alpha1=1e-8, cg_tol=1e-9), eg=K.EgConfig(0.25), residual_tol=1e-7,
                       max_iter=77, safeguard_every=3).to_c()
    assert (c.alpha1, c.cg_tol, c.has_cg_tol, c.eg_stepsize, c.residual_tol, c.max_iter, c.safeguard_every) == (
        1e-8, 1e-9, 1, 0.25, 1e-7, 77, 3)
    assert K.SolverConfig().to_c().has_cg_tol == 0


def test_configs_are_seeded_and_shaped():
    from paper_2310_14087_b200 import configs
    a, b = configs.config2(), configs.config2()
    assert np.array_equal(a.xs, b.xs) and a.xs.shape == (500, 5) and a.xt.shape == (500, 5)
    assert np.all(np.abs(a.xs) <= 1.0) and np.all(np.abs(a.ys) <= 1.0)
    c3 = configs.config3(n=300)
    assert c3.xs.shape == (300, 10) and np.all(np.linalg.norm(c3.xs, axis=1) <= 1.0 + 1e-15)
    assert c3.bandwidth_sq == 2.25 and c3.lambda2 == 1.0 / 300
    m = configs.config5_member(6)
    assert m.bandwidth_sq == pytest.approx(1.5 ** 2) and m.xs.shape == (1000, 10)
    c4 = configs.config4(n=64)
    assert c4.xs.shape == (64, 64) and np.allclose(np.linalg.norm(c4.xs, axis=1), 1.0)


def test_eg_stepsize_rule():
    from paper_2310_14087_b200 import configs
    q = np.array([[2.0, 0.0], [0.0, 2.0]])
    k = np.eye(2)
    s = configs.eg_stepsize(q, k, 0.5)
    assert s == pytest.approx(0.5 / (np.sqrt(8.0) / 1.0 + np.sqrt(2.0)))


# ------------------------------------------------------------- batches

def fake_result(seed, l=6):  # noqa: E741
    from paper_2310_14087_b200.batch import BatchResult
    return BatchResult(seed, seed % 7 + 1, seed % 2 == 0, 1e-7 * (seed + 1), float(seed), -float(seed), 1.0,
                       np.arange(l, dtype=float) + seed)


def test_shard_spreads_sigma_groups():
    from paper_2310_14087_b200.batch import shard
    seeds = list(range(512))
    for world in (1, 2, 4, 8):
        parts = [shard(seeds, world, r) for r in range(world)]
        assert sorted(sum(parts, [])) == seeds
        for p in parts:
            counts = np.bincount(np.array(p) % 4, minlength=4)
            assert counts.max() - counts.min() <= 1


def test_pack_unpack_and_local_runner():
    from paper_2310_14087_b200.batch import pack, run_local, unpack
    r = fake_result(5)
    u = unpack(pack(r, 6))
    assert u.seed == 5 and u.iterations == r.iterations and np.array_equal(u.gamma_hat, r.gamma_hat)
    out = run_local(list(range(10)), fake_result, concurrency=3)
    assert [o.seed for o in out] == list(range(10))

    def boom(s):
        raise RuntimeError("x")
    with pytest.raises(RuntimeError):
        run_local([1, 2], boom, concurrency=2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gather_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2310_14087_b200.batch import gather_to_root, run_local, shard
    seeds = list(range(11))
    mine = shard(seeds, world, rank)
    res = run_local(mine, fake_result, concurrency=2)
    allr = gather_to_root(res, 6, world, rank)
    if rank == 0:
        q.put([(r.seed, r.iterations, r.gamma_hat.tolist()) for r in allr])
    dist.barrier()
    dist.destroy_process_group()


def test_multiprocess_gather_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [g[0] for g in got] == list(range(11))
    for seed, it, gam in got:
        ref = fake_result(seed)
        assert it == ref.iterations and np.array_equal(gam, ref.gamma_hat)


def _failing_gather_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2310_14087_b200.batch import run_and_gather, shard

    def solve(s):
        if rank == 1:
            raise FloatingPointError("member diverged")
        return fake_result(s)
    try:
        run_and_gather(shard(list(range(11)), world, rank), solve, 2, 6, world, rank)
        q.put((rank, "no error"))
    except FloatingPointError as e:
        q.put((rank, f"local: {e}"))
    except RuntimeError as e:
        q.put((rank, f"remote: {e}"))
    dist.destroy_process_group()


def test_multiprocess_gather_propagates_member_failure():
    """a rank whose member solve raises still joins the collective, and every rank raises
    (no rank is left blocked in all_gather)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_failing_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got[1] == "local: member diverged"
    assert got[0].startswith("remote:")


def _host_plane_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2310_14087_b200.rowshard import host_collective
    a = np.arange(6, dtype=float) * (rank + 1)
    host_collective(0, a, 0, rank, world)
    g = np.full(3 * world, -1.0)
    g[3 * rank:3 * rank + 3] = [10 * rank, 10 * rank + 1, 10 * rank + 2]
    host_collective(1, g, 3, rank, world)
    q.put((rank, a.tolist(), g.tolist()))
    dist.destroy_process_group()


def test_host_data_plane_collectives_gloo():
    """kot_problem_shard_host's two collectives (sum of T̃, gather of y) over a gloo group, in place on
    the library's staging buffer: identical on every rank."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_host_plane_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=120) for _ in range(3))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, a, g in got:
        assert a == (np.arange(6) * 6.0).tolist()
        assert g == [0, 1, 2, 10, 11, 12, 20, 21, 22]


# ------------------------------------------------------ row sharding (config 4)

def test_row_blocks_partition():
    from paper_2310_14087_b200.rowshard import row_block
    for n in (1, 7, 64, 8192, 8191):
        for world in (1, 2, 3, 8):
            blocks = [row_block(n, r, world) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            for (a0, a1), (b0, b1) in zip(blocks, blocks[1:]):
                assert a1 == b0 and a0 <= a1
            block = -(-n // world)
            assert all(r0 == min(n, g * block) for g, (r0, _) in enumerate(blocks))  # allgather layout
    with pytest.raises(ValueError):
        row_block(5, 2, 2)


@pytest.mark.parametrize("n_pos", [2, 9])
def test_row_block_decomposition_of_middle_operator(n_pos):
    """NumPy restatement of what each rank computes (shard.cu / ssn.cu middle_operator_fast):
    per-block coefficient-scaled partial T̃_g, summed (the all-reduce), then per-block rows of y
    (the all-gather) — equals the oracle's Φ∘𝒯∘Φ* middle operator."""
    from conftest import symmetric_with_signs
    from paper_2310_14087_b200.rowshard import row_block
    rng = np.random.default_rng(n_pos)
    n = 11
    a = rng.standard_normal((n, n))
    r = np.triu(a) + 3 * np.eye(n)
    q = a @ a.T + np.eye(n)
    po = O.Problem(q=q, z=rng.standard_normal(n), q_sq=1.0, r=r, l1=0.5, l2=0.4, embed=None)
    dc = O.sym_eig(symmetric_with_signs(rng, n, n_pos))
    mu = 0.3
    op = O.eliminator(dc, O.cross_coeffs(dc), mu)
    v = rng.standard_normal(n)
    ref = O.middle_operator(po, op, mu)(v) - (q @ v) / (2 * 0.4) - mu * v
    vals, p = dc.vals, dc.vecs
    k = int(np.sum(vals > 0))
    b = r @ p
    # coefficient matrix W in the eigenbasis (psdcone.py:113-121)
    w = np.zeros((n, n))
    for i in range(n):
        for j in range(n):
            if i < k and j < k:
                w[i, j] = 1.0 / mu
            elif (i < k) != (j < k):
                a_, b_ = (i, j) if i < k else (j, i)
                eta = vals[a_] / (vals[a_] - vals[b_])
                w[i, j] = eta / (mu + 1.0 - eta)
    for world in (1, 2, 4):
        t = sum(w * (b[r0:r1].T @ np.diag(v[r0:r1]) @ b[r0:r1])
                for r0, r1 in (row_block(n, g, world) for g in range(world)))
        y = np.empty(n)
        for g in range(world):
            r0, r1 = row_block(n, g, world)
            y[r0:r1] = np.einsum("ia,ab,ib->i", b[r0:r1], t, b[r0:r1])
        assert np.allclose(y, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


def _uid_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2310_14087_b200 import rowshard
    obj = [rowshard.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)  # what rowshard.shard_rows does before kot_problem_shard
    q.put((rank, obj[0], rowshard.row_block(8192, rank, world)))
    dist.barrier()
    dist.destroy_process_group()


def test_nccl_unique_id_broadcast_gloo():
    """Rank 0's 128-byte ncclUniqueId (libkotgpu dlopens NCCL; no GPU needed) reaches every rank."""
    from paper_2310_14087_b200 import rowshard
    try:
        rowshard.unique_id()
    except Exception as exc:  # libnccl absent in this environment
        pytest.skip(f"NCCL unavailable: {exc}")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_uid_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted([q.get(timeout=120) for _ in range(2)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len(got[0][1]) == 128 and got[0][1] == got[1][1]
    assert got[0][2] == (0, 4096) and got[1][2] == (4096, 8192)
