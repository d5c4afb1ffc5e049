"""Batched independent OT problems (BASELINE config 5) sharded across GPUs.

SURVEY.md §8(e): the problems are independent, so they are partitioned over
the ranks with no data-path collective.  σ = [0.5, 1, 1.5, 2][s % 4] drives the
iteration count, and plain round-robin over 4 or 8 ranks would give each rank
a single σ group, so every σ group is dealt out across the ranks separately
(member j of group g → rank (j + g) mod world).  Each rank runs ``concurrency`` solves at
once on its GPU (one host thread and one CUDA stream per problem: every
eigensolve is latency-bound, so concurrent problems fill the SMs), then the
fixed-size result records are gathered to rank 0 with ``torch.distributed``
(NCCL over NVLink on the GPU box, gloo in the CPU tests).

Record layout (float64): [seed, iterations, converged, residual_norm,
ot_estimate, objective, total_ms, γ̂_0 … γ̂_{ℓ−1}].
"""

from __future__ import annotations

import threading
import time
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np

HEADER = 7


@dataclass(frozen=True)
class BatchResult:
    seed: int
    iterations: int
    converged: bool
    residual_norm: float
    ot_estimate: float
    objective: float
    total_ms: float
    gamma_hat: np.ndarray


def shard(seeds: Sequence[int], world: int, rank: int, groups: int = 4) -> list[int]:
    """Per-σ-group round-robin: every rank gets an equal share (±1) of every σ group."""
    seen: dict[int, int] = {}
    mine = []
    for s in seeds:
        g = s % groups
        j = seen.get(g, 0)
        seen[g] = j + 1
        if (j + g) % world == rank:
            mine.append(s)
    return mine


def pack(res: BatchResult, l: int) -> np.ndarray:  # noqa: E741
    rec = np.full(HEADER + l, np.nan)
    rec[:HEADER] = [res.seed, res.iterations, float(res.converged), res.residual_norm, res.ot_estimate,
                    res.objective, res.total_ms]
    rec[HEADER:HEADER + res.gamma_hat.size] = res.gamma_hat
    return rec


def unpack(rec: np.ndarray) -> BatchResult:
    return BatchResult(int(rec[0]), int(rec[1]), bool(rec[2]), float(rec[3]), float(rec[4]), float(rec[5]),
                       float(rec[6]), rec[HEADER:].copy())


def gpu_solve_member(seed: int, cfg_kwargs: dict, device: int) -> BatchResult:
    """Assemble + solve one config-5 member on ``device`` (the GPU path)."""
    import paper_2310_14087_b200 as K
    from paper_2310_14087_b200 import configs

    wl = configs.config5_member(seed)
    sx, sy, sxy = K.build_kernel_specs(wl.d, wl.bandwidth_sq)
    t0 = time.perf_counter()
    pd = K.assemble(K.SampleSet(wl.xs), K.SampleSet(wl.ys), K.FillingPoints(wl.xt, wl.yt), wl.lambda1,
                    wl.lambda2, sx, sy, sxy, device=device)
    step = configs.eg_stepsize(pd.q_mat, pd.pair_gram(), pd.lambda2)
    newton = K.NewtonConfig(**configs.PROFILES[cfg_kwargs.get("profile", "tight")])
    cfg = K.SolverConfig(newton=newton, eg=K.EgConfig(step), residual_tol=cfg_kwargs.get("residual_tol", 1e-6),
                         max_iter=cfg_kwargs.get("max_iter", 500))
    from paper_2310_14087_b200.solver import _run
    rep = _run(pd, cfg, None, False, want_x=False)
    obj = K.objective(pd, rep.gamma_hat)
    return BatchResult(seed, rep.iterations, rep.termination == "converged", rep.residual_norm,
                       float(rep.ot_estimate), obj, (time.perf_counter() - t0) * 1e3, rep.gamma_hat)


def run_local(seeds: Sequence[int], solve_fn: Callable[[int], BatchResult], concurrency: int = 4
              ) -> list[BatchResult]:
    """Solve ``seeds`` with up to ``concurrency`` concurrent workers (threads; the C ABI releases the GIL)."""
    out: dict[int, BatchResult] = {}
    errors: list[BaseException] = []
    queue = list(seeds)
    lock = threading.Lock()

    def worker():
        while True:
            with lock:
                if not queue or errors:
                    return
                s = queue.pop(0)
            try:
                r = solve_fn(s)
            except BaseException as exc:  # surfaced after join
                with lock:
                    errors.append(exc)
                return
            with lock:
                out[s] = r

    threads = [threading.Thread(target=worker) for _ in range(max(1, min(concurrency, len(seeds))))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    return [out[s] for s in seeds]


def run_and_gather(seeds: Sequence[int], solve_fn: Callable[[int], BatchResult], concurrency: int, l: int,  # noqa: E741
                   world: int, rank: int, device=None) -> list[BatchResult] | None:
    """run_local on this rank's seeds, then gather_to_root — a local failure still joins the collective."""
    res: list[BatchResult] = []
    err: BaseException | None = None
    try:
        res = run_local(seeds, solve_fn, concurrency)
    except Exception as e:  # noqa: BLE001 — re-raised on every rank by gather_to_root
        err = e
    return gather_to_root(res, l, world, rank, device=device, error=err)


def gather_to_root(results: list[BatchResult], l: int, world: int, rank: int, device=None,  # noqa: E741
                   error: BaseException | None = None) -> list[BatchResult] | None:
    """Gather fixed-size records to rank 0 (one all_gather of a padded [max_per_rank, HEADER+ℓ] block).

    Every rank takes part even when its own solves failed (``error``): the failure is all-reduced
    first and then raised on every rank, so no rank is left waiting in the collective."""
    recs = np.stack([pack(r, l) for r in results]) if results else np.zeros((0, HEADER + l))
    if world == 1:
        if error is not None:
            raise error
        return [unpack(r) for r in recs]
    import torch
    import torch.distributed as dist

    # [records on this rank, failed] — per-rank shard sizes differ by the σ-group dealing
    cnt = torch.tensor([recs.shape[0], 1 if error is not None else 0], dtype=torch.int64, device=device)
    dist.all_reduce(cnt, op=dist.ReduceOp.MAX)
    if int(cnt[1].item()):
        if error is not None:
            raise error
        raise RuntimeError("a batch member failed on another rank")
    per = max(int(cnt[0].item()), 1)
    buf = np.full((per, HEADER + l), np.nan)
    buf[:recs.shape[0]] = recs
    t = torch.from_numpy(buf)
    if device is not None:
        t = t.to(device)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    if rank != 0:
        return None
    rows = [p.cpu().numpy() for p in parts]
    allrecs = [unpack(r) for blk in rows for r in blk if not np.isnan(r[0])]
    return sorted(allrecs, key=lambda r: r.seed)
