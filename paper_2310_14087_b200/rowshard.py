"""Sharding of the Newton-CG matvec across GPUs (BASELINE config 4, ℓ = 8192).

SURVEY.md §8(e).  The reference's middle operator (newton.py:70-95,
psdcone.py:113-121) applied through B = R·P in the split H form:

    Φ(𝒯[Φ*(v)])_i = (H v)_i/μ + 2 Σ_{a∈s, b∈s̄} B_ia B_ib ξ_ab C_ab,   C = B_sᵀ diag(v) B_s̄

Rank g takes a column range of the mixed-sign block (both DMMA GEMMs) and its two folded
row blocks (g and 2N−1−g of 2N) of the H / Q GEMVs; the partial y vectors are summed with
one all-reduce of ℓ doubles per matvec.  Once per Newton step every rank forms its folded
row blocks of B = R·P (equal shares of R's triangle) and two all-gathers complete B.
Everything else (eigensolve, Φ, EG, CG vectors) stays replicated, so every rank takes
identical control decisions and returns identical results.  ``row_block`` / ``shard_info``
report the contiguous block of the legacy "blocked" form (``kot_middle_operator(form=2)``).

The NCCL communicator is created by the library itself from an ncclUniqueId
that rank 0 draws and ``torch.distributed`` broadcasts (any process group,
gloo or nccl, can carry the 128 bytes).
"""

from __future__ import annotations

import ctypes as C

from . import _lib


def row_block(n: int, rank: int, world: int) -> tuple[int, int]:
    """Rows [r0, r1) owned by ``rank`` (shard.cu:problem_shard)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("invalid rank/world")
    block = -(-n // world)
    r0 = min(n, rank * block)
    return r0, min(n, r0 + block)


def unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _lib.check(_lib.lib().kot_nccl_unique_id(buf))
    return buf.raw


def shard_rows(pd, group=None, device: int | None = None) -> tuple[int, int]:
    """Collective: split ``pd``'s CG matvec over the ranks of ``group`` (torch.distributed).

    Returns this rank's row block.  With a world of one this is a no-op."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dp = pd.device_problem(device)
    if world == 1:
        _lib.check(_lib.lib().kot_problem_shard(dp.handle, None, 0, 1))
        return 0, pd.n
    obj = [unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    _lib.check(_lib.lib().kot_problem_shard(dp.handle, obj[0], rank, world))
    return shard_info(pd)[2:]


def host_collective(op: int, arr, block: int, rank: int, world: int, group=None) -> None:
    """The host data plane of kot_problem_shard_host on a float64 host array, in place.

    op 0: sum over the ranks of ``group``; op 1: all-gather of every rank's ``block`` values
    (rank g's at ``arr[g·block:(g+1)·block]``)."""
    import torch
    import torch.distributed as dist

    t = torch.from_numpy(arr)  # shares memory (the library's pinned staging buffer)
    if op == 0:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    elif op == 1:
        parts = [torch.empty(block, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, t[rank * block:(rank + 1) * block].clone(), group=group)
        t.copy_(torch.cat(parts))
    else:
        raise ValueError(f"unknown collective {op}")


def shard_rows_host(pd, group=None, device: int | None = None) -> tuple[int, int]:
    """Collective: the same row split as :func:`shard_rows`, with the two exchanges (sum of T̃,
    gather of y) carried by ``group``'s own collectives on host tensors (e.g. a gloo group) instead of
    NCCL — for ranks that share one GPU (tests) or hosts without NCCL.  Returns this rank's block."""
    import numpy as np
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dp = pd.device_problem(device)
    if world == 1:
        _lib.check(_lib.lib().kot_problem_shard(dp.handle, None, 0, 1))
        return 0, pd.n

    def comm(_user, op, buf, count, block, rk, wd):
        try:
            host_collective(op, np.ctypeslib.as_array(buf, shape=(count,)), block, rk, wd, group)
            return 0
        except Exception:  # reported as a status by the library
            return 1

    cb = _lib.CommFn(comm)
    dp._comm_cb = cb  # keep the trampoline alive as long as the device problem
    _lib.check(_lib.lib().kot_problem_shard_host(dp.handle, cb, None, rank, world))
    return shard_info(pd)[2:]


def shard_info(pd) -> tuple[int, int, int, int]:
    """(rank, world, r0, r1) of the device problem."""
    v = [C.c_int() for _ in range(4)]
    _lib.check(_lib.lib().kot_problem_shard_info(pd.device_problem().handle, *[C.byref(x) for x in v]))
    return tuple(x.value for x in v)


def emulate_shards(pd, world: int) -> None:
    """Single-device test hook: compute the ``world`` row blocks in turn (no NCCL)."""
    _lib.check(_lib.lib().kot_problem_shard(pd.device_problem().handle, None, 0, int(world)))
