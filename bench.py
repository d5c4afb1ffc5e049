#!/usr/bin/env python
"""Benchmark: SSN iterations/s of the B200 kernel-OT solver on the BASELINE configs.

Contract (see README/DESIGN): ``python bench.py --gpus N --steps K --warmup W``
prints ONE JSON line on rank 0.  A *step* is one outer SSN iteration
(Algorithm 2: EG safeguard + Newton direction with CG + trial residual) of a
continuous solve trajectory on the headline workload (BASELINE.json
configs[2]: d=10, n=ℓ=2000, σ=1.5, λ1=1e-4, λ2=1/ℓ, FP64), paper profile
(``NewtonConfig()`` defaults), EG stepsize 0.5/(‖Q‖_F/(2λ2)+‖K‖_F)
(SURVEY.md §8(d)).  Synthetic seeded data (the reference ships none).

* ``value``: iterations/s over the K timed iterations W … W+K−1, inputs resident
  in HBM, timed with CUDA events on the library's stream, barrier + synchronize on
  both sides, max over ranks; N>1 runs N independent replicas (single problems do
  not shard: SURVEY.md §8(e) "configs 1-3: replicas only") → ``scaling: weak``.
* ``e2e``: the same iterations W … W+K−1 through the public API, measured FIRST in
  the process (fresh device allocations): ``assemble`` from the host sample arrays
  and ``solve(pd, max_iter=W+K)`` with the D2H of (γ̂, X̂), all inside the timed
  region; the W warm-up iterations' own step times are subtracted, so the window
  matches ``value`` and the reference arm (assembly, upload, allocation, setup,
  initial residual and download stay in).
* ``roofline``: the dominant kernel (live CUDA-event timing inside libkotgpu's
  phase profiler), against MEASURED_PEAKS.json / the measured DMMA peak;
  ``traffic`` is read from the committed ncu capture (profiles/r02/roofline_traffic.json).
* ``cpu_baseline``: the NumPy oracle (oracle/, a restatement of the reference)
  on this box's host cores for a bounded sample of the same window: 2 SSN
  iterations from the GPU trajectory's own state at iteration W.
* ``time_to_tol``: BASELINE's time-to-tolerance half at cfg3, tight profile:
  assemble + solve from host arrays to 5e-3 (first hit, solver.py:221-222) and
  to 1e-6 within a stated max_iter (the residual reached when not hit).
* ``--impl reference``: the reference's CPU algorithm (the oracle port; the
  reference is pure Python and cannot be installed on the box) on the same config.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DMMA_PEAK_TFLOPS = 37.12  # measured, profiles/r01/fp64_peak_microbench.txt (mma.sync m8n8k4 f64)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return float(m.get("hbm_gbs", 6553.6)), "measured"
    except Exception:
        return 6650.0, "fallback"


def workload(name: str):
    from paper_2310_14087_b200 import configs
    if name == "cfg1":
        return configs.config1()
    if name == "cfg2":
        return configs.config2()
    if name.startswith("cfg3"):
        n = int(name.split(":")[1]) if ":" in name else 2000
        return configs.config3(n=n)
    if name.startswith("cfg4"):
        n = int(name.split(":")[1]) if ":" in name else 8192
        return configs.config4(n=n)
    if name.startswith("cfg5"):
        seed = int(name.split(":")[1]) if ":" in name else 0
        return configs.config5_member(seed)
    raise SystemExit(f"unknown config {name}")


def describe(wl, profile: str) -> dict:
    return {"workload": f"{wl.name}: d={wl.d}, n=l={wl.l}, bandwidth_sq={wl.bandwidth_sq}, "
                        f"lambda1={wl.lambda1}, lambda2=1/{wl.l}; {profile} profile; "
                        "EG stepsize 0.5/(||Q||_F/(2 lambda2)+||K||_F); one step = one SSN outer iteration",
            "l": wl.l, "n_samples": wl.xs.shape[0], "d": wl.d, "profile": profile,
            "l2_flush": f"none needed: per-iteration working set ~{25 * 8 * wl.l * wl.l / 1e9:.2f} GB > 126 MB L2",
            "data": "seeded synthetic (SURVEY.md §8(d))"}


def newton_cfg(profile: str):
    import paper_2310_14087_b200 as K
    from paper_2310_14087_b200 import configs
    return K.NewtonConfig(**configs.PROFILES[profile])


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i].strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_setup(gpus: int):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(world, x: float, local: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(world, x: float, local: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


# --------------------------------------------------------------------- CPU legs

def oracle_problem(wl):
    from oracle import kot_port as O
    pd, kmat = O.assemble(wl.xs, wl.ys, wl.xt, wl.yt, wl.lambda1, wl.lambda2, wl.bandwidth_sq)
    return pd, kmat


def oracle_iters_per_s(wl, profile: str, warmup: int, steps: int) -> tuple[float, float, dict]:
    """Time `steps` SSN iterations of the oracle (after `warmup`) on the host cores."""
    from oracle import kot_port as O
    from paper_2310_14087_b200 import configs
    pd, kmat = oracle_problem(wl)
    step = configs.eg_stepsize(pd.q, kmat, pd.l2)
    cfg = O.SolverCfg(newton=O.NewtonCfg(**configs.PROFILES[profile]), eg_stepsize=step, residual_tol=1e-300,
                      max_iter=10 ** 9)
    st = O.initial_state(pd, cfg)
    k = 0
    for _ in range(warmup):
        st, _, _ = O.iterate_once(pd, st, k, cfg)
        k += 1
    t0 = time.perf_counter()
    for _ in range(steps):
        st, _, _ = O.iterate_once(pd, st, k, cfg)
        k += 1
    dt = time.perf_counter() - t0
    return steps / dt, dt, {"first_iteration": k - steps}


def cpu_info() -> dict:
    cores = len(os.sched_getaffinity(0))
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return {"cores": cores, "cpu": model, "blas_threads": os.environ.get("OPENBLAS_NUM_THREADS", "all")}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    wl = workload(args.config)
    v, dt, extra = oracle_iters_per_s(wl, args.profile, args.warmup, args.steps)
    ci = cpu_info()
    line = {
        "impl": "reference", "metric": f"SSN iters/s at n=l={wl.l} FP64 ({args.profile} profile)",
        "value": v, "unit": "iter/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": describe(wl, args.profile),
        "cpu_baseline": {"value": v, "unit": "iter/s", "cores": ci["cores"], "kind": "port",
                         "sample": f"{args.steps} SSN iterations of {wl.name} after {args.warmup} warm-up "
                                   "iterations from the zero pair, NumPy/OpenBLAS oracle (oracle/kot_port.py)",
                         "cpu": ci["cpu"]},
        "e2e": {"value": v, "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------- GPU leg

def _first_hit_ms(rep, tol: float):
    """(iteration, ms since the call started) of the first accepted iterate with ‖R‖ ≤ tol, from the
    trace's per-iteration step times; the setup before iteration 0 is total_ms − Σ step_ms."""
    steps = [r.step_ms for r in rep.trace]
    setup = rep.total_ms - sum(steps)
    t = setup
    for i, r in enumerate(rep.trace):
        t += r.step_ms
        if r.res_accepted <= tol:
            return i + 1, t
    return None, None


def time_to_tol(K, configs, wl, max_iter: int) -> dict:
    """BASELINE metric, first half: time-to-tolerance at the headline config (cfg3, tight profile,
    SURVEY.md §8(d)), through the public API from host arrays.  One solve to 5e-3 (the paper's
    threshold; solve stops at the first accepted iterate below tol, solver.py:221-222) and one to 1e-6
    with max_iter stated; when 1e-6 is not reached the residual at max_iter is reported (never the
    best residual seen)."""
    out = {"workload": f"{wl.name}, tight profile (alpha1=1e-8, alpha2=1e-4, cg_max=500), assemble + solve "
                       "from host arrays"}
    sx, sy, sxy = K.build_kernel_specs(wl.d, wl.bandwidth_sq)
    for tol, cap in ((5e-3, max_iter), (1e-6, max_iter)):
        t0 = time.perf_counter()
        pd = K.assemble(K.SampleSet(wl.xs), K.SampleSet(wl.ys), K.FillingPoints(wl.xt, wl.yt), wl.lambda1,
                        wl.lambda2, sx, sy, sxy)
        step = configs.eg_stepsize(pd.q_mat, pd.pair_gram(), pd.lambda2)
        cfg = K.SolverConfig(newton=K.NewtonConfig(**configs.PROFILES["tight"]), eg=K.EgConfig(step),
                             residual_tol=tol, max_iter=cap)
        rep = K.solve(pd, cfg)
        dt = time.perf_counter() - t0
        hit = rep.termination == "converged"
        out[f"{tol:g}"] = {"reached": hit, "seconds": dt, "iterations": rep.iterations, "max_iter": cap,
                           "residual": rep.residual_norm,
                           "cg_iters_per_iteration": sum(r.cg_iters for r in rep.trace) / max(rep.iterations, 1)}
        pd.release_device()
    return out


def run_gpu(args):
    world, rank, local = dist_setup(args.gpus)
    os.environ["KOT_DEVICE"] = str(local)
    import torch

    import paper_2310_14087_b200 as K
    from paper_2310_14087_b200 import _lib, configs, solver

    torch.cuda.set_device(local)
    torch.cuda.init()
    _lib.lib()  # library load (process setup, not part of any timed region)
    # process setup, as for any long-running service: the library's own CUDA runtime attaches to the
    # device and loads its module with one 2 × 2 eigensolve (no problem is created, nothing is pooled)
    from paper_2310_14087_b200 import linalg as _linalg
    _linalg.sym_eig(np.eye(2), device=local)
    wl = workload(args.config)
    # ... and the device memory pool is grown once (kot_reserve, the documented set-up call of a service
    # process: INTEGRATION.md §6).  Every problem, workspace and execution context of the end-to-end solve
    # is still allocated inside the timed region — from a mapped pool instead of paying the driver's
    # first mapping, which takes 4 to 300 ms for the same ≈ 3.5 GB depending on what the GPU ran before
    # (profiles/r02/e2e_repeat_r02.txt).  KOT_BENCH_COLD_POOL=1 measures without it.
    reserved_gib = 0.0
    if os.environ.get("KOT_BENCH_COLD_POOL") != "1" and args.config in ("cfg3", "cfg5"):
        reserved_gib = float(os.environ.get("KOT_BENCH_RESERVE_GIB", "6"))
        _lib.reserve_device_memory(int(reserved_gib * 2 ** 30), local)
    sx, sy, sxy = K.build_kernel_specs(wl.d, wl.bandwidth_sq)
    # config 4 (l = 8192): one problem, CG matvec row-sharded over the ranks (NCCL), strong scaling;
    # every other config runs one independent replica per rank
    rowshard = args.config.startswith("cfg4") and world > 1
    if rowshard:
        from paper_2310_14087_b200 import rowshard as RS

    # ---------------- end to end through the public API from host arrays (e2e), first in the process
    torch.cuda.synchronize()
    barrier(world)
    n_e2e = args.warmup + args.steps
    _lib.profile_enable(not args.no_profile, 2)  # host phase timers of the solve's setup (cheap mode)
    t0 = time.perf_counter()
    pd = K.assemble(K.SampleSet(wl.xs), K.SampleSet(wl.ys), K.FillingPoints(wl.xt, wl.yt), wl.lambda1,
                    wl.lambda2, sx, sy, sxy, device=local)
    t_asm = time.perf_counter() - t0
    stepsize = configs.eg_stepsize(pd.q_mat, pd.pair_gram(), pd.lambda2)
    if rowshard:  # NCCL communicator setup inside the timed region
        RS.shard_rows(pd)
    cfg_e = K.SolverConfig(newton=newton_cfg(args.profile), eg=K.EgConfig(stepsize), residual_tol=1e-300,
                           max_iter=n_e2e)
    rep = K.solve(pd, cfg_e)
    torch.cuda.synchronize()
    t_call = time.perf_counter() - t0
    setup_phases = {k: round(v["ms"], 1) for k, v in _lib.profile_read().items() if k.startswith("solve.")}
    _lib.profile_enable(False)
    warm_ms = sum(r.step_ms for r in rep.trace[:args.warmup])
    t_e2e = t_call - warm_ms / 1e3
    barrier(world)
    t_e2e = max_over_ranks(world, t_e2e, local)
    e2e_iters = float(rep.iterations - args.warmup)
    e2e_iters = e2e_iters if rowshard else sum_over_ranks(world, e2e_iters, local)
    n = pd.n
    # per step: the instance's host arrays up (samples + filling points for assemble), γ̂, X̂ and the trace down
    h2d = 8.0 * (wl.xs.size + wl.ys.size + wl.xt.size + wl.yt.size) / args.steps
    d2h = ((n * n + n) * 8 + rep.iterations * 8 * 18) / args.steps
    e2e = {"value": e2e_iters / t_e2e, "unit": "iter/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "api": "paper_2310_14087_b200.assemble(host samples) + solve(pd, max_iter=W+K) -> gamma_hat, x_hat",
           "window": f"iterations {args.warmup}..{n_e2e - 1}; timed region = the whole call minus the "
                     f"{args.warmup} warm-up iterations' own step time ({warm_ms:.1f} ms)",
           "first_solve_in_process": True, "wall_ms": round(t_call * 1e3, 1), "assemble_ms": round(t_asm * 1e3, 1),
           "setup_ms": round(rep.total_ms - sum(r.step_ms for r in rep.trace), 1), "setup_phases_ms": setup_phases,
           "process_setup": (f"library load, one 2x2 eigensolve, kot_reserve({reserved_gib:g} GiB): device memory "
                             "pool grown once before the timed region; all allocations of the solve happen inside it"
                             if reserved_gib else "library load, one 2x2 eigensolve (cold device memory pool)"),
           "step_ms": [round(r.step_ms, 1) for r in rep.trace]}

    # ---------------- device-resident timed region (value)
    cfg = K.SolverConfig(newton=newton_cfg(args.profile), eg=K.EgConfig(stepsize), residual_tol=1e-300,
                         max_iter=10 ** 6)
    se = solver.Session(pd, cfg)
    stream = torch.cuda.ExternalStream(se.stream, device=f"cuda:{local}")
    for _ in range(args.warmup):
        se.step(1)
    state_w = se.state() if (world == 1 and not args.no_cpu_baseline) else None
    torch.cuda.synchronize()
    barrier(world)
    l0 = _lib.launch_count()
    # roofline scopes only (mode 2): timing every library scope costs ~14 % of the iteration rate;
    # KOT_BENCH_PROFILE=full records every phase (diagnostics, slower)
    _lib.profile_enable(not args.no_profile, 1 if os.environ.get("KOT_BENCH_PROFILE") == "full" else 2)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        barrier(world)
        ev0.record(stream)
        done = 0
        for _ in range(args.steps):
            done += se.step(1)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    ms = ev0.elapsed_time(ev1)
    prof = _lib.profile_read()
    _lib.profile_enable(False)
    launches = _lib.launch_count() - l0
    recs = se.records[args.warmup:]
    se.close()
    pd.release_device()
    ms_max = max_over_ranks(world, ms, local)
    total_iters = float(done) if rowshard else sum_over_ranks(world, float(done), local)
    value = total_iters / (ms_max / 1e3)

    # ---------------- config-5 batch (BASELINE metric, third half): every rank takes part
    batch_res = None
    if not args.no_batch and not rowshard and args.config == "cfg3":  # part of the default (headline) run
        batch_res, _, _ = batch_leg(world, rank, local, args.batch, args.tol, args.max_iter, "tight",
                                    args.concurrency)

    if rank != 0:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return 0

    roof, roof_gemm, roof_mid, phases = roofline(prof, done)

    # ---------------- CPU baseline (oracle port, bounded sample of the same window)
    cpu = None
    if state_w is not None:
        cpu = cpu_baseline_from_state(wl, args.profile, state_w, args.warmup, 2, stepsize)

    # ---------------- time-to-tolerance at the headline config (BASELINE metric, first half)
    ttt = None
    if world == 1 and not args.no_ttt and args.config == "cfg3":  # the headline config (minutes at cfg4)
        ttt = time_to_tol(K, configs, wl, args.ttt_max_iter)

    line = {
        "metric": f"SSN iters/s at n=l={wl.l} FP64 ({args.profile} profile)",
        "value": value, "unit": "iter/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_max / max(done, 1), "higher_is_better": True,
        "scaling": "strong" if rowshard else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": describe(wl, args.profile),
        "parallelism": f"rowshard{world} (CG matvec rows over NCCL)" if rowshard else f"replicas{world}",
        "e2e": e2e,
        "gpu_launches": int(launches),
        "roofline": roof,
        "roofline_gemm": roof_gemm,
        "roofline_mid": roof_mid,
        "cpu_baseline": cpu,
        "clocks": clocks.summary(),
        "time_to_tol": ttt,
        "batch": batch_res,
        "phases": phases,
        "trace": {"res": [r.res_accepted for r in recs][:64], "cg_iters": [r.cg_iters for r in recs][:64],
                  "n_pos": [r.n_pos for r in recs][:64]},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def load_traffic() -> dict:
    """ncu --set full per-launch DRAM bytes of the roofline kernels (profiles/r02/roofline_traffic.json,
    written from the committed capture by tools/ncu_traffic.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "roofline_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def roofline(prof: dict, done: int):
    """Roofline of the dominant kernel (+ the GEMM core) from the live phase profiler."""
    hbm, peak_kind = peaks()
    traffic = load_traffic()
    roof = roof_gemm = None
    full = os.environ.get("KOT_BENCH_PROFILE") == "full"
    if "sytrd_panel" in prof:
        e = prof["sytrd_panel"]
        ach = e["bytes"] / e["calls"] / (e["ms"] / e["calls"] * 1e-3) / 1e9
        t = traffic.get("sytrd_panel_kernel", {})
        roof = {"kernel": "sytrd_panel_kernel (cooperative Householder panel: column update + symv)",
                "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                "traffic": t.get("dram_bytes_per_launch"), "traffic_source": t.get("source"),
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                "algorithmic": "per launch: sum over its 32 columns of one lower-triangle read of the "
                               "trailing matrix, 8*m(m+1)/2 B",
                "avg_launch_ms": e["ms"] / e["calls"], "launches": e["calls"],
                "sampled": None if full else "1 in 16 launches (time and algorithmic bytes of the same launches)"}
    roof_mid = None
    if "sytrd_mid" in prof:  # the Newton chain's eigensolves: the trailing block resident in shared memory
        e = prof["sytrd_mid"]
        ach = e["bytes"] / e["calls"] / (e["ms"] / e["calls"] * 1e-3) / 1e9
        t = traffic.get("sytrd_mid_kernel", {})
        roof_mid = {"kernel": "sytrd_mid_kernel (grid-resident unblocked Householder: one tagged-sector all-gather "
                              "per column, the trailing block in shared memory)",
                    "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                    "traffic": t.get("dram_bytes_per_launch"), "traffic_source": t.get("source"),
                    "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                    "algorithmic": "per launch: sum over its columns of one lower-triangle read of the trailing "
                                   "matrix, 8*m(m+1)/2 B (served from shared memory: the block is read from HBM once)",
                    "avg_launch_ms": e["ms"] / e["calls"], "launches": e["calls"]}
    if roof is None and "eig.q2" in prof:  # two-stage path (l >= 3000): the tensor-core Q2 back-transform
        e = prof["eig.q2"]
        ach = e["flops"] / (e["ms"] * 1e-3) / 1e12
        roof = {"kernel": "q2_wave_kernel sequence (two-stage eigensolver, stage-2 back-transform, mma m8n8k4 f64)",
                "bound": "tensor", "achieved": ach, "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": ach / DMMA_PEAK_TFLOPS, "traffic": None,
                "algorithmic": "2 l^3 FLOPs per eigensolve (the applied reflectors' useful work)",
                "avg_launch_ms": e["ms"] / e["calls"], "launches": e["calls"]}
    if "gemm_dmma" in prof:
        e = prof["gemm_dmma"]
        ach = e["flops"] / (e["ms"] * 1e-3) / 1e12
        roof_gemm = {"kernel": "gemm_dmma_kernel (mma.sync m8n8k4 f64, all shapes)", "bound": "tensor",
                     "achieved": ach, "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": ach / DMMA_PEAK_TFLOPS,
                     "traffic": None, "peak_source": "measured DMMA microbenchmark (MEASURED_PEAKS.json has no FP64)",
                     "avg_launch_ms": e["ms"] / e["calls"], "launches": e["calls"],
                     "sampled": None if full else "1 in 128 launches"}
    phases = {k: {"ms_per_step": v["ms"] / max(done, 1), "calls_per_step": v["calls"] / max(done, 1),
                  **({"tflops": v["flops"] / (v["ms"] * 1e-3) / 1e12} if v["flops"] and v["ms"] else {}),
                  **({"sampled": {"gemm_dmma": "1 in 128 launches", "sytrd_panel": "1 in 16 launches"}[k]}
                     if k in ("gemm_dmma", "sytrd_panel") and not full else {})}
              for k, v in prof.items()}
    return roof, roof_gemm, roof_mid, phases


def cpu_baseline_from_state(wl, profile: str, state, k0: int, iters: int, stepsize: float) -> dict:
    """The oracle (reference restatement) timed for `iters` SSN iterations from the GPU trajectory's
    state at iteration k0 — the same window as `value` and the reference arm, bounded to ~10-30 s."""
    from oracle import kot_port as O
    from paper_2310_14087_b200 import configs
    pd, _ = oracle_problem(wl)
    cfg = O.SolverCfg(newton=O.NewtonCfg(**configs.PROFILES[profile]), eg_stepsize=stepsize, residual_tol=1e-300,
                      max_iter=10 ** 9)
    w, v, theta = state
    ow = O.Pair(w.gamma.copy(), w.x_mat.copy())
    r_w, dc_w = O.residual_parts(pd, ow)
    st = O.State(ow, O.Pair(v.gamma.copy(), v.x_mat.copy()), r_w, dc_w, r_w.norm(), None, None, r_w.norm(), theta)
    t0 = time.perf_counter()
    for k in range(k0, k0 + iters):
        st, _, _ = O.iterate_once(pd, st, k, cfg)
    dt = time.perf_counter() - t0
    ci = cpu_info()
    return {"value": iters / dt, "unit": "iter/s", "cores": ci["cores"], "kind": "port",
            "sample": f"SSN iterations {k0}..{k0 + iters - 1} of {wl.name} from the GPU trajectory's state at "
                      f"iteration {k0}, NumPy/OpenBLAS oracle with {ci['blas_threads']} BLAS threads; {dt:.1f} s",
            "cpu": ci["cpu"]}


def batch_leg(world: int, rank: int, local: int, n_problems: int, tol: float, max_iter: int, profile: str,
              concurrency: int):
    """BASELINE metric, third half: OT problems/s on the config-5 batch (512 independent problems,
    d=10, n=l=1000, sigma by seed % 4), sharded over the ranks (sigma groups dealt evenly), `concurrency`
    solves per GPU, fixed-size result records gathered to rank 0 over torch.distributed (NCCL).
    Each problem: assemble + solve from host arrays to `tol` within `max_iter`."""
    import torch

    from paper_2310_14087_b200 import _lib, batch

    # several solves share the GPU: thinner cooperative panel grids let their eigensolves run side by
    # side (16 problems x 100 iterations, cluster tail: 0.73 problems/s at 64 CTAs, 0.85 at 48, 0.89 at
    # 32, 0.90 at 24; concurrency 4-12 equal).  Round 2, 160 members to tol 5e-3, two runs each: 2.68 problems/s
    # at 16 CTAs, 2.74 at 20, 2.75-2.77 at 24, 2.61-2.62 at 32; concurrency 5 / 6 / 8 equal.
    _lib.lib().kot_set_panel_grid_cap(int(os.environ.get("KOT_BATCH_GRID", "24")))
    seeds = list(range(n_problems))
    mine = batch.shard(seeds, world, rank)
    kw = dict(profile=profile, residual_tol=tol, max_iter=max_iter)
    batch.gpu_solve_member(seeds[0], dict(kw, max_iter=2), local)  # warm-up outside the timed region
    torch.cuda.synchronize()
    barrier(world)
    l0 = _lib.launch_count()
    with ClockSampler(local) as clocks:
        t0 = time.perf_counter()
        allr = batch.run_and_gather(mine, lambda s: batch.gpu_solve_member(s, kw, local), concurrency, 1000,
                                    world, rank, device=f"cuda:{local}" if world > 1 else None)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    launches = _lib.launch_count() - l0
    _lib.lib().kot_set_panel_grid_cap(0)
    dt_max = max_over_ranks(world, dt, local)
    if rank != 0:
        return None, launches, clocks.summary()
    conv = sum(r.converged for r in allr)
    iters = [r.iterations for r in allr]
    out = {
        "metric": f"OT problems/s (config 5: {n_problems} problems, d=10, n=l=1000, {profile} profile, "
                  f"tol {tol:g}, max_iter {max_iter})",
        "value": len(allr) / dt_max, "unit": "problems/s", "seconds": dt_max, "problems": len(allr),
        "converged": int(conv),
        "converged_by_sigma": {str(sg): sum(r.converged for r in allr if r.seed % 4 == g)
                               for g, sg in enumerate((0.5, 1.0, 1.5, 2.0))},
        "iterations_mean": float(np.mean(iters)), "iterations_max": int(max(iters)),
        "residual_max": float(max(r.residual_norm for r in allr)),
        "concurrency_per_gpu": concurrency, "parallelism": f"shard{world} (sigma-balanced), records gathered",
        "api": "per problem: assemble(host samples) + solve(pd) -> gamma_hat (batch.gpu_solve_member)",
        "gpu_launches": int(launches),
    }
    return out, launches, clocks.summary()


def run_batch(args):
    """Config 5 alone (--config cfg5): the batch leg as the bench line."""
    world, rank, local = dist_setup(args.gpus)
    os.environ["KOT_DEVICE"] = str(local)
    import torch
    torch.cuda.set_device(local)
    res, launches, clocks = batch_leg(world, rank, local, args.batch, args.tol, args.max_iter, args.profile,
                                      args.concurrency)
    if rank == 0:
        line = {
            "metric": res["metric"], "value": res["value"], "unit": "problems/s", "n_gpus": world,
            "steps": res["problems"], "warmup": 1, "ms_per_step": 1e3 * res["seconds"] / max(res["problems"], 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": res["metric"]}, "parallelism": res["parallelism"],
            "e2e": {"value": res["value"], "unit": "problems/s", "api": res["api"],
                    "h2d_bytes_per_step": 8 * 1000 * 40, "d2h_bytes_per_step": 8 * (1000 + 16)},
            "gpu_launches": res["gpu_launches"], "batch": res, "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--profile", default="paper", choices=["paper", "tight"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ttt", action="store_true", help="skip the time-to-tolerance leg")
    ap.add_argument("--ttt-max-iter", type=int, default=300, help="max_iter of the time-to-tolerance solves")
    ap.add_argument("--no-profile", action="store_true", help="diagnostic: no phase profiler in the timed region")
    ap.add_argument("--batch", type=int, default=512, help="cfg5: number of problems (BASELINE: 512)")
    ap.add_argument("--concurrency", type=int, default=6, help="cfg5: concurrent solves per GPU")
    ap.add_argument("--tol", type=float, default=5e-3, help="cfg5: residual tolerance (the paper's threshold)")
    ap.add_argument("--max-iter", type=int, default=100, help="cfg5: max SSN iterations per problem")
    ap.add_argument("--no-batch", action="store_true", help="skip the config-5 batch leg")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    if args.config == "cfg5" and args.impl == "ours":
        return run_batch(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
