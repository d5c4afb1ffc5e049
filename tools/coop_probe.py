"""Does a background COOPERATIVE grid slow the Newton chain more than the same plain grid
(diagnostic)?  cfg3 Newton chain alone (safeguard_every=10**6) while a background thread launches
back-to-back 64-CTA, 400 µs spin grids (tools/microbench/libspin.so) cooperatively or plainly."""
import ctypes as C
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2310_14087_b200 as K  # noqa: E402
from paper_2310_14087_b200 import _lib, configs, solver  # noqa: E402

spin = C.CDLL(os.path.join(ROOT, "tools", "microbench", "libspin.so"))
wl = configs.config3()
sx, sy, sxy = K.build_kernel_specs(wl.d, wl.bandwidth_sq)
pd = K.assemble(K.SampleSet(wl.xs), K.SampleSet(wl.ys), K.FillingPoints(wl.xt, wl.yt), wl.lambda1, wl.lambda2,
                sx, sy, sxy)
step = configs.eg_stepsize(pd.q_mat, pd.pair_gram(), pd.lambda2)


def bg(kind, stop):
    coop = 1 if kind.startswith("coop") else 0
    ctas = int(kind.split("_")[1])
    while not stop.is_set():
        for _ in range(8):
            spin.spin_launch(ctas, 256, 400, coop, 64)
        spin.spin_sync()


for kind in ("none", "coop_64", "plain_64", "coop_128", "plain_128", "none"):
    cfg = K.SolverConfig(eg=K.EgConfig(step), residual_tol=1e-300, max_iter=10 ** 6, safeguard_every=10 ** 6)
    se = solver.Session(pd, cfg)
    se.step(3)
    stop = threading.Event()
    th = threading.Thread(target=bg, args=(kind, stop)) if kind != "none" else None
    if th:
        th.start()
        time.sleep(0.3)
    _lib.profile_enable(True, 1)
    t0 = time.perf_counter()
    se.step(6)
    dt = time.perf_counter() - t0
    prof = _lib.profile_read()
    _lib.profile_enable(False)
    stop.set()
    if th:
        th.join()
    se.close()
    pick = {k: round(prof[k]["ms"] / 6, 2) for k in ("host.newton", "host.trial_resid") if k in prof}
    print(f"background={kind}: {6 / dt:.2f} it/s  per iteration {pick}", flush=True)
