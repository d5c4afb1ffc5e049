"""Concurrent-solve determinism probe: the same config-5 members solved one at a time and then by
N host threads at once must give bit-identical results (diagnostic).

python tools/conc_probe.py N_PROBLEMS MAX_ITER THREADS [preassemble]"""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np

import paper_2310_14087_b200 as K
from paper_2310_14087_b200 import configs
from paper_2310_14087_b200.solver import _run

nprob, mi, thr = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
pre = len(sys.argv) > 4 and sys.argv[4] == "pre"


def build(seed):
    wl = configs.config5_member(seed)
    sx, sy, sxy = K.build_kernel_specs(wl.d, wl.bandwidth_sq)
    pd = K.assemble(K.SampleSet(wl.xs), K.SampleSet(wl.ys), K.FillingPoints(wl.xt, wl.yt), wl.lambda1,
                    wl.lambda2, sx, sy, sxy)
    step = configs.eg_stepsize(pd.q_mat, pd.pair_gram(), pd.lambda2)
    cfg = K.SolverConfig(newton=K.NewtonConfig(), eg=K.EgConfig(step), residual_tol=1e-12, max_iter=mi)
    return pd, cfg


def solve(seed, pds=None):
    pd, cfg = pds[seed] if pds else build(seed)
    rep = _run(pd, cfg, None, False, want_x=False)
    return rep.residual_norm, float(np.sum(rep.gamma_hat))


ref = {s: solve(s) for s in range(nprob)}
pds = {s: build(s) for s in range(nprob)} if pre else None
out, errs = {}, []
queue = list(range(nprob))
lock = threading.Lock()


def worker():
    while True:
        with lock:
            if not queue:
                return
            s = queue.pop(0)
        try:
            out[s] = solve(s, pds)
        except Exception as e:  # noqa: BLE001
            errs.append((s, repr(e)[:200]))


ts = [threading.Thread(target=worker) for _ in range(thr)]
for t in ts:
    t.start()
for t in ts:
    t.join()
bad = [s for s in out if out[s] != ref[s]]
print(f"threads={thr} pre={pre}: {len(out)} solved, {len(bad)} differ from the sequential run {bad[:8]}, "
      f"errors {errs[:3]}", flush=True)
