import sys, time, cProfile, pstats
sys.path.insert(0, '.')
import numpy as np
import paper_2310_14087_b200 as K
from paper_2310_14087_b200 import configs, _lib
wl = configs.config3()
sx, sy, sxy = K.build_kernel_specs(wl.d, wl.bandwidth_sq)
def asm():
    return K.assemble(K.SampleSet(wl.xs), K.SampleSet(wl.ys), K.FillingPoints(wl.xt, wl.yt), wl.lambda1, wl.lambda2, sx, sy, sxy)
pd = asm()
pr = cProfile.Profile(); pr.enable(); pd2 = asm(); pr.disable()
pstats.Stats(pr).sort_stats('cumulative').print_stats(18)
step = configs.eg_stepsize(pd2.q_mat, pd2.pair_gram(), pd2.lambda2)
cfg = K.SolverConfig(newton=K.NewtonConfig(**configs.PROFILES["paper"]), eg=K.EgConfig(step), residual_tol=1e-300, max_iter=3)
K.solve(pd, cfg)
pr = cProfile.Profile(); pr.enable(); rep = K.solve(pd2, cfg); pr.disable()
pstats.Stats(pr).sort_stats('cumulative').print_stats(14)
