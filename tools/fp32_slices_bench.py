"""FP32 input: QB time-to-eps with FP64-class (8) vs FP32-class (4 or 3 slices) A passes,
on a config-5-like low-rank-plus-noise FP32 matrix (rows x cols given), b = 128,
sparse sign zeta = 4, P = 1, eps = 5e-2 (the config-5 settings) with a block cap."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2506_03859_b200 as fqb  # noqa: E402
from paper_2506_03859_b200 import FarpcaConfig, SketchSpec  # noqa: E402

m, n = (int(x) for x in (sys.argv[1:3] if len(sys.argv) > 2 else (100000, 20000)))
eng = fqb.default_engine(0)
r = 500
sig = 1.0 / np.arange(1, r + 1)
a = eng.gen_lowrank(m, n, sig, seed=42, noise=1e-3).float()
a = a.t().contiguous().t()
cfg = FarpcaConfig(eps=5e-2, power=1, block=128, sketch=SketchSpec(3, 0.0, 7, zeta=4), relative=True,
                   max_iters=12)
for nsl in (8, 4, 3):
    e = fqb.Engine(0)
    e.set_fp32_slices(nsl)
    out = []
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        try:
            res = e.run_fixed_precision(a, cfg, output="device")
        except fqb.ToleranceNotReached as ex:
            res = ex.partial
        torch.cuda.synchronize()
        out.append((time.perf_counter() - t, res))
    dt, res = out[-1]
    print(f"{m} x {n} FP32, {nsl} slices: {dt * 1e3:8.1f} ms (engine {res.elapsed_ms:.1f} ms, "
          f"{res.gpu_launches} launches)  rank {res.rank} blocks {res.blocks} "
          f"E/|A|^2 {res.residual_sq / res.norm_a_sq:.6e}  runs {[round(o[0] * 1e3, 1) for o in out]}", flush=True)
    e.close()
