"""Device time of run_fixed_precision on the BASELINE configs 3 and 4 at full size (A generated on the GPU).

    python tools/config_time.py [c3|c4]      (FQB_OZAKI=0 for the DMMA A passes)
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2506_03859_b200 as fqb
from paper_2506_03859_b200 import FarpcaConfig, SketchKind, SketchSpec

DEV = torch.device("cuda:0")


which = sys.argv[1] if len(sys.argv) > 1 else "c4"
if which == "c4":
    sig = 10.0 ** (-3.0 * np.arange(1, 2001, dtype=np.float64) / 2000)
    a = fqb.default_engine(0).gen_lowrank_det(100000, 20000, sig, 42)
    cfg = FarpcaConfig(eps=1e-3, power=2, block=100, sketch=SketchSpec(SketchKind.SparseGaussian, 0.0, 7, zeta=8),
                       relative=True)
else:
    sig = (1.0 + np.arange(0, 1000, dtype=np.float64)) ** -1.5
    a = fqb.default_engine(0).gen_lowrank_det(20000, 20000, sig, 42, 1e-4 / np.sqrt(20000))
    cfg = FarpcaConfig(eps=1e-2, power=1, block=64, sketch=SketchSpec(SketchKind.SparseSign, 0.0, 7, zeta=8),
                       relative=True)
eng = fqb.Engine(0)
for i in range(2):
    t0 = time.perf_counter()
    try:
        r = eng.run_fixed_precision(a, cfg, output="device")
    except fqb.ToleranceNotReached as e:
        r = e.partial
    torch.cuda.synchronize()
    print(f"{which} run {i}: rank {r.rank} blocks {r.blocks} converged {r.converged} device {r.elapsed_ms:.1f} ms "
          f"wall {1e3 * (time.perf_counter() - t0):.1f} ms launches {r.gpu_launches}", flush=True)
    del r

if os.environ.get("FQB_PROFILE"):
    import collections
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA], acc_events=True) as prof:
        try:
            r = eng.run_fixed_precision(a, cfg, output="device")
        except fqb.ToleranceNotReached as e:
            r = e.partial
        torch.cuda.synchronize()
    agg = collections.defaultdict(lambda: [0, 0.0])
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            name = ev.name
            for junk in ("void ", "farqb::", "(anonymous namespace)::", "<unnamed>::"):
                name = name.replace(junk, "")
            name = name.split("(")[0]
            agg[name][0] += 1
            agg[name][1] += ev.device_time_total
    tot = sum(v[1] for v in agg.values())
    print(f"kernel time {tot / 1e3:.1f} ms")
    for k, (c, us) in sorted(agg.items(), key=lambda x: -x[1][1])[:15]:
        print(f"{us / 1e3:9.2f} ms {100 * us / tot:5.1f}%  {c:5d}x  {k[:80]}")
