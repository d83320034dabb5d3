"""Warm per-kernel times of one run_fixed_precision (CUPTI via torch.profiler).

Unlike an ncu launch list (caches flushed and kernels serialised per launch),
this is the steady state the bench sees.  Usage:
    python tools/kernel_profile.py [--config c4|c2] [--svd] [--runs N]
"""
import argparse
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_2506_03859_b200 as fqb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--svd", action="store_true")
ap.add_argument("--runs", type=int, default=3)
ap.add_argument("--config", default="c4", choices=["c4", "c2"])
args = ap.parse_args()

eng = fqb.Engine(0)
if args.config == "c4":
    a = bench.make_matrix(eng)
    cfg = bench.config()
else:
    import numpy as np
    from paper_2506_03859_b200 import FarpcaConfig, SketchKind, SketchSpec
    a = eng.gen_lowrank(8000, 8000, 10.0 ** (-np.arange(1, 901) / 50.0), seed=42)
    cfg = FarpcaConfig(eps=1e-3, power=2, block=50, sketch=SketchSpec(SketchKind.StdBernoulli, 0.5, 7),
                       relative=True)
for _ in range(2):
    eng.run_fixed_precision(a, cfg, output="device", svd=args.svd)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA], acc_events=True) as prof:
    for _ in range(args.runs):
        r = eng.run_fixed_precision(a, cfg, output="device", svd=args.svd)
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        name = ev.name
        for junk in ("void ", "farqb::", "(anonymous namespace)::", "<unnamed>::"):
            name = name.replace(junk, "")
        name = name.split("(")[0]
        agg[name][0] += 1
        agg[name][1] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
tot = sum(v[1] for v in agg.values()) / args.runs
print(f"per run: {tot:.1f} us of kernel time; engine elapsed {r.elapsed_ms * 1e3:.1f} us")
for k, (c, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{us / args.runs:9.1f} us {100 * us / args.runs / tot:5.1f}%  {c // args.runs:4d}x  {k[:90]}")

# host side: CUDA runtime calls made by the library (CUPTI runtime trace) and GPU idle gaps
rt = collections.defaultdict(lambda: [0, 0.0])
kern = []
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CPU and ev.name.startswith("cuda"):
        rt[ev.name][0] += 1
        rt[ev.name][1] += ev.cpu_time_total
    elif ev.device_type == torch.autograd.DeviceType.CUDA:
        nm = ev.name
        for junk in ("void ", "farqb::", "(anonymous namespace)::", "<unnamed>::"):
            nm = nm.replace(junk, "")
        kern.append((ev.time_range.start, ev.time_range.end, nm.split("(")[0][:50]))
print("host CUDA runtime calls per run:")
for k, (c, us) in sorted(rt.items(), key=lambda x: -x[1][1])[:8]:
    print(f"  {us / args.runs:9.1f} us  {c // args.runs:5d}x  {k}")
kern.sort()
gl = [(b[0] - a[1], a[2], b[2]) for a, b in zip(kern, kern[1:]) if b[0] > a[1]]
gaps = sorted((g[0] for g in gl), reverse=True)
print(f"GPU idle between kernels per run: {sum(gaps) / args.runs:.1f} us over {len(gaps) // args.runs} gaps; "
      f"largest {[round(g, 1) for g in gaps[:8]]}  (includes the gaps between runs)")
print("largest gaps (after -> before):")
for g, a_, b_ in sorted(gl, reverse=True)[:14]:
    print(f"  {g:8.1f} us  {a_}  ->  {b_}")
