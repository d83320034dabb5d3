import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, collections
from torch.profiler import profile, ProfilerActivity
import paper_2506_03859_b200 as fqb
eng = fqb.Engine(0)
for (m, n) in [(8000, 50), (8000, 8000), (100000, 100)]:
    a = torch.randn(n, m, dtype=torch.float64, device="cuda").t()
    for _ in range(3): eng.frob_norm_sq(a.data_ptr(), m, n, m) if hasattr(eng, "frob_norm_sq") else None
    with profile(activities=[ProfilerActivity.CUDA], acc_events=True) as prof:
        for _ in range(10): eng.frob_norm_sq(a.data_ptr(), m, n, m)
        torch.cuda.synchronize()
    agg = collections.defaultdict(lambda: [0, 0.0])
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            agg[ev.name.split("(")[0][-40:]][0] += 1; agg[ev.name.split("(")[0][-40:]][1] += ev.device_time_total
    print(m, n, {k: round(v[1] / v[0], 1) for k, v in agg.items()})
