"""Where the end-to-end (host A in, host factors out) C4 step spends its time.

    FQB_HOST_STATS=1 python tools/e2e_probe.py [steps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_03859_b200 as fqb  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
eng = fqb.Engine(0)
a = bench.make_matrix(eng)
cfg = bench.config()
a_host = torch.empty((bench.N, bench.M), dtype=torch.float64, pin_memory=True)
a_host.copy_(a.t())
a_cm = a_host.t()
# raw H2D rate of the same bytes
d = torch.empty_like(a)
torch.cuda.synchronize()
t0 = time.perf_counter()
d.t().copy_(a_host, non_blocking=True)
torch.cuda.synchronize()
print(f"H2D 16 GB (torch copy_ from pinned): {time.perf_counter() - t0:.3f} s")
del d
for i in range(steps):
    t0 = time.perf_counter()
    r = eng.run_fixed_precision(a, cfg, output="device", svd=True)
    t1 = time.perf_counter()
    r = None
    t2 = time.perf_counter()
    r = eng.run_fixed_precision(a_cm, cfg, output="host", svd=True)
    t3 = time.perf_counter()
    print(f"step {i}: device-in/device-out {t1 - t0:.3f} s (engine {0:.0f}), host-in/host-out {t3 - t2:.3f} s "
          f"(engine device time {r.elapsed_ms:.1f} ms)", flush=True)
    r = None
