"""Time fqb_sym_eig (small-l solver vs FQB_EIG=syevd) at the SVD-assembly size, with a
per-kernel breakdown via torch.profiler when --profile is given."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2506_03859_b200 as fqb  # noqa: E402

eng = fqb.default_engine(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(0)
q, _ = np.linalg.qr(rng.standard_normal((n, n)))
m = (q * 10.0 ** (-2 * np.arange(n) / 50.0)) @ q.T
m = torch.from_numpy(np.asfortranarray(0.5 * (m + m.T))).cuda()
for mode in ["small", "syevd"]:
    os.environ["FQB_EIG"] = mode
    for _ in range(3):
        eng.sym_eig(m)
    t = time.perf_counter()
    for _ in range(20):
        _, _, small = eng.sym_eig(m)
    print(f"n={n} {mode:6s}: {(time.perf_counter() - t) / 20 * 1e6:8.1f} us per call (small path: {small})")
if "--profile" in sys.argv:
    os.environ["FQB_EIG"] = "small"
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(5):
            eng.sym_eig(m)
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15))
