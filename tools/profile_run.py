"""One warm-up + one timed C4 (bench workload) run_fixed_precision, for ncu launch lists.

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python tools/profile_run.py
Kernels of the second run follow the marker launch count printed to stdout.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_03859_b200 as fqb  # noqa: E402

eng = fqb.Engine(0)
a = bench.make_matrix(eng)
torch.cuda.synchronize()
cfg = bench.config()
n_runs = int(os.environ.get("FQB_PROFILE_RUNS", "2"))
for i in range(n_runs):
    before = eng.launch_count
    r = eng.run_fixed_precision(a, cfg, output="device", svd=True)
    print(f"run {i}: launches {before}..{eng.launch_count} rank={r.rank} blocks={r.blocks} "
          f"ms={r.elapsed_ms:.3f}", flush=True)
