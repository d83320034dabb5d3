"""Gather-SpMM GB/s for the C3 sketch shape, per FQB_SPMM_VPL setting (run once per env)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_03859_b200 as fqb  # noqa: E402

eng = fqb.Engine(0)
r = bench.sketch_roofline(eng, torch.device("cuda:0"), bench.peaks())
print(os.environ.get("FQB_SPMM_VPL", "auto"), f"{r['achieved']:.0f} GB/s frac {r['frac']:.3f} {r['launch_us']:.2f} us")
