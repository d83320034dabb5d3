import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2506_03859_b200 as fqb
eng = fqb.Engine(0); st = torch.cuda.Stream(); eng.set_stream(st.cuda_stream)
a = bench.make_matrix(torch.device("cuda:0")); torch.cuda.synchronize(); cfg = bench.config()
for svd in (False, True):
    ts = [round(eng.run_fixed_precision(a, cfg, output="device", svd=svd).elapsed_ms, 2) for _ in range(6)]
    print(os.environ.get("FQB_EIG", "syevj"), "svd" if svd else "qb", ts, flush=True)
r = eng.run_fixed_precision(a, cfg, output="host", svd=True)
import numpy as np
print("sigma top", r.sigma[-3:], "bottom", r.sigma[:2], "recon", np.linalg.norm((r.u * r.sigma) @ r.v.T - r.q @ r.bt.T))
