"""One C4-shape A pass on the INT8 emulation, for an ncu capture of k_ozaki<true,7>.

    python tools/ozaki_c4_once.py [tn|nn] [reps]
A = the bench's C4 matrix (fqb_gen_lowrank_det), sliced once; W = A'Y (tn) or Y = A G
(nn) with b = 100 (two 50-column chunks on CTA pairs), run `reps` times.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_03859_b200 as fqb  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "tn"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
eng = fqb.Engine(0)
a = bench.make_matrix(eng)
m, n, b = bench.M, bench.N, bench.BLOCK
trans = which == "tn"
k, rows = (m, n) if trans else (n, m)
x = torch.randn(b, k, dtype=torch.float64, device="cuda").t()
out = torch.empty(b, rows, dtype=torch.float64, device="cuda").t()
sl = eng.slice_operand(a.data_ptr(), m, n, m)
for _ in range(reps):
    sl.gemm(trans, b, 1.0, x.data_ptr(), k, 0.0, out.data_ptr(), rows)
torch.cuda.synchronize()
sl.free()
print("done", which, float(out.abs().sum()))
