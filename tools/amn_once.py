"""One C4-shape projection Y -= Q C on the MN-major INT8 path (k_ozaki AMN variant), for ncu:
Q 100000 x l (its A'Y-layout slices, as the engine keeps them), C l x 100, l = argv[1] (1000)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_03859_b200 as fqb  # noqa: E402

l = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
m, b = 100000, 100
eng = fqb.Engine(0)
q = torch.randn(l, m, dtype=torch.float64, device="cuda").t()
c = torch.randn(b, l, dtype=torch.float64, device="cuda").t()
y = torch.randn(b, m, dtype=torch.float64, device="cuda").t()
sl = eng.slice_operand(q.data_ptr(), m, l, m)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(reps):
    if i == reps - 1:
        e0.record()
    sl.gemm_mn(b, -1.0, c.data_ptr(), l, 1.0, y.data_ptr(), m)
e1.record()
torch.cuda.synchronize()
print(f"Y -= Q C, l = {l}: {e0.elapsed_time(e1) * 1e3:.1f} us (last of {reps})")
sl.free()
