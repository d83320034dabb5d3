"""Drive fqb_slice_operand on a C2-sized A (8000 x 8000 FP64) for an ncu capture of
k_line_max / k_slice_a:  ncu -k regex:k_slice_a --set full python tools/slice_profile.py"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2506_03859_b200 as fqb  # noqa: E402

eng = fqb.default_engine(0)
m = n = 8000
a = torch.randn((n, m), dtype=torch.float64, device="cuda").t()
for _ in range(3):
    with eng.slice_operand(a.data_ptr(), m, n, m) as sl:
        pass
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    with eng.slice_operand(a.data_ptr(), m, n, m) as sl:
        pass
e.record()
torch.cuda.synchronize()
print(f"slice_operand (both layouts, incl. alloc/free): {s.elapsed_time(e) / 10 * 1e3:.1f} us")
