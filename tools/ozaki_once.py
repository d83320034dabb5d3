"""One C2-shape k_ozaki launch (W = A'Y, 8000 x 50 x 8000, pre-sliced operands) after a
warm-up: the ncu target for the dominant kernel (ncu -k regex:k_ozaki -s 5 -c 1)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2506_03859_b200 as fqb  # noqa: E402

eng = fqb.default_engine(0)
m = n = 8000
b = 50
a = torch.randn((n, m), dtype=torch.float64, device="cuda").t()
y = torch.randn((b, m), dtype=torch.float64, device="cuda").t()
w = torch.empty((b, n), dtype=torch.float64, device="cuda").t()
with eng.slice_operand(a.data_ptr(), m, n, m) as sl:
    sl.gemm(True, b, 1.0, y.data_ptr(), m, 0.0, w.data_ptr(), n)
    for _ in range(8):
        sl.gemm_again(1.0, 0.0, w.data_ptr(), n)
torch.cuda.synchronize()
print("done")
