"""C4-shape calls of the tall-skinny Gram kernel (tsmm.cu), for ncu: S = Y'Y with Y
100000 x 100 (the accept step's shape), then 20000 x 100 (the power passes')."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_03859_b200 as fqb  # noqa: E402

eng = fqb.Engine(0)
b = 100
for rows in (100000, 20000):
    y = torch.randn(b, rows, dtype=torch.float64, device="cuda").t()
    r = torch.triu(torch.randn(b, b, dtype=torch.float64, device="cuda")).t().contiguous().t()
    for _ in range(2):
        s = eng.gram(y)
        z = eng.mul_upper(y, r)
torch.cuda.synchronize()
print("done", float(s.abs().sum()))
