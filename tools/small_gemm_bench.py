"""The small FP64 GEMMs of a C2 block (b = 50, l up to 200, m = n = 8000), timed one by one."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_03859_b200 as fqb

eng = fqb.Engine(0)
st = torch.cuda.Stream()
eng.set_stream(st.cuda_stream)
m = n = 8000
b = 50
shapes = [  # (name, trans, M, N, K)
    ("S = W'W", True, b, b, n),
    ("G = W R^-1", False, n, b, b),
    ("[Q|Y]'Y l=150", True, 200, b, m),
    ("Y -= Q C l=150", False, m, b, 150),
    ("Q'ys l=150", True, 150, b, m),
    ("Bt cd l=150", False, n, b, 150),
    ("t = B G l=150", True, 150, b, n),
    ("U = Q Ut l=200", False, m, 200, 200),
    ("BB' l=200", True, 200, 200, n),
]
for name, tr, M, N, K in shapes:
    a = torch.randn((M, K) if not tr else (K, M), dtype=torch.float64, device="cuda").t().contiguous().t()
    bb = torch.randn((K, N), dtype=torch.float64, device="cuda").t().contiguous().t()
    c = torch.zeros((M, N), dtype=torch.float64, device="cuda").t().contiguous().t()
    args = (tr, M, N, K, 1.0, a.data_ptr(), a.stride(1) if a.dim() == 2 else 1, bb.data_ptr(), bb.stride(1), 0.0,
            c.data_ptr(), c.stride(1))
    for _ in range(5):
        eng.gemm(*args)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record()
        for _ in range(50):
            eng.gemm(*args)
        e1.record()
    e1.synchronize()
    us = e0.elapsed_time(e1) / 50 * 1e3
    print(f"{name:18s} {'TN' if tr else 'NN'} {M}x{N}x{K}: {us:6.1f} us  {2*M*N*K/us/1e6:6.2f} TF/s")

print("--- cuBLAS (torch.matmul) on the same shapes ---")
for name, tr, M, N, K in shapes:
    a = torch.randn((K, M) if tr else (M, K), dtype=torch.float64, device="cuda")
    bb = torch.randn((K, N), dtype=torch.float64, device="cuda")
    op = (lambda: a.t() @ bb) if tr else (lambda: a @ bb)
    for _ in range(5):
        op()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        op()
    e1.record()
    e1.synchronize()
    us = e0.elapsed_time(e1) / 50 * 1e3
    print(f"{name:18s} {'TN' if tr else 'NN'} {M}x{N}x{K}: {us:6.1f} us  {2*M*N*K/us/1e6:6.2f} TF/s")
