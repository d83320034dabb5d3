"""The FP64 products of one C4 block outside the A passes (m = 100000, n = 20000, b = 100),
timed one by one on the engine's DMMA path, and the B-side products on the INT8 sliced path
(B' sliced once, like Q) for comparison.

    python tools/small_gemm_c4.py [l]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_03859_b200 as fqb  # noqa: E402

l = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
eng = fqb.Engine(0)
st = torch.cuda.Stream()
eng.set_stream(st.cuda_stream)
m, n, b = 100000, 20000, 100


def cm(r, c):
    return torch.randn(c, r, dtype=torch.float64, device="cuda").t()   # column-major r x c


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


shapes = [  # (name, trans, M, N, K, per-block count)
    ("S = W'W", True, b, b, n, 4),
    ("G = W R^-1", False, n, b, b, 4),
    ("S = Y'Y (m)", True, b, b, m, 2),
    ("ys = Y R^-1 (m)", False, m, b, b, 2),
    (f"T = B G l={l}", True, l, b, n, 1),
    (f"W -= B' T l={l}", False, n, b, l, 3),
    (f"B_j' = W Ri", False, n, b, b, 1),
]
tot = 0.0
for name, tr, M, N, K, cnt in shapes:
    a = cm(K, M) if tr else cm(M, K)
    bb = cm(K, N)
    c = cm(M, N)
    us = timed(lambda: eng.gemm(tr, M, N, K, 1.0, a.data_ptr(), a.stride(1), bb.data_ptr(), bb.stride(1), 0.0,
                                c.data_ptr(), c.stride(1)))
    tot += cnt * us
    print(f"{name:22s} {'TN' if tr else 'NN'} {M}x{N}x{K}: {us:7.1f} us  {2*M*N*K/us/1e6:6.2f} TF/s  x{cnt}/block")
print(f"DMMA products per block at l={l}: {tot:.0f} us")

# the Grams on the tall-skinny kernel (tsmm.cu: upper tiles only)
for name, K in (("ts_gram S = W'W", n), ("ts_gram S = Y'Y (m)", m)):
    y = cm(K, b)
    s_out = cm(b, b)
    us = timed(lambda: eng.gram(y, out=s_out, sync=False))
    print(f"{name:22s} {K}x{b}: {us:7.1f} us ({2*K*b*b/us/1e6:6.2f} TF/s full-product equivalent)")

for name, M in (("ts_trmm G = W R^-1", n), ("ts_trmm ys = Y R^-1 (m)", m)):
    y = cm(M, b)
    r = torch.triu(cm(b, b)).t().contiguous().t()
    us = timed(lambda: eng.mul_upper(y, r, sync=False))
    print(f"{name:22s} {M}x{b}: {us:7.1f} us ({2*M*b*b/us/1e6:6.2f} TF/s full-product equivalent)")

# B-side products on the INT8 path: B' (n x l) sliced once
bt = cm(n, l)
g = cm(n, b)
t = cm(l, b)
wout = cm(n, b)
tout = cm(l, b)
sl = eng.slice_operand(bt.data_ptr(), n, l, bt.stride(1))
us_tn = timed(lambda: sl.gemm(True, b, 1.0, g.data_ptr(), g.stride(1), 0.0, tout.data_ptr(), tout.stride(1)))
us_mn = timed(lambda: sl.gemm_mn(b, -1.0, t.data_ptr(), t.stride(1), 1.0, wout.data_ptr(), wout.stride(1)))
print(f"INT8 T = B G (B' sliced, K = n): {us_tn:7.1f} us   INT8 W -= B' T (MN-major, K = l): {us_mn:7.1f} us")
sl.free()

# b x b Cholesky + inverse (k_chol_inv_reg)
S = cm(b, b)
S = (S.t() @ S + b * torch.eye(b, dtype=torch.float64, device="cuda")).contiguous()
if hasattr(eng, "chol_upper_inv"):
    us = timed(lambda: eng.chol_upper_inv(S))
    print(f"chol b={b}: {us:.1f} us")
