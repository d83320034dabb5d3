"""DMMA GEMM throughput on the QB loop's dominant shapes (CUDA events, engine stream)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_03859_b200 as fqb  # noqa: E402

SHAPES = [  # (name, trans, M, N, K)
    ("C2 A'Y", True, 8000, 50, 8000), ("C2 AG", False, 8000, 50, 8000),
    ("C1 A'Y", True, 2000, 20, 2000), ("C1 AG", False, 2000, 20, 2000),
    ("C3 A'Y", True, 20000, 64, 20000), ("C3 AG", False, 20000, 64, 20000),
    ("C4 A'Y", True, 20000, 100, 100000), ("C4 AG", False, 100000, 100, 20000),
    ("C2 QtY", True, 200, 50, 8000), ("C2 Y-QC", False, 8000, 50, 150),
]
only = os.environ.get("FQB_GEMM_ONLY")
eng = fqb.Engine(0)
stream = torch.cuda.Stream()
eng.set_stream(stream.cuda_stream)
for name, trans, M, N, K in SHAPES:
    if only and only not in name:
        continue
    a = torch.randn((M, K) if trans else (K, M), dtype=torch.float64, device="cuda").t()  # col-major (K x M) or (M x K)
    b = torch.randn((N, K), dtype=torch.float64, device="cuda").t()
    c = torch.empty((N, M), dtype=torch.float64, device="cuda").t()
    torch.cuda.synchronize()
    args = (trans, M, N, K, 1.0, a.data_ptr(), a.stride(1), b.data_ptr(), b.stride(1), 0.0, c.data_ptr(), c.stride(1))
    for _ in range(3):
        eng.gemm(*args)
    reps = int(os.environ.get("FQB_GEMM_REPS", "20"))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record()
        for _ in range(reps):
            eng.gemm(*args)
        e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    ref = (a.t() if trans else a) @ b
    err = ((c - ref).abs().max() / ref.abs().max()).item()
    print(f"{name:10s} {'TN' if trans else 'NN'} {M}x{N}x{K}: {ms*1e3:9.1f} us  {2*M*N*K/ms/1e9:6.2f} TFLOP/s  relerr {err:.1e}", flush=True)
    del a, b, c, ref
    torch.cuda.empty_cache()
