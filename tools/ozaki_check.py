"""Accuracy and speed of the emulated FP64 GEMM vs DMMA and a float64 reference."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_03859_b200 as fqb
eng = fqb.Engine(0)
st = torch.cuda.Stream(); eng.set_stream(st.cuda_stream)
torch.manual_seed(0)
cases = [("small", True, 300, 20, 1000), ("small nn", False, 257, 33, 999), ("n1", True, 128, 1, 128),
         ("C2 A'Y", True, 8000, 50, 8000), ("C2 AG", False, 8000, 50, 8000), ("C3", True, 20000, 64, 20000),
         ("C1", False, 2000, 20, 2000)]
only = os.environ.get("OZ_ONLY")
for name, trans, M, N, K in cases:
    if only and only != name:
        continue
    a = torch.randn((M, K) if trans else (K, M), dtype=torch.float64, device="cuda").t()
    if name.startswith("small"):
        a = a * torch.logspace(-6, 6, a.shape[1], dtype=torch.float64, device="cuda")  # wild column scales
    b = torch.randn((N, K), dtype=torch.float64, device="cuda").t()
    c = torch.zeros((N, M), dtype=torch.float64, device="cuda").t()
    c2 = torch.zeros((N, M), dtype=torch.float64, device="cuda").t()
    torch.cuda.synchronize()
    args = (trans, M, N, K, 1.0, a.data_ptr(), a.stride(1), b.data_ptr(), b.stride(1), 0.0)
    eng.gemm_emulated(*args, c.data_ptr(), c.stride(1))
    eng.gemm(*args, c2.data_ptr(), c2.stride(1))
    torch.cuda.synchronize()
    ref = ((a.t() if trans else a).cpu() @ b.cpu())  # CPU float64 BLAS
    bound = ((a.t() if trans else a).abs().cpu() @ b.abs().cpu())
    e_oz = float(((c.cpu() - ref).abs() / bound).max())
    e_dm = float(((c2.cpu() - ref).abs() / bound).max())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    with torch.cuda.stream(st):
        e0.record()
        for _ in range(reps):
            eng.gemm(*args, c2.data_ptr(), c2.stride(1))
        e1.record()
    e1.synchronize()
    t_dm = e0.elapsed_time(e1) / reps
    with torch.cuda.stream(st):
        e0.record()
        for _ in range(reps):
            eng.gemm_emulated(*args, c.data_ptr(), c.stride(1))
        e1.record()
    e1.synchronize()
    t_oz = e0.elapsed_time(e1) / reps
    print(f"{name:9s} {M}x{N}x{K}: err/|A||B| ozaki {e_oz:.2e} dmma {e_dm:.2e}   "
          f"time ozaki(incl slicing) {t_oz*1e3:.1f} us dmma {t_dm*1e3:.1f} us", flush=True)
