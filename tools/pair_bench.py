"""A pass with b > 64 (BASELINE config 4 shape, 100000 x 20000, b = 100): the sliced-A
INT8 GEMM with two column chunks run sequentially (FQB_OZ_PAIR=0) vs on CTA pairs that
share every A tile through cluster multicast (default).  Each variant in its own process
(the switch is read once)."""
import os
import subprocess
import sys

CODE = r'''
import sys, torch
sys.path.insert(0, ".")
import paper_2506_03859_b200 as fqb
eng = fqb.default_engine(0)
m, n, b = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
a = torch.randn((n, m), dtype=torch.float64, device="cuda").t()
y = torch.randn((b, m), dtype=torch.float64, device="cuda").t()
w = torch.empty((b, n), dtype=torch.float64, device="cuda").t()
g = torch.randn((b, n), dtype=torch.float64, device="cuda").t()
yn = torch.empty((b, m), dtype=torch.float64, device="cuda").t()
with eng.slice_operand(a.data_ptr(), m, n, m) as sl:
    for name, trans, bp, cp in (("TN W=A'Y", True, y, w), ("NN Y=AG", False, g, yn)):
        for _ in range(3):
            sl.gemm(trans, b, 1.0, bp.data_ptr(), bp.stride(1), 0.0, cp.data_ptr(), cp.stride(1))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            sl.gemm(trans, b, 1.0, bp.data_ptr(), bp.stride(1), 0.0, cp.data_ptr(), cp.stride(1))
        e1.record(); e1.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"  {name}: {ms:.3f} ms  ({8.0 * m * n / ms / 1e6:.0f} GB/s of A slices)")
    # accuracy spot check against FP64 (cuBLAS via torch)
    ref = a.t() @ y
    sl.gemm(True, b, 1.0, y.data_ptr(), y.stride(1), 0.0, w.data_ptr(), w.stride(1))
    print("  max rel err vs torch FP64:", float((w - ref).abs().max() / ref.abs().max()))
'''
m, n, b = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (100000, 20000, 100)))
for pair in ("0", "1"):
    env = dict(os.environ, FQB_OZ_PAIR=pair)
    print(f"FQB_OZ_PAIR={pair}  ({m} x {n}, b = {b})", flush=True)
    subprocess.run([sys.executable, "-c", CODE, str(m), str(n), str(b)], env=env, check=True)
