"""A/B timing of the A-pass kernel at the BASELINE config 4 shape (100000 x 20000, b = 100)
across environment variants, each in its own process (the switches are read once).

    python tools/ozaki_ab.py "FQB_OZ_L2HINT=0" "FQB_OZ_L2HINT=1" ...
Prints, per variant, the TN (W = A'Y) and NN (Y = A G) k_ozaki launch (+ fixup) times on
pre-sliced operands (fqb_sliced_gemm_again), CUDA events, mean of 10 after 3 warm-ups.
"""
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
out = []
with eng.slice_operand(a.data_ptr(), m, n, m) as sl:
    for name, trans in (("tn", True), ("nn", False)):
        k, rows = (m, n) if trans else (n, m)
        x = torch.randn((b, k), dtype=torch.float64, device="cuda").t()
        c = torch.empty((b, rows), dtype=torch.float64, device="cuda").t()
        sl.gemm(trans, b, 1.0, x.data_ptr(), k, 0.0, c.data_ptr(), rows)
        for _ in range(3):
            sl.gemm_again(1.0, 0.0, c.data_ptr(), rows)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            sl.gemm_again(1.0, 0.0, c.data_ptr(), rows)
        e1.record(); e1.synchronize()
        out.append(f"{name} {e0.elapsed_time(e1) / 10:.3f} ms")
print("  ".join(out))
'''

if __name__ == "__main__":
    variants = sys.argv[1:] or [""]
    shape = os.environ.get("AB_SHAPE", "100000,20000,100").split(",")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for v in variants:
        env = dict(os.environ)
        for kv in v.split():
            k, val = kv.split("=", 1)
            env[k] = val
        r = subprocess.run([sys.executable, "-c", CODE] + shape, env=env, cwd=root, capture_output=True, text=True)
        print(f"{v or 'default':40s} {r.stdout.strip()} {r.stderr.strip()[-300:] if r.returncode else ''}", flush=True)
