"""Elementwise error of the FP64 products on the B200: cuBLAS DGEMM (torch.matmul) and the
INT8 emulation (fqb_gemm_emulated, the k_ozaki path), against an extended-precision
(x87 long double) product, on sampled entries.

    [FQB_OZ_DIAGS=7] python tools/ozaki_accuracy.py

Per shape (C = A' B, A k x m, B k x n, randn, and a low-rank A like the bench's) prints
max over sampled entries of |C - C_exact| / (|A'| |B|)_ij  and  / (u * (|A'| |B|)_ij)
for each method.  The emulation variant is whatever the process's FQB_OZ_DIAGS selects.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_03859_b200 as fqb  # noqa: E402

U = 2.0 ** -53


def emulated(eng, a, b):
    """C = A' B through fqb_gemm_emulated (device pointers)."""
    k, m = a.shape
    n = b.shape[1]
    ad = a.t().contiguous().t().cuda()            # k x m column-major
    bd = b.t().contiguous().t().cuda()
    cd = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()
    eng.gemm_emulated(True, m, n, k, 1.0, ad.data_ptr(), k, bd.data_ptr(), k, 0.0, cd.data_ptr(), m)
    torch.cuda.synchronize()
    return cd.cpu()


def errors(got, a, b, rows, cols):
    ar = a[:, rows].numpy().astype(np.longdouble)
    bc = b[:, cols].numpy().astype(np.longdouble)
    exact = ar.T @ bc
    bound = np.abs(ar).T @ np.abs(bc)
    err = np.abs(got[rows][:, cols].numpy().astype(np.longdouble) - exact)
    r = err / bound
    return float(r.max()), float(r.mean())


def main():
    eng = fqb.default_engine(0)
    diags = os.environ.get("FQB_OZ_DIAGS", "8")
    print(f"emulation: 7 slices, diagonals d <= {int(diags) - 1}")
    g = torch.Generator().manual_seed(5)
    for k, m, n, kind in ((65, 512, 50, "randn"), (1000, 512, 50, "randn"), (20000, 256, 50, "randn"),
                          (100000, 128, 100, "randn"), (100000, 128, 100, "lowrank")):
        if kind == "randn":
            a = torch.randn((k, m), dtype=torch.float64, generator=g)
        else:   # columns of a rank-100 matrix with decaying spectrum (the bench's A is such a product)
            x = torch.randn((k, 100), dtype=torch.float64, generator=g)
            y = torch.randn((100, m), dtype=torch.float64, generator=g)
            a = (x * (10.0 ** (-3.0 * torch.arange(1, 101, dtype=torch.float64) / 100))) @ y
        b = torch.randn((k, n), dtype=torch.float64, generator=g)
        rows = np.arange(0, m, max(1, m // 32))
        cols = np.arange(n)
        dg = (a.cuda().t() @ b.cuda()).cpu()
        em = emulated(eng, a, b)
        e_d = errors(dg, a, b, rows, cols)
        e_e = errors(em, a, b, rows, cols)
        print(f"k={k:6d} m={m:4d} n={n:3d} {kind:8s}  DGEMM max {e_d[0]:.2e} ({e_d[0] / U:5.2f} u) mean "
              f"{e_d[1]:.2e}   emulated max {e_e[0]:.2e} ({e_e[0] / U:5.2f} u) mean {e_e[1]:.2e}", flush=True)


if __name__ == "__main__":
    main()
