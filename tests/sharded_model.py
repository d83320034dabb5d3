"""Numpy model of the engine's row-sharded QB loop.  TEST INFRASTRUCTURE ONLY.

Mirrors paper_2506_03859_b200/csrc/engine.cu step by step (explicit Q,
CholeskyQR2 + two-pass block Gram-Schmidt, B_j' = (W_j - B' C) R^-1,
E -= ||B_j||^2), with `allreduce` called at exactly the points where the
engine calls comm_allreduce_sum (csrc/comm.cu).  Run on CPU under
torch.distributed/gloo it checks that those reduction points give the same
factorization as an unsharded run (tests/test_multirank_cpu.py).
"""
from __future__ import annotations

import numpy as np


def _chol_upper(s: np.ndarray, tol: float, dref: float) -> np.ndarray | None:
    """R with R'R = S and the reference pivot rule (matrix_core.cpp:117-140)."""
    s = np.array(s, dtype=np.float64)
    b = s.shape[0]
    max_diag = dref if dref > 0 else float(np.max(np.diag(s)))
    l = np.zeros_like(s)
    for j in range(b):
        d = s[j, j] - l[j, :j] @ l[j, :j]
        if not d > tol * max_diag:
            return None
        l[j, j] = np.sqrt(d)
        l[j + 1:, j] = (s[j + 1:, j] - l[j + 1:, :j] @ l[j, :j]) / l[j, j]
    return l.T


def qb_sharded(a_local: np.ndarray, eps: float, power: int, b: int, max_iters: int, omega, allreduce):
    """Fixed-precision relative-eps QB on this rank's row block; returns
    (Q_local, Bt, rank, E, norm_a_sq, residual trace)."""
    m, n = a_local.shape
    norm = allreduce(np.array([np.sum(a_local * a_local)]))[0]
    eps_sq = (eps * np.sqrt(norm)) ** 2
    q = np.zeros((m, 0))
    bt = np.zeros((n, 0))
    trace = 0.0
    diag_max = 0.0
    trace_hist = []
    for j in range(max_iters):
        om = omega(n, b, j)
        if power >= 1:
            g = om
            for k in range(1, power + 1):
                y0 = a_local @ g
                w = allreduce(a_local.T @ y0)
                if bt.shape[1]:
                    w = w - bt @ (bt.T @ g)
                r = _chol_upper(w.T @ w, 0.0, 0.0)
                g = w @ np.linalg.inv(r)
            x = g
        else:
            x = om
        yj = a_local @ x
        wj = allreduce(a_local.T @ yj)
        cd = allreduce(np.hstack([q, yj]).T @ yj)
        l = q.shape[1]
        c1, d = cd[:l], cd[l:]
        dref = max(diag_max, float(np.max(np.diag(d))))
        if l:
            yp = yj - q @ c1
            s1 = allreduce(yp.T @ yp)
            r1 = _chol_upper(s1, 1e-12, dref)
        else:
            yp = yj
            r1 = _chol_upper(d, 1e-12, dref)
        if r1 is None:
            raise RuntimeError("degenerate block")
        q1 = yp @ np.linalg.inv(r1)
        if l:
            c2 = allreduce(q.T @ q1)
            q1 = q1 - q @ c2
        r2 = _chol_upper(allreduce(q1.T @ q1), 0.0, 0.0)
        qj = q1 @ np.linalg.inv(r2)
        rinv = np.linalg.inv(r1) @ np.linalg.inv(r2)
        if l:
            c = c1 + c2 @ r1
            wj = wj - bt @ c
        btj = wj @ rinv
        trace += float(np.sum(btj * btj))
        diag_max = dref
        q = np.hstack([q, qj])
        bt = np.hstack([bt, btj])
        trace_hist.append(norm - trace)
        if norm - trace < eps_sq:
            break
    return q, bt, q.shape[1], norm - trace, norm, trace_hist
