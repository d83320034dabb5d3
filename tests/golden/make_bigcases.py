"""Golden runs of the UNMODIFIED reference at BASELINE configs 4 and 3 (full size).

    python tests/golden/make_bigcases.py c4 [c3]

Writes tests/golden/c4.json / c3.json.  The matrix is made on the CPU by the host
twin of the deterministic generator (oracle/detgen.c, fqo_det_lowrank), which is
bit-identical to the GPU's fqb_gen_lowrank_det: the GPU test regenerates it on the
device, checks the 64-bit fingerprint recorded here (fqo_checksum == fqb_checksum)
and the sampled entries, and then compares its factorization with this one.  Omega
is the oracle's fixed-zeta generator (bit-identical to the device's, detmath.h),
fed to the reference through its BlockSource plugin (driver.hpp:67-73).

The reference runs single-threaded (kernels.hpp:5-8) through its public granular
API (make_state / power_iterate_block / accept_block / assemble_svd, the steps of
run_fixed_precision, driver.cpp:347-388) so the per-block E trace is recorded; the
wall time of that call is stored with the host's CPU model.  Q.B parity is carried
by probes, since U, V do not fit a fixture: the reference's U diag(sigma) V' at
4096 random entries and applied to two Gaussian vectors (every 50th row kept).

TEST INFRASTRUCTURE: run here once (hours for c4); the JSON is committed.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import PORT_LIB, SPARSE_GAUSSIAN, SPARSE_SIGN, Oracle  # noqa: E402

CASES = {
    # BASELINE configs[3]: 100000 x 20000, rank 2000, sigma_i = 10^(-3i/2000) (i = 1..2000),
    # sparse Gaussian zeta = 8, b = 100, P = 2, eps = 1e-3 relative
    "c4": dict(m=100000, n=20000, sigma=("pow10", 2000, 3.0), noise=0.0, kind=SPARSE_GAUSSIAN, zeta=8, block=100,
               power=2, eps=1e-3, max_iters=0),
    # config 4's matrix with the reference's own default StdBernoulli (p = ln n / n, sparse and
    # centered: z = p A 1 and B's row sums in every product), b = 100, P = 1, first 4 blocks
    "c4sb": dict(m=100000, n=20000, sigma=("pow10", 2000, 3.0), noise=0.0, kind=2, zeta=0, block=100,
                 power=1, eps=1e-3, max_iters=4),
    # BASELINE configs[2]: 20000^2, rank-1000 signal sigma_i = (1+i)^-1.5 (i = 0..999) + 1e-4 N(0,1)/sqrt(n),
    # sparse sign zeta = 8, b = 64, P = 1, eps = 1e-2; unreachable, so capped at 6 blocks
    "c3": dict(m=20000, n=20000, sigma=("inv15", 1000), noise=1e-4, kind=SPARSE_SIGN, zeta=8, block=64, power=1,
               eps=1e-2, max_iters=6),
}
SEED_A, SEED_OMEGA = 42, 7


def sigma_of(spec) -> np.ndarray:
    if spec[0] == "pow10":
        r, dec = spec[1], spec[2]
        return 10.0 ** (-dec * np.arange(1, r + 1, dtype=np.float64) / r)
    r = spec[1]
    return (1.0 + np.arange(0, r, dtype=np.float64)) ** -1.5


def det_lib():
    lib = C.CDLL(PORT_LIB)
    lib.fqo_det_lowrank.argtypes = [C.c_int64, C.c_int64, C.c_int, C.c_void_p, C.c_uint64, C.c_double, C.c_int64,
                                    C.c_int64, C.c_void_p, C.c_int64]
    lib.fqo_checksum.restype = C.c_uint64
    lib.fqo_checksum.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64]
    return lib


def port_default_density(kind: int, n: int) -> float:
    """driver.cpp:449-455 (the oracle port's fqo_default_density)."""
    lib = C.CDLL(PORT_LIB)
    lib.fqo_default_density.restype = C.c_double
    lib.fqo_default_density.argtypes = [C.c_int, C.c_int]
    return float(lib.fqo_default_density(kind, n))


def noise_scale(case) -> float:
    return float(case["noise"]) / float(np.sqrt(case["n"])) if case["noise"] else 0.0


def make(name: str) -> dict:
    case = CASES[name]
    m, n = case["m"], case["n"]
    sig = sigma_of(case["sigma"])
    lib = det_lib()
    t0 = time.time()
    a = np.empty((n, m), dtype=np.float64).T          # column-major m x n
    st = lib.fqo_det_lowrank(m, n, len(sig), sig.ctypes.data, SEED_A, noise_scale(case), 0, m, a.ctypes.data, m)
    assert st == 0, st
    t_gen = time.time() - t0
    csum = int(lib.fqo_checksum(a.ctypes.data, m, n, m, 0, m))
    rng = np.random.default_rng(20261020)
    si = rng.integers(0, m, 64)
    sj = rng.integers(0, n, 64)
    print(f"[{name}] A generated in {t_gen:.1f} s, checksum {csum:016x}", flush=True)

    port = Oracle("port")
    ref = Oracle("reference")

    p_eff = 0.0 if case["zeta"] else port_default_density(case["kind"], n)

    def src(nn, bb, bid):
        return port.gen_sketch(case["kind"], p_eff, SEED_OMEGA, nn, bb, bid, zeta=case["zeta"])

    t0 = time.perf_counter()
    res = ref.run(a, eps=case["eps"], power=case["power"], block=case["block"], kind=case["kind"], seed=SEED_OMEGA,
                  zeta=case["zeta"], max_iters=case["max_iters"], relative=True, source=src, want_vectors=True,
                  traced=True)
    t_ref = time.perf_counter() - t0
    print(f"[{name}] reference: status {res.status} rank {res.rank} blocks {res.blocks} in {t_ref:.1f} s",
          flush=True)
    samples = [float(a[i, j]) for i, j in zip(si, sj)]
    del a
    u, v, s = res.u, res.v, res.sigma
    # probes of the reference's U diag(sigma) V'
    pi = rng.integers(0, m, 4096)
    pj = rng.integers(0, n, 4096)
    ent = np.einsum("ik,k,ik->i", u[pi], s, v[pj])
    probes = []
    for t in range(2):
        x = np.random.default_rng(100 + t).standard_normal(n)
        y = u @ (s * (v.T @ x))
        probes.append({"seed": 100 + t, "rows_step": 50, "y": y[::50].tolist(), "norm": float(np.linalg.norm(y))})
    cpu = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    cpu = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {
        "case": name, "m": m, "n": n, "sigma_spec": list(case["sigma"]), "noise": case["noise"],
        "noise_scale": noise_scale(case), "seed_a": SEED_A, "seed_omega": SEED_OMEGA, "kind": case["kind"],
        "zeta": case["zeta"], "p": p_eff, "block": case["block"], "power": case["power"], "eps": case["eps"],
        "max_iters": case["max_iters"],
        "checksum": f"{csum:016x}", "a_samples": {"i": si.tolist(), "j": sj.tolist(), "v": samples},
        "status": res.status, "rank": res.rank, "blocks": res.blocks, "converged": res.converged,
        "block_ids": res.block_ids, "block_residuals": res.block_residuals.tolist(),
        "residual_sq": res.residual_sq, "norm_a_sq": res.norm_a_sq, "sigma": s.tolist(),
        "qb_entries": {"i": pi.tolist(), "j": pj.tolist(), "v": ent.tolist()},
        "qb_probes": probes,
        "reference_seconds": t_ref, "generate_seconds": t_gen, "reference_threads": 1,
        "host": {"cpu": cpu, "nproc": os.cpu_count(), "machine": platform.machine()},
        "how": "tests/golden/make_bigcases.py: oracle/detgen.c matrix, oracle/_ref traced reference run",
    }


if __name__ == "__main__":
    for nm in sys.argv[1:] or ["c3"]:
        out = make(nm)
        path = os.path.join(ROOT, "tests", "golden", f"{nm}.json")
        with open(path, "w") as f:
            json.dump(out, f)
        print(f"wrote {path}", flush=True)
