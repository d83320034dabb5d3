"""Host side of the deterministic generator (oracle/detgen.c, include/farqb/detmath.h).

The GPU twin is compared bit for bit in tests/test_gpu_bigcases.py; here: the libm-free
log / Box-Muller are accurate, the factors are orthonormal (A's singular values are
sigma), row shards are bit-equal to rows of the whole, the fingerprint is additive over
shards, the thread count changes nothing, and the committed golden fingerprints are
reproduced from their seeds.
"""
import ctypes as C
import json
import math
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle.oracle import PORT_LIB

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    L = C.CDLL(PORT_LIB)
    L.fqo_det_log.restype = C.c_double
    L.fqo_det_log.argtypes = [C.c_double]
    L.fqo_det_box_muller.argtypes = [C.c_double, C.c_double, C.POINTER(C.c_double)]
    L.fqo_det_lowrank.argtypes = [C.c_int64, C.c_int64, C.c_int, C.c_void_p, C.c_uint64, C.c_double, C.c_int64,
                                  C.c_int64, C.c_void_p, C.c_int64]
    L.fqo_checksum.restype = C.c_uint64
    L.fqo_checksum.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64]
    return L


def _gen(lib, m, n, sig, seed, ns, row0=0, rows=None):
    rows = m - row0 if rows is None else rows
    a = np.empty((n, rows)).T
    assert lib.fqo_det_lowrank(m, n, len(sig), sig.ctypes.data, seed, ns, row0, rows, a.ctypes.data, rows) == 0
    return a


def test_det_log_and_box_muller_accuracy(lib):
    xs = np.random.default_rng(1).random(20000)
    worst = max(abs(lib.fqo_det_log(float(x)) - math.log(x)) / abs(math.log(x)) for x in xs if x != 1.0)
    assert worst < 4 * 2.2e-16
    for x in (2.0 ** -53, 0.5, 0.7071067811865476, 0.7071067811865477, 1.0 - 2 ** -53):
        assert abs(lib.fqo_det_log(x) - math.log(x)) <= 4 * 2.2e-16 * abs(math.log(x))
    z = (C.c_double * 2)()
    for u1, u2 in zip(xs[:3000], xs[3000:6000]):
        lib.fqo_det_box_muller(u1, u2, z)
        r = math.sqrt(-2 * math.log(u1))
        assert abs(z[0] - r * math.cos(2 * math.pi * u2)) <= 1e-15 * max(r, 1)
        assert abs(z[1] - r * math.sin(2 * math.pi * u2)) <= 1e-15 * max(r, 1)


def test_lowrank_spectrum_shards_and_fingerprint(lib):
    m, n, r = 1500, 700, 90
    sig = 10.0 ** (-3.0 * np.arange(1, r + 1) / r)
    a = _gen(lib, m, n, sig, 42, 0.0)
    s = np.linalg.svd(a, compute_uv=False)[:r]
    assert np.max(np.abs(s - sig)) <= 1e-13
    b = _gen(lib, m, n, sig, 42, 0.0, row0=400, rows=333)
    assert np.array_equal(b, a[400:733])
    h = lib.fqo_checksum(a.ctypes.data, m, n, m, 0, m)
    parts = (lib.fqo_checksum(a.ctypes.data, 400, n, m, 0, m) + lib.fqo_checksum(b.ctypes.data, 333, n, 333, 400, m)
             + lib.fqo_checksum(a.ctypes.data + 733 * 8, m - 733, n, m, 733, m)) % 2**64
    assert parts == h
    c = _gen(lib, m, n, sig, 43, 0.0)
    assert lib.fqo_checksum(c.ctypes.data, m, n, m, 0, m) != h


def test_thread_count_does_not_change_bits():
    code = ("import ctypes as C, numpy as np, sys; sys.path.insert(0, %r);"
            "from oracle.oracle import PORT_LIB; L = C.CDLL(PORT_LIB);"
            "L.fqo_det_lowrank.argtypes = [C.c_int64, C.c_int64, C.c_int, C.c_void_p, C.c_uint64, C.c_double,"
            " C.c_int64, C.c_int64, C.c_void_p, C.c_int64];"
            "L.fqo_checksum.restype = C.c_uint64;"
            "L.fqo_checksum.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64];"
            "s = (1.0 + np.arange(120)) ** -1.5; a = np.empty((611, 1333)).T;"
            "L.fqo_det_lowrank(1333, 611, 120, s.ctypes.data, 9, 1e-4, 0, 1333, a.ctypes.data, 1333);"
            "print(L.fqo_checksum(a.ctypes.data, 1333, 611, 1333, 0, 1333))") % ROOT
    outs = set()
    for t in ("1", "3", "8"):
        env = dict(os.environ, OMP_NUM_THREADS=t)
        outs.add(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                                check=True).stdout.strip())
    assert len(outs) == 1


@pytest.mark.parametrize("name", ["c3"])
def test_golden_fingerprint_reproduces(lib, name):
    """The committed golden case's matrix is what its seed makes (c3: 20000^2, ~25 s)."""
    p = os.path.join(ROOT, "tests", "golden", f"{name}.json")
    if not os.path.exists(p):
        pytest.skip("golden case not generated")
    with open(p) as f:
        g = json.load(f)
    spec = g["sigma_spec"]
    sig = ((1.0 + np.arange(spec[1])) ** -1.5 if spec[0] == "inv15"
           else 10.0 ** (-spec[2] * np.arange(1, spec[1] + 1) / spec[1]))
    a = _gen(lib, g["m"], g["n"], sig, g["seed_a"], g["noise_scale"])
    assert f"{lib.fqo_checksum(a.ctypes.data, g['m'], g['n'], g['m'], 0, g['m']):016x}" == g["checksum"]
    assert [float(a[i, j]) for i, j in zip(g["a_samples"]["i"], g["a_samples"]["j"])] == g["a_samples"]["v"]
