"""The k_ozaki schedule switches, each read once per process, so every variant runs in a
subprocess: FQB_OZ_WIDE=0/1 (the same 34 exact int32 products in 14 or 12 MMAs per
k-step -- identical bits) and FQB_OZ_DIAGS=7 (diagonals p + q <= 6 only: 28 products; its
error, measured against an extended-precision product, stays within a few u |A||B|, the
class of an FP64 DGEMM -- tools/ozaki_accuracy.py has the side-by-side numbers)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2506_03859_b200 as fqb
eng = fqb.default_engine(0)
out = []
for (trans, m, n, k, seed) in ((True, 700, 100, 5000, 1), (False, 900, 50, 3000, 2), (True, 300, 37, 65, 3)):
    g = torch.Generator().manual_seed(seed)
    a = torch.randn((k, m) if trans else (m, k), dtype=torch.float64, generator=g)
    b = torch.randn((k, n), dtype=torch.float64, generator=g)
    ad = a.t().contiguous().t().cuda(); bd = b.t().contiguous().t().cuda()
    c = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()
    eng.gemm_emulated(trans, m, n, k, 1.0, ad.data_ptr(), ad.stride(1), bd.data_ptr(), bd.stride(1), 0.0,
                      c.data_ptr(), m)
    torch.cuda.synchronize()
    out.append(c.cpu().numpy())
np.savez(sys.argv[2], *out)
'''


def _run(tmp_path, env_extra, tag):
    path = str(tmp_path / f"{tag}.npz")
    env = dict(os.environ)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", CODE, ROOT, path], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    with np.load(path) as z:
        return [z[f"arr_{i}"] for i in range(len(z.files))]


def _inputs():
    out = []
    for (trans, m, n, k, seed) in ((True, 700, 100, 5000, 1), (False, 900, 50, 3000, 2), (True, 300, 37, 65, 3)):
        g = torch.Generator().manual_seed(seed)
        a = torch.randn((k, m) if trans else (m, k), dtype=torch.float64, generator=g)
        b = torch.randn((k, n), dtype=torch.float64, generator=g)
        out.append(((a.t() if trans else a).numpy(), b.numpy()))
    return out


def test_wide_and_narrow_schedules_give_identical_bits(tmp_path):
    wide = _run(tmp_path, {"FQB_OZ_WIDE": "1"}, "wide")
    narrow = _run(tmp_path, {"FQB_OZ_WIDE": "0"}, "narrow")
    for w, nw in zip(wide, narrow):
        assert np.array_equal(w.view(np.uint64), nw.view(np.uint64))


@pytest.mark.parametrize("wide", ["0", "1"])
def test_trimmed_diagonals_stay_fp64_class(tmp_path, wide):
    got = _run(tmp_path, {"FQB_OZ_DIAGS": "7", "FQB_OZ_WIDE": wide}, f"d7w{wide}")
    full = _run(tmp_path, {"FQB_OZ_WIDE": wide}, f"d8w{wide}")
    u = 2.0 ** -53
    for c7, c8, (aa, b) in zip(got, full, _inputs()):
        rows = np.arange(0, aa.shape[0], 7)
        ar = aa[rows].astype(np.longdouble)
        exact = ar @ b.astype(np.longdouble)
        bound = np.abs(ar) @ np.abs(b).astype(np.longdouble)
        e7 = np.abs(c7[rows].astype(np.longdouble) - exact) / bound
        e8 = np.abs(c8[rows].astype(np.longdouble) - exact) / bound
        assert float(e7.max()) <= 8 * u           # measured up to ~5.4 u at k = 65
        assert float(e8.max()) <= 3.6 * u         # the full scheme (test_gpu_ozaki's 4e-16 bar)
        assert not np.array_equal(c7, c8)          # the trimmed kernel really ran


def test_s50_and_s56_spacings_give_identical_bits(tmp_path):
    """Chunks of <= 50 columns on 50-row Z slices (10 MMAs per k-step, diagonal 7 partly
    zeroed by tcgen05.st) against the 56-row spacing: the same exact int32 sums, so the same
    bits -- paired (n = 100), single (n = 50) and ragged (n = 37, k = 65) launches."""
    s50 = _run(tmp_path, {"FQB_OZ_S50": "1"}, "s50")
    s56 = _run(tmp_path, {"FQB_OZ_S50": "0"}, "s56")
    for a, b in zip(s50, s56):
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
