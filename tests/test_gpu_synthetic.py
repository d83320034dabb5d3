"""Device-side test matrices (synthetic.cu) against the reference's gen_synthetic.

tests/golden/matrices.npz holds the reference's own gen_synthetic outputs
(slow128: kind slow, n 128, seed 5; fast96: fast, 96, 68; slow200: slow, 200, 64;
made by tests/golden/make_golden.py from oracle/_ref).  The device run follows the
same algorithm (Philox Gaussian panels, two block Gram-Schmidt + CholeskyQR rounds
per panel, A = U diag(sigma) V') in a different summation order, and the Gaussians
differ by a few ulp (CUDA vs glibc libm): agreement to 1e-13 of max|A|.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2506_03859_b200 as fqb  # noqa: E402


@pytest.fixture(scope="module")
def eng():
    return fqb.default_engine(0)


@pytest.mark.parametrize("name,kind,n,seed", [("slow128", 0, 128, 5), ("fast96", 1, 96, 68), ("slow200", 0, 200, 64)])
def test_gen_synthetic_matches_reference(eng, golden_mats, name, kind, n, seed):
    a, r = eng.gen_synthetic(kind, n, seed)
    ref = golden_mats[name]
    got = a.cpu().numpy()
    assert got.shape == ref.shape
    assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()
    assert r == (n if kind == 0 else min(n, 828))


def test_random_orthonormal_is_orthonormal_and_deterministic(eng):
    q = eng.random_orthonormal(3000, 150, seed=9)
    qtq = (q.t() @ q).cpu().numpy()
    assert np.abs(qtq - np.eye(150)).max() < 1e-14
    q2 = eng.random_orthonormal(3000, 150, seed=9)
    assert torch.equal(q, q2)
    q3 = eng.random_orthonormal(3000, 150, seed=9, stream=0xFA000002)
    assert not torch.equal(q, q3)


def test_block_diagonal_v_kind(eng):
    a, r = eng.gen_synthetic(2, 120, seed=3, d=4)
    s = np.linalg.svd(a.cpu().numpy(), compute_uv=False)
    want = 1.0 / np.arange(1, 121, dtype=np.float64) ** 2
    assert np.abs(s - want).max() <= 1e-13


def test_gen_lowrank_spectrum_and_noise(eng):
    m, n, r = 5000, 1200, 300
    sig = 10.0 ** (-np.arange(1, r + 1) / 50.0)
    a = eng.gen_lowrank(m, n, sig, seed=42)
    s = torch.linalg.svdvals(a).cpu().numpy()
    assert np.abs(s[:r] - sig).max() <= 5e-12 and s[r:].max() <= 1e-13   # svdvals itself: ~1e-12
    an = eng.gen_lowrank(m, n, sig, seed=42, noise=1e-4)
    noise = (an - a).cpu().numpy()
    # N(0,1)/sqrt(n) entries scaled by 1e-4: Frobenius^2 ~ 1e-8 m
    assert abs(np.sum(noise ** 2) / (1e-8 * m) - 1.0) < 0.02
