"""The b x b Cholesky of the CholeskyQR steps (fqb_chol_factor <- rsvd::chol_factor,
matrix_core.cpp:117-140) against numpy: R = L', R^-1, and the relative pivot floor.

Sizes cover the register-resident kernel (n <= 128, its 8-row slot groups ragged) and the
shared/global-memory kernel above 128.  Tolerances: ||R'R - Z|| <= 1e-13 ||Z||,
||R R^-1 - I|| <= 1e-13 cond(Z)^(1/2)-scaled, R against numpy's factor 1e-12 relative.
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


def spd(n, cond, seed):
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    ev = np.logspace(0, -np.log10(cond), n)
    return (q * ev) @ q.T


@pytest.mark.parametrize("n", [1, 2, 15, 16, 17, 31, 33, 50, 64, 100, 127, 128, 129, 200])
@pytest.mark.parametrize("cond", [10.0, 1e8])
def test_chol_matches_numpy(eng, n, cond):
    z = spd(n, cond, 100 + n)
    zd = torch.from_numpy(z).cuda()
    r, ri, bad = eng.chol_factor(zd, pivot_tol=0.0)
    assert not bad
    r, ri = r.cpu().numpy(), ri.cpu().numpy()
    assert np.all(np.tril(r, -1) == 0.0) and np.all(np.tril(ri, -1) == 0.0)
    nz = np.linalg.norm(z)
    assert np.linalg.norm(r.T @ r - z) <= 1e-13 * nz * max(1.0, n / 16)
    assert np.linalg.norm(r @ ri - np.eye(n)) <= 1e-13 * np.sqrt(cond) * n
    ref = np.linalg.cholesky(z).T
    assert np.linalg.norm(r - ref) <= 1e-12 * np.sqrt(cond) * np.linalg.norm(ref)


@pytest.mark.parametrize("n", [40, 100, 128, 160])
def test_chol_pivot_floor(eng, n):
    # Z = L L' with chosen pivots: pivot j of the Schur complement is l_jj^2
    rng = np.random.default_rng(n)
    L = np.tril(rng.standard_normal((n, n)) * 0.1, -1)
    d = np.ones(n)
    j_small = n // 2 + 3
    d[j_small] = 1e-7
    np.fill_diagonal(L, np.sqrt(d))
    z = L @ L.T
    zd = torch.from_numpy(z).cuda()
    # the floor below the small pivot: a valid factor
    _, _, bad = eng.chol_factor(zd, pivot_tol=1e-9)
    assert not bad
    # above it: rank deficient, identity outputs
    r, ri, bad = eng.chol_factor(zd, pivot_tol=1e-6)
    assert bad
    assert np.array_equal(r.cpu().numpy(), np.eye(n)) and np.array_equal(ri.cpu().numpy(), np.eye(n))
    # diag_ref overrides max_diag: 1e-9 * 1e3 = 1e-6 > 1e-7 -> deficient
    _, _, bad = eng.chol_factor(zd, pivot_tol=1e-9, diag_ref=1e3)
    assert bad


@pytest.mark.parametrize("n", [16, 100])
def test_chol_nonpositive_and_nan(eng, n):
    z = spd(n, 10.0, 7)
    z[5, 5] = -1.0
    _, _, bad = eng.chol_factor(torch.from_numpy(z).cuda(), pivot_tol=0.0)
    assert bad
    z = spd(n, 10.0, 8)
    z[n - 1, n - 1] = np.nan
    _, _, bad = eng.chol_factor(torch.from_numpy(z).cuda(), pivot_tol=0.0)
    assert bad


def test_chol_deterministic(eng):
    z = torch.from_numpy(spd(100, 100.0, 9)).cuda()
    r1, i1, _ = eng.chol_factor(z, pivot_tol=0.0)
    r2, i2, _ = eng.chol_factor(z, pivot_tol=0.0)
    assert torch.equal(r1, r2) and torch.equal(i1, i2)
