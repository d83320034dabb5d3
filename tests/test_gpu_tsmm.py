"""The tall-skinny b x b products of the CholeskyQR steps (tsmm.cu) against torch FP64:
fqb_gram (S = Y'Y from the upper tiles mirrored, per-SM partials summed in a fixed order)
and fqb_mul_upper (Z = Y R, R upper triangular, its lower part never read).

Bars: FP64 GEMM class -- |S - Y'Y| <= 1e-14 K max|S|, exact symmetry, bitwise
repeatability; |Z - Y triu(R)| <= 1e-14 b max(|Y| |R|).  b > 128 (Gram) / b > 104 (Y R) take
the general GEMM.
"""
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2506_03859_b200 as fqb  # noqa: E402


@pytest.fixture(scope="module")
def eng():
    return fqb.default_engine(0)


def colmajor(r, c, ld=None, seed=0):
    g = torch.Generator().manual_seed(seed)
    ld = ld or r
    buf = torch.randn((c, ld), dtype=torch.float64, generator=g).cuda()
    return buf.t()[:r, :]   # r x c view, stride (1, ld)


@pytest.mark.parametrize("k,b", [(100000, 100), (20000, 100), (8000, 50), (77, 13), (33, 1), (5, 7), (4096, 104),
                                 (4097, 105), (3000, 128), (500, 130), (1, 64), (100001, 64)])
def test_gram_matches_torch(eng, k, b):
    y = colmajor(k, b, seed=k + b)
    s = eng.gram(y)
    ref = y.t() @ y
    assert torch.equal(s, s.t())
    err = (s - ref).abs().max().item()
    assert err <= 1e-14 * max(k, 16) * ref.abs().max().item()
    assert torch.equal(eng.gram(y), s)   # deterministic


def test_gram_odd_leading_dimension(eng):
    y = colmajor(5001, 100, ld=5003, seed=3)
    s = eng.gram(y)
    ref = y.t() @ y
    assert (s - ref).abs().max().item() <= 1e-14 * 5001 * ref.abs().max().item()


@pytest.mark.parametrize("m,b", [(100000, 100), (20000, 100), (8000, 50), (65, 13), (1, 1), (129, 104), (300, 105),
                                 (1000, 128), (64, 64), (100003, 20)])
def test_mul_upper_matches_torch(eng, m, b):
    y = colmajor(m, b, seed=m)
    r = colmajor(b, b, seed=m + 1).t().contiguous().t()   # column-major b x b
    r_poison = r.clone()
    idx = torch.tril_indices(b, b, -1)
    r_poison[idx[0], idx[1]] = float("nan")   # the strictly lower part must not be read
    z = eng.mul_upper(y, r_poison)
    ref = y @ torch.triu(r)
    scale = (y.abs() @ torch.triu(r).abs()).max().item()
    assert torch.isfinite(z).all()
    assert (z - ref).abs().max().item() <= 1e-14 * b * scale


def test_mul_upper_odd_leading_dimension(eng):
    y = colmajor(7777, 100, ld=7781, seed=5)
    r = torch.triu(colmajor(100, 100, seed=6)).t().contiguous().t()
    z = eng.mul_upper(y, r)
    ref = y @ r
    assert (z - ref).abs().max().item() <= 1e-14 * 100 * (y.abs() @ r.abs()).max().item()
