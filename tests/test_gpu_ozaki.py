"""The INT8 tensor-core FP64 emulation (ozaki.cu) behind fqb_gemm_emulated and the engine's A passes.

Accuracy bar: an FP64 GEMM's.  On a sample of rows, every element of C must be
within 4e-16 of the bound |A| |B| (elementwise absolute product) plus the final
rounding (2^-53 |C|) of the exact result, computed in extended precision
(numpy longdouble) -- what the slicing argument in ozaki.cu guarantees
(dropped terms ~2^-55 of max|row| * max|col|).  A plain FP64 reference would
itself be off by ~sqrt(K) u |A||B| and could not resolve this bar.
The engine with the emulation forced on must keep every parity property of the
FP64 path: identical rank / blocks / ids and E within 1e-10 ||A||^2.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2506_03859_b200 as fqb  # noqa: E402
from oracle.oracle import SketchArrays  # noqa: E402
from paper_2506_03859_b200 import FarpcaConfig, SketchSpec  # noqa: E402


@pytest.fixture(scope="module")
def eng():
    return fqb.default_engine(0)


def _run_emulated(eng, trans, a, b, c0, alpha, beta):
    """a: (k x m if trans else m x k), b: k x n, c0: m x n, all float64 CPU tensors."""
    m, n = c0.shape
    k = b.shape[0]
    ad = a.cuda().t().contiguous().t()
    bd = b.cuda().t().contiguous().t()
    cd = c0.cuda().t().contiguous().t()
    # column-major and contiguous: ld = rows (stride(1) is ambiguous for one column)
    eng.gemm_emulated(trans, m, n, k, alpha, ad.data_ptr(), ad.shape[0], bd.data_ptr(), bd.shape[0], beta,
                      cd.data_ptr(), cd.shape[0])
    torch.cuda.synchronize()
    return cd.cpu()


def _check_rows(got, aa, b, c0, alpha, beta, rows):
    """Extended-precision check of C[rows, :] (aa = op(A), m x k)."""
    ar = aa[rows].numpy().astype(np.longdouble)
    bl = b.numpy().astype(np.longdouble)
    exact = alpha * (ar @ bl) + beta * c0[rows].numpy().astype(np.longdouble)
    bound = abs(alpha) * (np.abs(ar) @ np.abs(bl)) + abs(beta) * np.abs(c0[rows].numpy())
    err = np.abs(got[rows].numpy().astype(np.longdouble) - exact)
    tol = 4e-16 * bound + 2.0 ** -53 * np.abs(exact) + 1e-300
    assert (err <= tol).all(), float(np.max(err / tol))


@pytest.mark.parametrize("trans", [True, False])
@pytest.mark.parametrize("m,n,k", [(8000, 50, 8000), (257, 33, 999), (128, 64, 64), (129, 1, 65), (1, 17, 3),
                                   (300, 64, 5000), (1000, 20, 127), (500, 56, 700), (500, 57, 700),
                                   (200, 49, 4096), (300, 50, 40000), (130, 100, 20000), (129, 7, 16385)])
def test_emulated_gemm_fp64_accuracy(eng, trans, m, n, k):
    g = torch.Generator(device="cpu").manual_seed(m + 3 * n + 7 * k + int(trans))
    a = torch.randn((k, m) if trans else (m, k), dtype=torch.float64, generator=g)
    b = torch.randn((k, n), dtype=torch.float64, generator=g)
    c0 = torch.randn((m, n), dtype=torch.float64, generator=g)
    got = _run_emulated(eng, trans, a, b, c0, 0.75, -0.5)
    aa = a.t() if trans else a
    rows = np.unique(np.linspace(0, m - 1, min(m, 48)).astype(int))
    _check_rows(got, aa, b, c0, 0.75, -0.5, rows)


def test_emulated_gemm_wild_scales_and_zero_lines(eng):
    """Rows / columns spanning 1e-150 .. 1e150, exact zero rows and columns, beta = 0."""
    m, n, k = 300, 40, 700
    g = torch.Generator(device="cpu").manual_seed(5)
    a = torch.randn((k, m), dtype=torch.float64, generator=g)          # trans: rows of C = columns of a
    a *= torch.logspace(-150, 150, m, dtype=torch.float64)
    a[:, 7] = 0.0
    a[13, :] = 0.0
    b = torch.randn((k, n), dtype=torch.float64, generator=g) * torch.logspace(-100, 100, n, dtype=torch.float64)
    b[:, 3] = 0.0
    c0 = torch.full((m, n), 7.0, dtype=torch.float64)
    got = _run_emulated(eng, True, a, b, c0, 1.0, 0.0)
    assert torch.isfinite(got).all()
    assert (got[7, :] == 0).all() and (got[:, 3] == 0).all()
    _check_rows(got, a.t(), b, c0, 1.0, 0.0, np.arange(0, m, 7))


@pytest.mark.parametrize("bad", [float("nan"), float("inf"), -float("inf")])
def test_emulated_gemm_non_finite_lines_give_nan(eng, bad):
    """An Inf/NaN in a row of op(A) or a column of B makes that row / column of C NaN (its
    digits are meaningless); every other element keeps the FP64 bar."""
    m, n, k = 260, 20, 300
    g = torch.Generator(device="cpu").manual_seed(11)
    a = torch.randn((k, m), dtype=torch.float64, generator=g)
    b = torch.randn((k, n), dtype=torch.float64, generator=g)
    a[17, 200] = bad        # row 200 of op(A) = A^T
    b[5, 4] = bad           # column 4 of B
    c0 = torch.zeros((m, n), dtype=torch.float64)
    got = _run_emulated(eng, True, a, b, c0, 1.0, 0.0)
    assert torch.isnan(got[200, :]).all() and torch.isnan(got[:, 4]).all()
    keep_r = np.array([r for r in range(0, m, 9) if r != 200])
    keep_c = [j for j in range(n) if j != 4]
    _check_rows(got[:, keep_c], a.t(), b[:, keep_c], c0[:, keep_c], 1.0, 0.0, keep_r)


def test_qb_non_finite_input_propagates(eng, monkeypatch):
    """Non-finite A: the engine stays on DMMA (the reference's Inf/NaN behaviour); no garbage result."""
    monkeypatch.setenv("FQB_OZAKI", "1")
    a = _lowrank(400, 300, 1.0 / np.arange(1, 41), seed=3)
    a[10, 20] = np.nan
    cfg = FarpcaConfig(eps=1e-2, power=1, block=20, sketch=SketchSpec(0, 0.0, 1), relative=True, max_iters=3)
    try:
        res = eng.run_fixed_precision(a, cfg, output="host")
    except fqb.RsvdError:
        return   # an error status (e.g. degenerate / tolerance) is acceptable
    assert not res.converged or not np.isfinite(res.residual_sq)


def test_emulated_gemm_is_deterministic(eng):
    m, n, k = 4000, 50, 6000
    g = torch.Generator(device="cpu").manual_seed(9)
    a = torch.randn((k, m), dtype=torch.float64, generator=g)
    b = torch.randn((k, n), dtype=torch.float64, generator=g)
    c = torch.zeros((m, n), dtype=torch.float64)
    r1 = _run_emulated(eng, True, a, b, c, 1.0, 0.0)
    r2 = _run_emulated(eng, True, a, b, c, 1.0, 0.0)
    assert torch.equal(r1, r2)


@pytest.mark.parametrize("n", [65, 100, 112, 113, 128, 200])
def test_emulated_gemm_wide_n_in_chunks(eng, n):
    """n > 64 runs as balanced chunks of <= 64 columns (config 4 has b = 100)."""
    m, k = 700, 900
    g = torch.Generator(device="cpu").manual_seed(n)
    a = torch.randn((k, m), dtype=torch.float64, generator=g)
    b = torch.randn((k, n), dtype=torch.float64, generator=g)
    c0 = torch.randn((m, n), dtype=torch.float64, generator=g)
    got = _run_emulated(eng, True, a, b, c0, 1.5, 0.25)
    _check_rows(got, a.t(), b, c0, 1.5, 0.25, np.arange(0, m, 13))


def _lowrank(m, n, sig, seed):
    rng = np.random.default_rng(seed)
    r = len(sig)
    u, _ = np.linalg.qr(rng.standard_normal((m, r)))
    v, _ = np.linalg.qr(rng.standard_normal((n, r)))
    return np.asfortranarray((u * sig) @ v.T)


@pytest.mark.parametrize("kind,zeta,power,block", [(2, 0, 2, 25), (0, 0, 1, 25), (3, 8, 3, 25), (4, 8, 0, 25),
                                                  (4, 8, 2, 100)])
def test_qb_with_emulation_matches_oracle(eng, port, monkeypatch, kind, zeta, power, block):
    """FQB_OZAKI=1 forces every A pass onto the INT8 tensor cores, even at this size (block 100: chunked)."""
    monkeypatch.setenv("FQB_OZAKI", "1")
    a = _lowrank(900, 700, 1.0 / np.arange(1, 251) ** 1.5, seed=40 + kind + power)
    p = 0.0 if kind == 0 or zeta else 0.5
    spec = SketchSpec(kind, p, 13, zeta=zeta)
    cfg = FarpcaConfig(eps=1e-2, power=power, block=block, sketch=spec, relative=True)
    res = eng.run_fixed_precision(a, cfg, output="host")

    def src(n, b, bid):
        s = eng.gen_sketch(spec, n, b, bid)
        if s.is_dense:
            return SketchArrays(True, s.rows, s.cols, dense=s.dense, p=s.p)
        return SketchArrays(False, s.rows, s.cols, col_ptr=s.col_ptr, row_idx=s.row_idx, values=s.values,
                            centered=s.centered, p=s.p, std_scale=s.std_scale)
    ref = port.run(a, eps=1e-2, power=power, block=block, kind=kind, p=p, seed=13, zeta=zeta, relative=True,
                   source=src)
    assert ref.status == 0 and res.converged
    assert (res.rank, res.blocks, res.block_ids) == (ref.rank, ref.blocks, ref.block_ids)
    na = ref.norm_a_sq
    assert abs(res.residual_sq - ref.residual_sq) <= 1e-10 * na
    assert np.max(np.abs(res.block_residuals - ref.block_residuals)) <= 1e-10 * na


def test_pass_timing_counts_the_a_passes(eng, monkeypatch):
    """fqb_set_pass_timing / fqb_pass_timing (the bench's live roofline timing): one event
    pair per A-pass k_ozaki launch -- 2P + 1 per block with a sparse Omega (P = 2: 5), the
    b = 100 block as one paired launch -- and 8 (MK + Kb + Mb) algorithmic bytes each."""
    monkeypatch.setenv("FQB_OZAKI", "1")
    m, n, b = 900, 700, 100
    a = _lowrank(m, n, 1.0 / np.arange(1, 251) ** 1.5, seed=5)
    cfg = FarpcaConfig(eps=1e-2, power=2, block=b, sketch=SketchSpec(4, 0.0, 13, zeta=8), relative=True)
    eng.set_pass_timing(True)
    res = eng.run_fixed_precision(a, cfg, output="host")
    ms, launches, nbytes = eng.pass_timing()
    eng.set_pass_timing(False)
    assert launches == 5 * res.blocks
    assert nbytes == pytest.approx(launches * 8.0 * (m * n + (m + n) * b), rel=1e-12)
    assert ms > 0.0
    eng.run_fixed_precision(a, cfg, output="host")            # disarmed: nothing more is recorded
    assert eng.pass_timing()[1] == 0


def test_emulation_on_and_off_agree(eng, monkeypatch):
    a = _lowrank(1500, 1200, 0.97 ** np.arange(300), seed=77)
    cfg = FarpcaConfig(eps=1e-3, power=2, block=40, sketch=SketchSpec(2, 0.5, 5), relative=True)
    monkeypatch.setenv("FQB_OZAKI", "1")
    r1 = eng.run_fixed_precision(a, cfg, output="host")
    monkeypatch.setenv("FQB_OZAKI", "0")
    r0 = eng.run_fixed_precision(a, cfg, output="host")
    assert (r1.rank, r1.blocks) == (r0.rank, r0.blocks)
    assert abs(r1.residual_sq - r0.residual_sq) <= 1e-11 * r0.norm_a_sq
    # different arithmetic (INT8 slices vs DMMA) -- so the emulation really ran ...
    assert not np.array_equal(r1.bt, r0.bt)
    # ... and Q B (unique for a given sketch) agrees to FP64 working accuracy
    qb1 = r1.q @ r1.bt.T
    qb0 = r0.q @ r0.bt.T
    assert np.abs(qb1 - qb0).max() <= 1e-10 * np.abs(a).max()


def test_sliced_operand_matches_one_shot_emulation(eng):
    """fqb_slice_operand + fqb_sliced_gemm (both layouts, repeated use) == fqb_gemm_emulated bit for bit."""
    m, n, nb = 1100, 900, 37
    g = torch.Generator(device="cpu").manual_seed(21)
    a = torch.randn((n, m), dtype=torch.float64, generator=g).cuda().t()        # m x n column-major
    with eng.slice_operand(a.data_ptr(), m, n, m) as sl:
        for trans in (True, False):
            k, rows = (m, n) if trans else (n, m)
            b = torch.randn((nb, k), dtype=torch.float64, generator=g).cuda().t()
            c0 = torch.randn((nb, rows), dtype=torch.float64, generator=g).cuda().t()
            c1, c2 = c0.clone(), c0.clone()
            for _ in range(2):
                c1.copy_(c0)
                sl.gemm(trans, nb, 0.5, b.data_ptr(), k, 2.0, c1.data_ptr(), rows)
            eng.gemm_emulated(trans, rows, nb, k, 0.5, a.data_ptr(), m, b.data_ptr(), k, 2.0, c2.data_ptr(), rows)
            torch.cuda.synchronize()
            assert torch.equal(c1, c2)
            want = 0.5 * ((a.t() if trans else a).cpu() @ b.cpu()) + 2.0 * c0.cpu()
            assert (c1.cpu() - want).abs().max().item() < 1e-12
    with pytest.raises(fqb.InvalidArgument):
        sl.gemm(True, nb, 1.0, b.data_ptr(), m, 0.0, c1.data_ptr(), n)


@pytest.mark.parametrize("m,n,nb", [(1100, 900, 37), (1000, 200, 100), (960, 130, 60), (64, 65, 8),
                                    (3000, 2000, 100), (1088, 1, 50), (5000, 257, 128)])
def test_sliced_gemm_mn_fp64_accuracy(eng, m, n, nb):
    """fqb_sliced_gemm_mn: A B from the A'Y-layout slices read MN-major (the engine's
    Y -= Q C), against an extended-precision product: odd numbers of 64-row k-blocks (the
    last row tile's second half absent), K not a multiple of 64, one chunk (S = 56 and
    S = 64) and paired chunks, alpha / beta.
    The scales are per column of A here, so the bound is normwise per column:
    |err_ij| <= 4e-16 sum_k max_i|A_ik| |B_kj| (+ 2^-53 |C_ij|) -- a row much smaller than
    its columns' maxima keeps absolute, not relative, accuracy (the engine's Q rows: the
    projection Y -= Q C only needs ||err|| small against ||C||)."""
    g = torch.Generator(device="cpu").manual_seed(m + n + nb)
    a = torch.randn((m, n), dtype=torch.float64, generator=g)
    a[:, ::7] *= 1e-3                                    # column scales differ
    a[::5, :] *= 1e-2                                    # and row scales
    b = torch.randn((n, nb), dtype=torch.float64, generator=g)
    c0 = torch.randn((m, nb), dtype=torch.float64, generator=g)
    ad = a.t().contiguous().t().cuda()
    bd = b.t().contiguous().t().cuda()
    c = c0.t().contiguous().t().cuda()
    with eng.slice_operand(ad.data_ptr(), m, n, m) as sl:
        sl.gemm_mn(nb, 0.75, bd.data_ptr(), n, -0.5, c.data_ptr(), m)
        torch.cuda.synchronize()
    rows = np.unique(np.linspace(0, m - 1, min(m, 64)).astype(int))
    an = a.numpy().astype(np.longdouble)
    bn = b.numpy().astype(np.longdouble)
    exact = 0.75 * (an[rows] @ bn) - 0.5 * c0.numpy()[rows].astype(np.longdouble)
    cmax = np.abs(an).max(axis=0)                          # per column of A
    bound = 0.75 * (cmax @ np.abs(bn))[None, :] + 0.5 * np.abs(c0.numpy()[rows])
    err = np.abs(c.cpu().numpy()[rows].astype(np.longdouble) - exact)
    tol = 4e-16 * bound + 2.0 ** -53 * np.abs(exact) + 1e-300
    assert (err <= tol).all(), float(np.max(err / tol))


@pytest.mark.parametrize("nb", [50, 100, 128])
def test_sliced_gemm_again_reuses_b_slices(eng, nb):
    """fqb_sliced_gemm_again: the previous product on the same B slices, bit for bit,
    with new alpha / beta (one chunk, and the paired two-chunk launch)."""
    m, n = 900, 700
    g = torch.Generator(device="cpu").manual_seed(nb)
    a = torch.randn((n, m), dtype=torch.float64, generator=g).t().contiguous().t().cuda()
    for trans, k, rows in ((True, m, n), (False, n, m)):
        b = torch.randn((nb, k), dtype=torch.float64, generator=g).t().cuda()
        c1 = torch.empty((nb, rows), dtype=torch.float64, device="cuda").t()
        c2 = torch.randn((nb, rows), dtype=torch.float64, device="cuda").t()
        c2_0 = c2.clone()
        with eng.slice_operand(a.data_ptr(), m, n, m) as sl:
            sl.gemm(trans, nb, 1.0, b.data_ptr(), k, 0.0, c1.data_ptr(), rows)
            sl.gemm_again(-2.0, 0.5, c2.data_ptr(), rows)
        torch.cuda.synchronize()
        assert torch.equal(c2, 0.5 * c2_0 - 2.0 * c1) or torch.allclose(c2, 0.5 * c2_0 - 2.0 * c1, rtol=0, atol=1e-12)


def test_tile_result_independent_of_tmem_history(eng):
    """Every accumulator diagonal is (re)initialised per tile: a CTA's 4th tile equals the
    same rows computed alone (the top diagonal of the 7-slice scheme has no sp = 0 product
    and once accumulated onto the previous tile's sum)."""
    M, K, N = 296 * 128, 64, 50          # 296 row tiles, one k-block: 74 CTAs x 4 whole tiles
    g = torch.Generator(device="cpu").manual_seed(5)
    a = torch.randn((K, M), dtype=torch.float64, generator=g).cuda().t()      # M x K column-major
    b = torch.randn((N, K), dtype=torch.float64, generator=g).cuda().t()      # K x N
    full = torch.empty((N, M), dtype=torch.float64, device="cuda").t()
    eng.gemm_emulated(False, M, N, K, 1.0, a.data_ptr(), M, b.data_ptr(), K, 0.0, full.data_ptr(), M)
    for t in (3, 7, 150, 295):
        part = torch.empty((N, 128), dtype=torch.float64, device="cuda").t()
        eng.gemm_emulated(False, 128, N, K, 1.0, a[t * 128:].data_ptr(), M, b.data_ptr(), K, 0.0, part.data_ptr(), 128)
        torch.cuda.synchronize()
        assert torch.equal(part, full[t * 128:(t + 1) * 128]), t


# ---------------------------------------------------------------- graded lines (the scheme's weak case)

def _check_rows_normwise(got, aa, b, c0, alpha, beta, rows):
    """The emulation's bound: per output (i, j), 2^-54-class relative to max|row_i(op A)| *
    sum_k |b_kj| (plus the final rounding) -- the normwise FP64 GEMM class, NOT elementwise."""
    ar = aa[rows].numpy().astype(np.longdouble)
    bl = b.numpy().astype(np.longdouble)
    exact = alpha * (ar @ bl) + beta * c0[rows].numpy().astype(np.longdouble)
    rowmax = np.abs(ar).max(axis=1, keepdims=True)
    colmax = np.abs(bl).max(axis=0, keepdims=True)
    k = ar.shape[1]
    # slice rounding of op(A) (<= 2^-55 rowmax per element) and of B (<= 2^-55 colmax), summed over k
    bound = abs(alpha) * (2.0 ** -54) * (rowmax @ np.abs(bl).sum(axis=0, keepdims=True)
                                         + np.abs(ar).sum(axis=1, keepdims=True) @ colmax)
    err = np.abs(got[rows].numpy().astype(np.longdouble) - exact)
    tol = bound + 4e-16 * abs(beta) * np.abs(c0[rows].numpy()) + 2.0 ** -53 * np.abs(exact) + 1e-300
    assert (err <= tol).all(), float(np.max(err / tol))
    # and how far from elementwise FP64 accuracy the small entries are (informational)
    elem = abs(alpha) * (np.abs(ar) @ np.abs(bl)) + 1e-300
    return float(np.max(err / elem))


@pytest.mark.parametrize("trans", [True, False])
def test_emulated_gemm_graded_within_lines(eng, trans):
    """Every line of op(A) spans 1e-8 .. 1 (columns of A graded for the row-scaled A G
    layout, rows graded for the column-scaled A'Y one) plus a few spikes: the normwise
    bound holds for every element."""
    m, n, k = 600, 64, 3000
    g = torch.Generator(device="cpu").manual_seed(31 + int(trans))
    opa = torch.randn((m, k), dtype=torch.float64, generator=g) * torch.logspace(-8, 0, k, dtype=torch.float64)
    opa[:, ::997] *= 1e3    # spikes
    b = torch.randn((k, n), dtype=torch.float64, generator=g)
    c0 = torch.zeros((m, n), dtype=torch.float64)
    a = opa.t().contiguous() if trans else opa       # trans: A is k x m with op(A) = A'
    got = _run_emulated(eng, trans, a, b, c0, 1.0, 0.0)
    rel = _check_rows_normwise(got, opa, b, c0, 1.0, 0.0, np.arange(0, m, 5))
    assert rel > 0.0


def _graded(m, n, sig, seed, rows: bool):
    a = _lowrank(m, n, sig, seed)
    d = np.logspace(-8, 0, m if rows else n)
    np.random.default_rng(seed).shuffle(d)
    return np.asfortranarray(a * d[:, None] if rows else a * d[None, :])


@pytest.mark.parametrize("rows", [False, True])
@pytest.mark.parametrize("kind,zeta,power", [(3, 8, 1), (0, 0, 2), (2, 0, 1)])
def test_qb_emulation_on_graded_matrix_matches_oracle(eng, port, monkeypatch, rows, kind, zeta, power):
    """A with its columns (rows) scaled by 1e-8 .. 1 -- every row (column) of A then spans
    eight decades, the emulation's weak case -- through the QB loop with every A pass on
    the INT8 tensor cores, against the oracle on the same Omega: same rank / blocks / ids,
    E within 1e-10 ||A||^2, top sigma within 1e-10 sigma_max, Q B within 1e-10 ||A||_F."""
    monkeypatch.setenv("FQB_OZAKI", "1")
    a = _graded(1600, 1300, 0.9 ** np.arange(400), 90 + kind + 3 * int(rows), rows)
    p = 0.5 if kind == 2 else 0.0
    spec = SketchSpec(kind, p, 17, zeta=zeta)
    cfg = FarpcaConfig(eps=1e-3, power=power, block=32, sketch=spec, relative=True)
    res = eng.run_fixed_precision(a, cfg, output="host", svd=True)

    def src(n, b, bid):
        s = eng.gen_sketch(spec, n, b, bid)
        if s.is_dense:
            return SketchArrays(True, s.rows, s.cols, dense=s.dense, p=s.p)
        return SketchArrays(False, s.rows, s.cols, col_ptr=s.col_ptr, row_idx=s.row_idx, values=s.values,
                            centered=s.centered, p=s.p, std_scale=s.std_scale)
    ref = port.run(a, eps=1e-3, power=power, block=32, kind=kind, p=p, seed=17, zeta=zeta, relative=True,
                   source=src, want_vectors=True)
    assert ref.status == 0 and res.converged
    assert (res.rank, res.blocks, res.block_ids) == (ref.rank, ref.blocks, ref.block_ids)
    na = ref.norm_a_sq
    assert abs(res.residual_sq - ref.residual_sq) <= 1e-10 * na
    assert np.max(np.abs(res.block_residuals - ref.block_residuals)) <= 1e-10 * na
    top = ref.sigma >= 1e-3 * ref.sigma[-1]
    assert np.max(np.abs(res.sigma[top] - ref.sigma[top])) <= 1e-10 * ref.sigma[-1]
    qb = res.q @ res.bt.T
    usv = (ref.u * ref.sigma) @ ref.v.T
    assert np.linalg.norm(qb - usv) <= 1e-10 * np.sqrt(na)
