"""FP32 input mode (BASELINE config 5): A stored in FP32, every product in FP64.

Contract: FP32 mode must agree with the FP64 reference
within 1e-4.  This mode is stricter: the loop runs in FP64 on the exactly
widened values, so it must match the oracle run on double(A_fp32) within the
FP64 parity bounds (rank / blocks / ids exact, E within 1e-10 ||A||^2), on both
A-pass paths (INT8-emulated and DMMA with one widened copy), for A on the host
or the device.
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


def _lowrank32(m, n, sig, seed, noise=0.0):
    rng = np.random.default_rng(seed)
    r = len(sig)
    u, _ = np.linalg.qr(rng.standard_normal((m, r)))
    v, _ = np.linalg.qr(rng.standard_normal((n, r)))
    a = (u * sig) @ v.T
    if noise:
        a += noise * rng.standard_normal((m, n)) / np.sqrt(n)
    return np.asfortranarray(a.astype(np.float32))


def _src(eng, spec):
    def src(n, b, bid):
        s = eng.gen_sketch(spec, n, b, bid)
        if s.is_dense:
            return SketchArrays(True, s.rows, s.cols, dense=s.dense, p=s.p)
        return SketchArrays(False, s.rows, s.cols, col_ptr=s.col_ptr, row_idx=s.row_idx, values=s.values,
                            centered=s.centered, p=s.p, std_scale=s.std_scale)
    return src


@pytest.mark.parametrize("ozaki", ["1", "0"])
@pytest.mark.parametrize("kind,zeta", [(0, 0), (1, 0), (2, 0), (3, 4), (4, 4)])
def test_fp32_input_matches_oracle_on_widened_a(eng, port, monkeypatch, ozaki, kind, zeta):
    """C5's four kinds (zeta = 4), P = 1, on a scaled-down low-rank-plus-noise FP32 matrix."""
    monkeypatch.setenv("FQB_OZAKI", ozaki)
    a32 = _lowrank32(900, 600, 1.0 / np.arange(1, 121), seed=50 + kind, noise=1e-3)
    p = 0.0 if kind == 0 or zeta else 0.5
    spec = SketchSpec(kind, p, 9, zeta=zeta)
    cfg = FarpcaConfig(eps=5e-2, power=1, block=32, sketch=spec, relative=True)
    res = eng.run_fixed_precision(a32, cfg, output="host")
    ref = port.run(np.asfortranarray(a32.astype(np.float64)), eps=5e-2, power=1, block=32, kind=kind, p=p, seed=9,
                   zeta=zeta, relative=True, source=_src(eng, spec))
    assert ref.status == 0 and res.converged
    assert (res.rank, res.blocks, res.block_ids) == (ref.rank, ref.blocks, ref.block_ids)
    na = ref.norm_a_sq
    assert abs(res.norm_a_sq - na) <= 1e-12 * na   # tree vs sequential summation order
    assert abs(res.residual_sq - ref.residual_sq) <= 1e-10 * na
    assert np.max(np.abs(res.block_residuals - ref.block_residuals)) <= 1e-10 * na


def test_fp32_device_input_equals_host_input_and_fp64_of_widened(eng):
    a32 = _lowrank32(3000, 2500, 0.9 ** np.arange(200), seed=3)
    cfg = FarpcaConfig(eps=1e-3, power=2, block=40, sketch=SketchSpec(2, 0.5, 4), relative=True)
    rh = eng.run_fixed_precision(a32, cfg, output="host")
    dev = torch.from_numpy(a32.T.copy()).cuda().t()          # float32, column-major on the device
    rd = eng.run_fixed_precision(dev, cfg, output="host")
    r64 = eng.run_fixed_precision(np.asfortranarray(a32.astype(np.float64)), cfg, output="host")
    assert rh.rank == rd.rank == r64.rank and rh.blocks == rd.blocks == r64.blocks
    assert np.array_equal(rh.bt, rd.bt) and rh.residual_sq == rd.residual_sq
    # same arithmetic on the same values as the FP64 run of double(A)
    assert abs(rh.residual_sq - r64.residual_sq) <= 1e-12 * r64.norm_a_sq
    qb32 = rh.q @ rh.bt.T
    assert np.abs(qb32 - r64.q @ r64.bt.T).max() <= 1e-11 * np.abs(a32).max()


def test_fp32_fixed_rank_and_svd(eng):
    a32 = _lowrank32(1200, 800, 1.0 / np.arange(1, 301) ** 1.2, seed=8)
    cfg = FarpcaConfig(eps=1e-2, power=1, block=25, sketch=SketchSpec(3, 0.0, 2, zeta=4), relative=True)
    r = eng.run_fixed_rank(a32, 60, cfg, output="host", svd=True)
    assert r.sigma.shape == (60,)
    s_true = np.linalg.svd(a32.astype(np.float64), compute_uv=False)[:60][::-1]
    # randomized QB with P = 1: the top of the spectrum is accurate
    assert np.allclose(r.sigma[-10:], s_true[-10:], rtol=1e-3)


def test_c5_shape_slice_fp32(eng):
    """C5's row count (400000) and b = 128 on a 4096-column slice, FP32, sparse sign zeta = 4,
    checked through size-independent properties: E equals the true residual, Q orthonormal."""
    m, n = 400000, 4096
    g = torch.Generator(device="cuda").manual_seed(5)
    r = 500
    sig = 1.0 / torch.arange(1, r + 1, dtype=torch.float64, device="cuda")
    x = torch.linalg.qr(torch.randn(m, r, dtype=torch.float64, device="cuda", generator=g))[0]
    y = torch.linalg.qr(torch.randn(n, r, dtype=torch.float64, device="cuda", generator=g))[0]
    a = ((x * sig) @ y.t()).float()
    a += 1e-3 * torch.randn(m, n, device="cuda", generator=g) / np.sqrt(n)
    del x, y
    a = a.t().contiguous().t()
    cfg = FarpcaConfig(eps=5e-2, power=1, block=128, sketch=SketchSpec(3, 0.0, 7, zeta=4), relative=True)
    try:
        res = eng.run_fixed_precision(a, cfg, output="device")
    except fqb.ToleranceNotReached as e:   # noise share decides reachability
        res = e.partial
    q, bt = res.q, res.bt
    assert float((q.t() @ q - torch.eye(res.rank, dtype=torch.float64, device="cuda")).abs().max()) < 1e-11
    tot = 0.0
    for c0 in range(0, n, 1024):
        d = a[:, c0:c0 + 1024].double() - q @ bt[c0:c0 + 1024].t()
        tot += float((d * d).sum())
    assert abs(res.residual_sq - tot) <= 1e-10 * res.norm_a_sq


@pytest.fixture(params=[4, 3])
def eng4(request):
    """A separate engine with FP32-class A passes (fqb_set_fp32_slices(4): 7-bit digits,
    10 products; (3): 8-bit digits, 8 products)."""
    e = fqb.Engine(0)
    e.set_fp32_slices(request.param)
    yield e
    e.close()


@pytest.mark.parametrize("kind,zeta", [(0, 0), (2, 0), (3, 4), (4, 4)])
def test_fp32_four_slices_within_the_fp32_contract(eng, eng4, port, monkeypatch, kind, zeta):
    """4 or 3 slices per operand: FP32-class products.  Against the FP64 oracle on double(A):
    the same rank / blocks / ids and E within the FP32-mode bar (1e-4 relative); against
    the 8-slice run on the same A and Omega: Q B within 1e-6 of A's scale (the QB of one
    sketch is unique, so this isolates the precision of the products)."""
    monkeypatch.setenv("FQB_OZAKI", "1")
    a32 = _lowrank32(900, 600, 1.0 / np.arange(1, 121), seed=70 + kind, noise=1e-3)
    p = 0.0 if kind == 0 or zeta else 0.5
    spec = SketchSpec(kind, p, 9, zeta=zeta)
    cfg = FarpcaConfig(eps=5e-2, power=1, block=32, sketch=spec, relative=True)
    res = eng4.run_fixed_precision(a32, cfg, output="host")
    a64 = np.asfortranarray(a32.astype(np.float64))
    ref = port.run(a64, eps=5e-2, power=1, block=32, kind=kind, p=p, seed=9, zeta=zeta, relative=True,
                   source=_src(eng4, spec))
    assert ref.status == 0 and res.converged
    assert (res.rank, res.blocks, res.block_ids) == (ref.rank, ref.blocks, ref.block_ids)
    na = ref.norm_a_sq
    assert abs(res.residual_sq - ref.residual_sq) <= 1e-4 * ref.residual_sq
    assert np.abs(res.q.T @ res.q - np.eye(res.rank)).max() < 1e-10
    r8 = eng.run_fixed_precision(a32, cfg, output="host")
    diff = np.abs(res.q @ res.bt.T - r8.q @ r8.bt.T).max()
    assert diff <= 1e-6 * np.abs(a64).max(), diff
    assert diff > 0.0   # different arithmetic really ran


def test_fp32_four_slices_default_is_eight(eng, monkeypatch):
    """The default engine keeps FP64-class passes for FP32 input (bit-equal to double(A))."""
    monkeypatch.setenv("FQB_OZAKI", "1")
    a32 = _lowrank32(700, 500, 0.9 ** np.arange(100), seed=4)
    cfg = FarpcaConfig(eps=1e-2, power=1, block=20, sketch=SketchSpec(0, 0.0, 3), relative=True)
    r32 = eng.run_fixed_precision(a32, cfg, output="host")
    r64 = eng.run_fixed_precision(np.asfortranarray(a32.astype(np.float64)), cfg, output="host")
    assert np.array_equal(r32.bt, r64.bt)
