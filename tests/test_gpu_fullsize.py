"""BASELINE configs at full size on the GPU.

C2 is checked against the reference itself (oracle/_ref, ~16 s on one core).  C3 and
C4 are checked against golden reference runs in test_gpu_bigcases.py; here, on other
seeds, through size-independent properties: E equals the true residual
||A - QB||_F^2 (computed on the GPU), Q is orthonormal, the per-block trace is
monotone, the rank reaches the spectrum's tail, and the run is deterministic.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2506_03859_b200 as fqb  # noqa: E402
from paper_2506_03859_b200 import FarpcaConfig, SketchKind, SketchSpec  # noqa: E402

DEV = torch.device("cuda:0")


def _true_residual(a, q, bt, chunk=8192):
    tot = 0.0
    for c0 in range(0, a.shape[1], chunk):
        c1 = min(a.shape[1], c0 + chunk)
        d = a[:, c0:c1] - q @ bt[c0:c1].t()
        tot += float((d * d).sum())
    return tot


def _c2_matrix():
    """BASELINE configs[1]: U diag(10^(-i/50)) V', 8000^2, U, V = random_orthonormal(8000, 900,
    seed 42) on the reference's factor streams (fqb_gen_lowrank)."""
    sig = 10.0 ** (-np.arange(1, 901, dtype=np.float64) / 50.0)
    return fqb.default_engine(0).gen_lowrank(8000, 8000, sig, seed=42)


def test_c2_matches_reference(reference):
    a = _c2_matrix()
    cfg = FarpcaConfig(eps=1e-3, power=2, block=50, sketch=SketchSpec(SketchKind.StdBernoulli, 0.5, 7),
                       relative=True)
    res = fqb.run_fixed_precision(a, cfg, output="host", svd=True)
    a_np = np.asfortranarray(a.cpu().numpy())
    eng = fqb.default_engine(0)
    spec = cfg.sketch

    from oracle.oracle import SketchArrays

    def src(n, b, bid):
        s = eng.gen_sketch(spec, n, b, bid)
        return SketchArrays(False, n, b, col_ptr=s.col_ptr, row_idx=s.row_idx, values=s.values,
                            centered=s.centered, p=s.p, std_scale=s.std_scale)
    ref = reference.run(a_np, eps=cfg.eps, power=cfg.power, block=cfg.block, kind=int(spec.kind), p=spec.p,
                        seed=spec.seed, relative=True, source=src, traced=True)
    assert ref.status == 0 and res.converged
    assert (res.rank, res.blocks, res.block_ids) == (ref.rank, ref.blocks, ref.block_ids) == (200, 4, [0, 1, 2, 3])
    na = ref.norm_a_sq
    assert abs(res.residual_sq - ref.residual_sq) <= 1e-10 * na
    assert np.max(np.abs(res.block_residuals - ref.block_residuals)) <= 1e-10 * na
    top = ref.sigma >= 1e-3 * ref.sigma[-1]
    assert np.max(np.abs(res.sigma[top] - ref.sigma[top])) <= 1e-10 * ref.sigma[-1]


def test_c4_tall_sparse_gaussian_full_size():
    """100000 x 20000, rank 2000, sigma_i = 10^(-3i/2000), sparse Gaussian zeta=8, b=100, P=2, eps=1e-3."""
    sig = 10.0 ** (-3.0 * np.arange(1, 2001, dtype=np.float64) / 2000)
    a = fqb.default_engine(0).gen_lowrank_det(100000, 20000, sig, 4)
    cfg = FarpcaConfig(eps=1e-3, power=2, block=100, sketch=SketchSpec(SketchKind.SparseGaussian, 0.0, 7, zeta=8),
                       relative=True)
    res = fqb.run_fixed_precision(a, cfg, output="device", svd=False)
    assert res.converged
    # optimal rank for 1e-3: tail energy of 10^(-3i/2000) -> about 1900-2000
    assert 1800 <= res.rank <= 2000
    q, bt = res.q, res.bt
    assert float((q.t() @ q - torch.eye(res.rank, dtype=torch.float64, device=DEV)).abs().max()) < 1e-12
    e_true = _true_residual(a, q, bt)
    assert abs(res.residual_sq - e_true) <= 1e-10 * res.norm_a_sq
    assert np.all(np.diff(res.block_residuals) <= 1e-12 * res.norm_a_sq)
    assert res.residual_sq < (1e-3) ** 2 * res.norm_a_sq


def test_c3_noise_floor_full_size():
    """20000^2 rank-1000 signal + 1e-4 N(0,1)/sqrt(n) noise, sparse sign zeta=8, b=64, P=1, eps=1e-2.

    SURVEY.md section 0.4 predicts the noise floor (||N||^2 = 1e-8 m = 2e-4, i.e.
    1.7e-4 of ||A||^2) keeps E above eps^2 = 1e-4 until max_iters = 157 blocks.
    The QB also captures noise directions (about l/n of ||N||^2), so depending on
    the draw the run either converges late or stops at the cap with
    ToleranceNotReached; both outcomes must carry a correct indicator."""
    sig = (1.0 + np.arange(0, 1000, dtype=np.float64)) ** -1.5
    a = fqb.default_engine(0).gen_lowrank_det(20000, 20000, sig, 3, 1e-4 / np.sqrt(20000))
    cfg = FarpcaConfig(eps=1e-2, power=1, block=64, sketch=SketchSpec(SketchKind.SparseSign, 0.0, 7, zeta=8),
                       relative=True)
    try:
        res = fqb.run_fixed_precision(a, cfg, output="device", svd=False)
        assert res.converged and res.residual_sq < 1e-4 * res.norm_a_sq
        assert res.blocks > 20   # far past the rank-1000 signal: the noise dominates
    except fqb.ToleranceNotReached as e:
        res = e.partial
        assert res.blocks == 157 and not res.converged and res.residual_sq >= 1e-4 * res.norm_a_sq
    assert res.rank == 64 * res.blocks and res.block_ids == list(range(res.blocks))
    e_true = _true_residual(a, res.q, res.bt)
    assert abs(res.residual_sq - e_true) <= 1e-10 * res.norm_a_sq
    assert np.all(np.diff(res.block_residuals) <= 1e-12 * res.norm_a_sq)
    q = res.q
    assert float((q.t() @ q - torch.eye(res.rank, dtype=torch.float64, device=DEV)).abs().max()) < 1e-11
