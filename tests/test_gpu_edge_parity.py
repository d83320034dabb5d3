"""Edge shapes and limits against the reference itself (oracle/_ref, run here on the CPU):
zero matrix, eps so large that no block is needed, single row / column, wide and tall A,
b equal to min(m, n), max_iters cap (ToleranceNotReached), a rank-deficient A whose later
blocks degenerate (BlockDegenerate with the same redraw ids).  Same status, rank, blocks and
block ids; E within 1e-10 ||A||^2 (the parity bar)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2506_03859_b200 as fqb  # noqa: E402
from paper_2506_03859_b200 import FarpcaConfig, SketchSpec  # noqa: E402

STATUS = {0: "ok", 3: "degenerate", 4: "tolerance"}


def _ours(a, cfg, rank=None):
    try:
        r = (fqb.run_fixed_precision(a, cfg, output="host", svd=False) if rank is None
             else fqb.run_fixed_rank(a, rank, cfg, output="host", svd=True))
        return "ok", r
    except fqb.ToleranceNotReached as e:
        return "tolerance", e.partial
    except fqb.BlockDegenerate as e:
        return "degenerate", e


def _compare(reference, a, *, eps=0.0, power=0, block=0, kind=0, p=0.0, seed=3, zeta=0, max_iters=0, rank=None,
             relative=True):
    cfg = FarpcaConfig(eps=eps, power=power, block=block, sketch=SketchSpec(kind, p, seed, zeta=zeta),
                       max_iters=max_iters, relative=relative)
    ref = reference.run(a, eps=eps, power=power, block=block, kind=kind, p=p, seed=seed, zeta=zeta,
                        max_iters=max_iters, rank=rank, relative=relative)
    st, got = _ours(a, cfg, rank)
    assert st == STATUS[ref.status], (st, ref.status, ref.message)
    na = max(float(np.sum(a * a)), 1e-300)
    if st == "degenerate":
        assert got.blocks_accepted == ref.blocks
        assert abs(got.residual_sq - ref.residual_sq) <= 1e-10 * na
        return ref, got
    if rank is None:
        assert (got.rank, got.blocks) == (ref.rank, ref.blocks)
    else:   # fixed rank: the reference reports the ApproxSvd rank, the QB keeps blocks * b columns
        assert ref.rank == rank and got.blocks == ref.blocks and got.rank == ref.blocks * got.resolved_block
    assert list(got.block_ids) == list(ref.block_ids)
    # fixed rank: the reference's residual is the ApproxSvd's (dropped sigma^2 added back)
    res = got.residual_sq if rank is None else got.svd_residual_sq
    assert abs(res - ref.residual_sq) <= 1e-10 * na
    return ref, got


def _lowrank(m, n, r, seed, decay=0.9):
    rng = np.random.default_rng(seed)
    u, _ = np.linalg.qr(rng.standard_normal((m, r)))
    v, _ = np.linalg.qr(rng.standard_normal((n, r)))
    return np.asfortranarray((u * decay ** np.arange(r)) @ v.T)


def test_zero_matrix(reference):
    _compare(reference, np.zeros((50, 40), order="F"), eps=1e-3, block=5)


def test_eps_needs_no_block(reference):
    ref, got = _compare(reference, _lowrank(60, 50, 20, 1), eps=2.0, block=5)
    assert got.rank == 0 and got.blocks == 0


@pytest.mark.parametrize("shape", [(1, 40), (40, 1), (3, 200), (300, 7)])
def test_thin_shapes(reference, shape):
    """eps above the indicator's rounding floor (the reference warns below 2.1e-7 |A|):
    at the floor, E = |A|^2 - sum |B_j|^2 is cancellation noise and whether it beats
    eps^2 after the last full-rank block is a coin flip on either side."""
    m, n = shape
    a = np.asfortranarray(np.random.default_rng(m * 7 + n).standard_normal(shape))
    _compare(reference, a, eps=1e-6, block=1, power=1)


def test_block_equals_min_dimension(reference):
    _compare(reference, _lowrank(80, 24, 24, 4), eps=1e-9, block=24, power=1)


def test_max_iters_cap(reference):
    ref, got = _compare(reference, _lowrank(120, 100, 60, 5, decay=0.98), eps=1e-9, block=8, max_iters=3, power=1)
    assert got.blocks == 3


@pytest.mark.parametrize("kind,zeta,p", [(0, 0, 0.0), (3, 4, 0.0), (1, 0, 0.3)])
def test_rank_deficient_degenerates_like_the_reference(reference, kind, zeta, p):
    """rank 12 with b = 5: the third block is degenerate after the pivot rule; the redraws
    (ids 2, 1002, 2002, 3002) fail the same way -> BlockDegenerate after 2 blocks."""
    _compare(reference, _lowrank(70, 60, 12, 6, decay=1.0), eps=1e-14, block=5, kind=kind, zeta=zeta, p=p, power=1)


def test_fixed_rank_wide(reference):
    _compare(reference, _lowrank(40, 300, 30, 7), rank=17, block=6, power=2)


def test_absolute_tolerance(reference):
    a = _lowrank(90, 70, 40, 8)
    _compare(reference, a, eps=1e-3 * np.linalg.norm(a), block=7, power=1, relative=False)
