"""The block Gram-Schmidt and B-side products on the INT8 tensor cores (engine.cu: Q'X and
Y -= Q C over Q's slices, T = B G and W -= B' T over B''s slices), against the oracle fed
the same Omega, on tall and wide matrices past the switch-on sizes (m, n >= 4096, l >= 200,
the A passes on the emulation), with ranks that end mid 128-column slice tile.  Each run is
repeated with the products on DMMA (FQB_OZ_Q=0 / FQB_OZ_B=0, read per run) and both must
meet the same bars: rank / blocks / ids exact, E and the per-block trace 1e-10 ||A||^2,
sigma 1e-10 sigma_max, Q orthonormal to 1e-12."""
import os

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


def _lowrank(m, n, sig, seed):
    rng = np.random.default_rng(seed)
    r = len(sig)
    u, _ = np.linalg.qr(rng.standard_normal((m, r)))
    v, _ = np.linalg.qr(rng.standard_normal((n, r)))
    return np.asfortranarray((u * sig) @ v.T)


def _arr(s):
    if s.is_dense:
        return SketchArrays(True, s.rows, s.cols, dense=s.dense, p=s.p)
    return SketchArrays(False, s.rows, s.cols, col_ptr=s.col_ptr, row_idx=s.row_idx, values=s.values,
                        centered=s.centered, p=s.p, std_scale=s.std_scale)


def _with_env(env, fn):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return fn()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("m,n,b,power,kind", [(4100, 8200, 64, 1, 3), (8200, 4100, 60, 2, 4), (4400, 4400, 50, 2, 0)])
def test_int8_bgs_and_b_products_match_oracle(eng, port, m, n, b, power, kind):
    sig = 0.98 ** np.arange(420)
    a = _lowrank(m, n, sig, seed=m + n + b)
    spec = SketchSpec(kind, 0.0, 31, zeta=8 if kind in (3, 4) else 0)
    cfg = FarpcaConfig(eps=2e-3, power=power, block=b, sketch=spec, relative=True)
    ad = torch.from_numpy(a).cuda()

    def src(nn, bb, bid):
        return _arr(eng.gen_sketch(spec, nn, bb, bid))
    ref = port.run(a, eps=2e-3, power=power, block=b, kind=kind, p=0.0, seed=31, zeta=spec.zeta, relative=True,
                   source=src)
    assert ref.status == 0
    assert ref.rank >= 4 * b   # the INT8 products switch on from l = 200
    na = ref.norm_a_sq
    results = {}
    for tag, env in (("int8", {"FQB_OZAKI": "1", "FQB_OZ_Q": "1", "FQB_OZ_B": "1"}),
                     ("dmma", {"FQB_OZAKI": "1", "FQB_OZ_Q": "0", "FQB_OZ_B": "0"})):
        res = _with_env(env, lambda: eng.run_fixed_precision(ad, cfg, output="host"))
        assert res.converged, tag
        assert (res.rank, res.blocks, res.block_ids) == (ref.rank, ref.blocks, ref.block_ids), tag
        assert abs(res.residual_sq - ref.residual_sq) <= 1e-10 * na, tag
        assert np.max(np.abs(res.block_residuals - np.asarray(ref.block_residuals))) <= 1e-10 * na, tag
        s = np.sort(np.linalg.svd(res.bt, compute_uv=False))
        rs = np.asarray(ref.sigma)
        top = rs >= 1e-3 * rs[-1]
        k = min(len(s), len(rs))
        assert np.max(np.abs(s[-k:][top[-k:]] - rs[-k:][top[-k:]])) <= 1e-10 * rs[-1], tag
        q = res.q
        assert np.abs(q.T @ q - np.eye(res.rank)).max() < 1e-12, tag
        results[tag] = res
    qb = [r.q @ r.bt.T for r in results.values()]
    assert np.linalg.norm(qb[0] - qb[1]) <= 1e-10 * np.sqrt(na)


@pytest.mark.parametrize("rows", [False, True])
def test_int8_products_on_graded_matrix_match_oracle(eng, port, rows):
    """The emulation's weak case at sizes where the Q- and B-side products run on the INT8
    tensor cores too: every row (column) of A spans eight decades (its columns (rows) scaled
    by 1e-8 .. 1).  Same bars as above, plus Q B within 1e-10 ||A||_F of the oracle's."""
    m, n, b = 4200, 4300, 64
    a = _lowrank(m, n, 0.98 ** np.arange(420), seed=700 + int(rows))
    d = np.logspace(-8, 0, m if rows else n)
    np.random.default_rng(701).shuffle(d)
    a = np.asfortranarray(a * d[:, None] if rows else a * d[None, :])
    spec = SketchSpec(3, 0.0, 41, zeta=8)
    cfg = FarpcaConfig(eps=2e-3, power=1, block=b, sketch=spec, relative=True)

    def src(nn, bb, bid):
        return _arr(eng.gen_sketch(spec, nn, bb, bid))
    ref = port.run(a, eps=2e-3, power=1, block=b, kind=3, p=0.0, seed=41, zeta=8, relative=True, source=src,
                   want_vectors=True)
    assert ref.status == 0 and ref.rank >= 4 * b
    res = _with_env({"FQB_OZAKI": "1", "FQB_OZ_Q": "1", "FQB_OZ_B": "1"},
                    lambda: eng.run_fixed_precision(torch.from_numpy(a).cuda(), cfg, output="host", svd=True))
    assert res.converged
    assert (res.rank, res.blocks, res.block_ids) == (ref.rank, ref.blocks, ref.block_ids)
    na = ref.norm_a_sq
    assert abs(res.residual_sq - ref.residual_sq) <= 1e-10 * na
    assert np.max(np.abs(res.block_residuals - np.asarray(ref.block_residuals))) <= 1e-10 * na
    top = ref.sigma >= 1e-3 * ref.sigma[-1]
    assert np.max(np.abs(res.sigma[top] - ref.sigma[top])) <= 1e-10 * ref.sigma[-1]
    usv = (ref.u * ref.sigma) @ ref.v.T
    assert np.linalg.norm(res.q @ res.bt.T - usv) <= 1e-10 * np.sqrt(na)
