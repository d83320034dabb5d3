"""Host Q, B' streamed out block by block (QbRun::push_host).

With host outputs, a run whose shape the handle has seen before copies each committed
block's Q / B' columns to pinned host memory on the copy stream while the next block
runs.  The host arrays must equal the device outputs bit for bit: on the first run of
a shape (copies after the loop), on repeats (streamed), when a later run outgrows the
learned capacity (host blocks regrown, committed columns copied again), across device
regrowths of Q / B' (whose old arrays the queued copies still read), and with the
INT8 A passes forced on.  FQB_OUT_TAIL=1 restores the copies after the loop."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2506_03859_b200 as fqb  # noqa: E402


def _matrix(m, n, decay, seed):
    rng = np.random.default_rng(seed)
    return np.asfortranarray(rng.standard_normal((m, n)) * decay ** np.arange(n))


def _same(rd, rh):
    assert rh.rank == rd.rank and rh.blocks == rd.blocks
    assert rh.residual_sq == rd.residual_sq
    assert np.array_equal(rd.q.cpu().numpy(), rh.q)
    assert np.array_equal(rd.bt.cpu().numpy(), rh.bt)


@pytest.mark.parametrize("ozaki", ["0", "1"])
def test_streamed_host_outputs_equal_device_outputs(monkeypatch, ozaki):
    monkeypatch.setenv("FQB_OZAKI", ozaki)
    eng = fqb.Engine(0)
    m, n, b = 2400, 1200, 24
    a = _matrix(m, n, 0.995, 5)
    sk = fqb.SketchSpec(fqb.SketchKind.SparseSign, 0.0, 7, zeta=8)
    loose = fqb.FarpcaConfig(eps=0.5, power=1, block=b, sketch=sk, relative=True)
    tight = fqb.FarpcaConfig(eps=0.2, power=1, block=b, sketch=sk, relative=True)
    rd_loose = eng.run_fixed_precision(a, loose, output="device")
    rd_tight = eng.run_fixed_precision(a, tight, output="device")
    # the tight run outgrows the device's first capacities (4 b, 8 b, ...) and the
    # host capacity the loose runs teach the handle
    assert rd_tight.rank > 8 * b > rd_loose.rank
    for cfg, rd in [(loose, rd_loose), (loose, rd_loose), (loose, rd_loose), (tight, rd_tight),
                    (tight, rd_tight), (loose, rd_loose)]:
        rh = eng.run_fixed_precision(a, cfg, output="host")
        _same(rd, rh)


def test_streamed_host_outputs_with_svd():
    eng = fqb.Engine(0)
    a = _matrix(1500, 700, 0.99, 9)
    cfg = fqb.FarpcaConfig(eps=5e-2, power=2, block=20, sketch=fqb.SketchSpec(2, 0.5, 3), relative=True)
    rd = eng.run_fixed_precision(a, cfg, output="device", svd=True)
    for _ in range(3):
        rh = eng.run_fixed_precision(a, cfg, output="host", svd=True)
        _same(rd, rh)
        assert np.array_equal(rd.sigma, rh.sigma)
        # host U is formed in 256-column blocks (each downloaded as it is done), so its
        # GEMM split can differ from the device path's: equal to rounding, not bitwise
        np.testing.assert_allclose(rh.u, rd.u.cpu().numpy(), rtol=0, atol=1e-13)
        np.testing.assert_allclose(rh.v, rd.v.cpu().numpy(), rtol=0, atol=1e-13)
