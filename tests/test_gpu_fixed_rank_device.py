"""run_fixed_rank with the ApproxSvd left on the device and rank not a multiple of the
block: the kept triplets (the last svd_r columns of the assembly) must equal the host
copy.  Regression: they were moved to the front with an overlapping in-place memcpy,
which corrupted them (found by tests/test_gpu_experiment.py's rank sweep)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2506_03859_b200 as fqb  # noqa: E402


@pytest.mark.parametrize("rank,block", [(25, 10), (7, 4), (61, 20)])
def test_device_and_host_svd_agree(rank, block):
    eng = fqb.default_engine(0)
    rng = np.random.default_rng(rank)
    m, n = 700, 300
    a = np.asfortranarray(rng.standard_normal((m, n)) * 0.9 ** np.arange(n))
    cfg = fqb.FarpcaConfig(eps=0.0, power=1, block=block, sketch=fqb.SketchSpec(0, 0.0, 3), relative=True)
    rd = eng.run_fixed_rank(a, rank, cfg, output="device", svd=True)
    rh = eng.run_fixed_rank(a, rank, cfg, output="host", svd=True)
    assert rd.svd_rank() == rh.svd_rank() == rank
    assert np.array_equal(rd.sigma, rh.sigma)
    assert np.array_equal(rd.u.cpu().numpy(), rh.u)
    assert np.array_equal(rd.v.cpu().numpy(), rh.v)
