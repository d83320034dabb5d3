"""RawF64 files straight to the device (fqb_load_raw_rows): full matrices and row shards
land bit-identical to the file, and a QB run on the loaded shard equals the run on the
host copy.  CPU-side parsing and error parity are in test_matrix_io.py."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2506_03859_b200 as fqb  # noqa: E402
from paper_2506_03859_b200 import FarpcaConfig, SketchKind, SketchSpec  # noqa: E402
from paper_2506_03859_b200 import matrix_io as mio  # noqa: E402
from paper_2506_03859_b200.dist import partition_rows  # noqa: E402


@pytest.mark.parametrize("m,n", [(1, 1), (3001, 257), (20000, 600)])
def test_device_rows_equal_file(tmp_path, m, n):
    a = np.asfortranarray(np.random.default_rng(n).standard_normal((m, n)))
    p = tmp_path / "a.raw"
    fqb.save_raw(p, a)
    eng = fqb.default_engine(0)
    d = mio.load_raw_rows(p, engine=eng)
    assert d.is_cuda and np.array_equal(d.cpu().numpy(), a)
    for k in range(4):
        r0, r1 = partition_rows(m, 4, k)
        s = mio.load_raw_rows(p, r0, r1 - r0, engine=eng)
        assert np.array_equal(s.cpu().numpy(), a[r0:r1])


def test_qb_on_loaded_matrix(tmp_path):
    rng = np.random.default_rng(1)
    u, _ = np.linalg.qr(rng.standard_normal((2500, 120)))
    v, _ = np.linalg.qr(rng.standard_normal((700, 120)))
    a = np.asfortranarray((u * 0.9 ** np.arange(120)) @ v.T)
    p = tmp_path / "a.raw"
    fqb.save_raw(p, a)
    cfg = FarpcaConfig(eps=1e-3, power=1, block=20, sketch=SketchSpec(SketchKind.SparseSign, 0.0, 4, zeta=8),
                       relative=True)
    r_file = fqb.run_fixed_precision(mio.load_raw_rows(p, engine=fqb.default_engine(0)), cfg, output="host")
    r_host = fqb.run_fixed_precision(a, cfg, output="host")
    assert (r_file.rank, r_file.blocks) == (r_host.rank, r_host.blocks)
    assert r_file.residual_sq == r_host.residual_sq
    assert np.array_equal(r_file.bt, r_host.bt)
