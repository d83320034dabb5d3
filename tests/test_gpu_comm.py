"""Row-sharded (NCCL) engine path on the one GPU this run has: a 1-rank
communicator exercises every all-reduce point of csrc/engine.cu, including the
A'Y passes split in two row halves whose first all-reduce overlaps the second half's
product.  The halves change the products' internal summation order (split-K / stream-K
partitions follow the shape), so the factorization must equal the single-GPU run to
rounding: same rank / blocks / ids, E within 1e-12 ||A||^2, Q B within 1e-10 ||A||_F (the
parity bar; power iterations amplify the reordered roundings to ~1e-12 relative)."""
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402

import paper_2506_03859_b200 as fqb  # noqa: E402
from paper_2506_03859_b200 import FarpcaConfig, SketchSpec  # noqa: E402


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("m,n,b", [(1600, 1200, 32), (6000, 3000, 100)])   # DMMA / INT8 (paired) A passes
def test_one_rank_nccl_comm_is_transparent(m, n, b):
    rng = np.random.default_rng(0)
    u, _ = np.linalg.qr(rng.standard_normal((m, 300)))
    v, _ = np.linalg.qr(rng.standard_normal((n, 300)))
    a = np.asfortranarray((u * 10.0 ** (-np.arange(300) / 60)) @ v.T)
    cfg = FarpcaConfig(eps=1e-4, power=2, block=b, sketch=SketchSpec(4, 0.0, 3, zeta=8), relative=True)
    plain = fqb.Engine(0)
    r0 = plain.run_fixed_precision(a, cfg, output="host")
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda:0"))
    try:
        eng = fqb.Engine(0)
        eng.attach_comm()
        c0 = eng.collective_count
        r1 = eng.run_fixed_precision(a, cfg, output="host")
        assert eng.collective_count > c0
        eng.detach_comm()
    finally:
        dist.destroy_process_group()
    assert (r1.rank, r1.blocks, r1.block_ids) == (r0.rank, r0.blocks, r0.block_ids)
    assert abs(r1.residual_sq - r0.residual_sq) <= 1e-12 * r0.norm_a_sq
    assert np.linalg.norm(r1.q @ r1.bt.T - r0.q @ r0.bt.T) <= 1e-10 * np.sqrt(r0.norm_a_sq)
