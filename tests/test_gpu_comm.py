"""Row-sharded (NCCL) engine path on the one GPU this run has: a 1-rank
communicator exercises every all-reduce point of csrc/engine.cu and must leave
the factorization bit-identical to the single-GPU run."""
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


def test_one_rank_nccl_comm_is_transparent():
    rng = np.random.default_rng(0)
    u, _ = np.linalg.qr(rng.standard_normal((1600, 300)))
    v, _ = np.linalg.qr(rng.standard_normal((1200, 300)))
    a = np.asfortranarray((u * 10.0 ** (-np.arange(300) / 60)) @ v.T)
    cfg = FarpcaConfig(eps=1e-4, power=2, block=32, sketch=SketchSpec(4, 0.0, 3, zeta=8), relative=True)
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
    assert r1.rank == r0.rank and r1.blocks == r0.blocks
    assert r1.residual_sq == r0.residual_sq
    assert np.array_equal(r1.q, r0.q) and np.array_equal(r1.bt, r0.bt)
