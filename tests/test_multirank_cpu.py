"""World-size-2 CPU (gloo) tests of the row-sharded multi-GPU host logic.

The device collectives are NCCL inside libfarqb and need GPUs; here the same
decomposition is exercised with gloo: row partitioning, the unique-id
exchange, and a numpy model of the engine's sharded loop (tests/sharded_model.py)
whose all-reduce points are those of csrc/engine.cu, checked against the CPU
oracle on the unsharded matrix with identical Omega blocks.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2506_03859_b200.dist import exchange_unique_id, partition_rows  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _matrix(m=400, n=300, seed=3):
    rng = np.random.default_rng(seed)
    u, _ = np.linalg.qr(rng.standard_normal((m, 120)))
    v, _ = np.linalg.qr(rng.standard_normal((n, 120)))
    return np.asfortranarray((u * 10.0 ** (-np.arange(120) / 30)) @ v.T)


def _omega(port_lib_path):
    from oracle.oracle import Oracle
    orc = Oracle("port")

    def om(n, b, bid):
        return orc.gen_sketch(3, 0.0, 9, n, b, bid, zeta=8).densify()
    return om


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        here = os.path.dirname(os.path.abspath(__file__))
        sys.path.insert(0, here)
        sys.path.insert(0, os.path.dirname(here))
        from sharded_model import qb_sharded
        a = _matrix()
        r0, r1 = partition_rows(a.shape[0], world, rank)
        uid = exchange_unique_id(lambda: bytes(range(128)), None)

        def allreduce(x):
            t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
            dist.all_reduce(t)
            return t.numpy()

        q, bt, l, e, norm, hist = qb_sharded(a[r0:r1], 1e-3, 1, 16, 20, _omega(None), allreduce)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), q=q, bt=bt, l=l, e=e, norm=norm, hist=np.array(hist),
                 r0=r0, r1=r1, uid=np.frombuffer(uid, dtype=np.uint8))
    finally:
        dist.destroy_process_group()


def test_partition_rows_covers_and_aligns():
    for m in (1, 15, 16, 17, 8000, 100000, 400001):
        for world in (1, 2, 3, 4, 8):
            if m < world:
                continue
            blocks = [partition_rows(m, world, r) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == m
            for (a0, a1), (b0, b1) in zip(blocks, blocks[1:]):
                assert a1 == b0 and a0 <= a1
            for r0, _ in blocks:
                assert r0 % 16 == 0


def test_two_rank_gloo_sharded_model_matches_oracle(tmp_path, port):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    res = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    # the unique id reached every rank intact
    for r in res:
        assert bytes(r["uid"]) == bytes(range(128))
    # replicated quantities agree bitwise across ranks
    assert np.array_equal(res[0]["bt"], res[1]["bt"]) and float(res[0]["e"]) == float(res[1]["e"])
    a = _matrix()
    q = np.vstack([r["q"] for r in res])
    bt = res[0]["bt"]
    l = int(res[0]["l"])
    # Q is orthonormal across the shards and E is the true residual
    assert np.abs(q.T @ q - np.eye(l)).max() < 1e-12
    assert abs(float(res[0]["e"]) - np.linalg.norm(a - q @ bt.T) ** 2) <= 1e-10 * float(res[0]["norm"])
    # same answer as the oracle fed the same Omega on the whole matrix
    om = _omega(None)

    from oracle.oracle import SketchArrays
    ref = port.run(a, eps=1e-3, power=1, block=16, kind=3, seed=9, zeta=8, relative=True, max_iters=20,
                   source=lambda n, b, bid: SketchArrays(True, n, b, dense=om(n, b, bid)))
    assert ref.rank == l
    assert abs(ref.residual_sq - float(res[0]["e"])) <= 1e-10 * ref.norm_a_sq
    np.testing.assert_allclose(res[0]["hist"], ref.block_residuals, atol=1e-10 * ref.norm_a_sq, rtol=0)
