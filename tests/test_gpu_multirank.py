"""The row-sharded engine (csrc/engine.cu reduction points) with
world size 2, against the oracle on the unsharded matrix.

Two processes share the one GPU of the test box.  They reduce through the engine's host
backend (fqb_comm_attach_host -> torch.distributed gloo), so no kernel of one rank ever
waits on the other's (each exchange is a host round trip); the reduction points, the
row partition, the replicated B / Grams and the per-rank Q rows are exactly those of
the NCCL path.  Checked: both ranks take identical decisions (rank, blocks, ids, E to
the bit), and against the CPU oracle run on the whole matrix with the same Omega: rank /
blocks / ids exact, E and the per-block trace within 1e-10 ||A||^2, the stacked Q
orthonormal, Q B against the oracle's U diag(sigma) V' within 1e-10 ||A||_F, and the
SVD assembly's sigma.
"""
import os
import pickle
import socket
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
M, N = 1300, 900
SIG = 0.93 ** np.arange(260)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir, case):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if case.get("ozaki"):
        os.environ["FQB_OZAKI"] = "1"
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2506_03859_b200 as fqb
        from paper_2506_03859_b200 import FarpcaConfig, SketchSpec
        from paper_2506_03859_b200.dist import partition_rows
        eng = fqb.Engine(0)
        r0, r1 = partition_rows(M, world, rank)
        a = eng.gen_lowrank_det(M, N, SIG, 11, 0.0, r0, r1 - r0)     # this rank's rows only
        eng.attach_comm(backend="host")
        spec = SketchSpec(case["kind"], case["p"], 5, zeta=case["zeta"])
        cfg = FarpcaConfig(eps=1e-3, power=case["power"], block=case["block"], sketch=spec, relative=True)
        res = eng.run_fixed_precision(a, cfg, output="host", svd=True)
        out = {"rank": res.rank, "blocks": res.blocks, "ids": res.block_ids, "e": res.residual_sq,
               "na": res.norm_a_sq, "trace": np.asarray(res.block_residuals), "q": np.asarray(res.q),
               "bt": np.asarray(res.bt), "sigma": np.asarray(res.sigma), "u": np.asarray(res.u),
               "rows": (r0, r1), "collectives": eng.collective_count, "converged": res.converged}
        with open(os.path.join(out_dir, f"r{rank}.pkl"), "wb") as f:
            pickle.dump(out, f)
        eng.detach_comm()
    finally:
        dist.destroy_process_group()


CASES = [
    dict(kind=4, p=0.0, zeta=8, power=2, block=40),
    dict(kind=2, p=0.5, zeta=0, power=1, block=32),
    dict(kind=3, p=0.0, zeta=8, power=1, block=100, ozaki=True),   # INT8 A passes, two chunks per pass
]


@pytest.mark.parametrize("case", CASES, ids=["sgauss-P2", "stdbern-P1", "ssign-b100-ozaki"])
def test_two_ranks_match_oracle_on_whole_matrix(port, case):
    import paper_2506_03859_b200 as fqb
    from oracle.oracle import SketchArrays
    from paper_2506_03859_b200 import SketchSpec
    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(world, _free_port(), d, case), nprocs=world, join=True,
                           start_method="spawn")
        outs = [pickle.load(open(os.path.join(d, f"r{r}.pkl"), "rb")) for r in range(world)]
    o0, o1 = outs
    # identical decisions and replicated results on both ranks
    assert (o0["rank"], o0["blocks"], o0["ids"], o0["e"]) == (o1["rank"], o1["blocks"], o1["ids"], o1["e"])
    assert np.array_equal(o0["bt"], o1["bt"]) and np.array_equal(o0["sigma"], o1["sigma"])
    assert o0["collectives"] > 0
    # the whole matrix and the oracle on it, same Omega
    eng = fqb.default_engine(0)
    a = eng.gen_lowrank_det(M, N, SIG, 11).cpu().numpy()
    spec = SketchSpec(case["kind"], case["p"], 5, zeta=case["zeta"])

    def src(n, b, bid):
        s = eng.gen_sketch(spec, n, b, bid)
        if s.is_dense:
            return SketchArrays(True, s.rows, s.cols, dense=s.dense, p=s.p)
        return SketchArrays(False, s.rows, s.cols, col_ptr=s.col_ptr, row_idx=s.row_idx, values=s.values,
                            centered=s.centered, p=s.p, std_scale=s.std_scale)
    ref = port.run(np.asfortranarray(a), eps=1e-3, power=case["power"], block=case["block"], kind=case["kind"],
                   p=case["p"], seed=5, zeta=case["zeta"], relative=True, source=src, want_vectors=True)
    assert ref.status == 0 and o0["converged"]
    assert (o0["rank"], o0["blocks"], o0["ids"]) == (ref.rank, ref.blocks, ref.block_ids)
    na = ref.norm_a_sq
    assert abs(o0["na"] - na) <= 1e-12 * na
    assert abs(o0["e"] - ref.residual_sq) <= 1e-10 * na
    assert np.max(np.abs(o0["trace"] - ref.block_residuals)) <= 1e-10 * na
    q = np.vstack([o0["q"], o1["q"]])
    assert o0["rows"][1] == o1["rows"][0] and q.shape[0] == M
    assert np.abs(q.T @ q - np.eye(q.shape[1])).max() < 1e-12
    usv = (ref.u * ref.sigma) @ ref.v.T
    assert np.linalg.norm(q @ o0["bt"].T - usv) <= 1e-10 * np.sqrt(na)
    top = ref.sigma >= 1e-3 * ref.sigma[-1]
    assert np.max(np.abs(o0["sigma"][top] - ref.sigma[top])) <= 1e-10 * ref.sigma[-1]
    # the SVD assembly's U rows of both ranks stack to an orthonormal U with U S V' = Q B
    u = np.vstack([o0["u"], o1["u"]])
    assert np.abs(u.T @ u - np.eye(u.shape[1])).max() < 1e-11
