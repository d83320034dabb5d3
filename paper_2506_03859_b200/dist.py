"""Row-sharded multi-GPU host logic (one process per GPU, torch.distributed plumbing).

The device side lives in libfarqb (csrc/comm.cu): with a communicator attached,
each rank passes its contiguous row block of A to run_fixed_precision and the
engine all-reduces ||A||^2, A'Y and the Gram blocks over NVLink with NCCL.
This module decides the row blocks and distributes the NCCL unique id.
"""
from __future__ import annotations

import ctypes as C


def partition_rows(m: int, world: int, rank: int, align: int = 16) -> tuple[int, int]:
    """Contiguous, balanced row block [r0, r1) of rank `rank`, boundaries on
    multiples of `align` rows (TMA-friendly) except the last one."""
    if not (0 <= rank < world) or m < 1:
        raise ValueError("bad partition request")
    chunks = (m + align - 1) // align
    c0 = (chunks * rank) // world
    c1 = (chunks * (rank + 1)) // world
    return min(m, c0 * align), min(m, c1 * align)


def exchange_unique_id(make_id, group=None) -> bytes:
    """Rank 0 calls make_id() -> 128 bytes; every rank gets the same bytes."""
    import torch.distributed as dist
    obj = [make_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def nccl_unique_id() -> bytes:
    from . import _native
    from .rsvd import _raise
    buf = C.create_string_buffer(128)
    st = _native.lib().fqb_comm_unique_id(buf)
    if st:
        _raise(st, "fqb_comm_unique_id")
    return buf.raw


def attach(engine, group=None) -> None:
    """Attach a NCCL communicator spanning `group` to `engine` (collective call)."""
    import torch.distributed as dist
    from . import _native
    from .rsvd import _raise
    uid = exchange_unique_id(nccl_unique_id, group)
    buf = C.create_string_buffer(uid, 128)
    st = _native.lib().fqb_comm_attach(engine._h, buf, dist.get_world_size(group), dist.get_rank(group))
    if st:
        _raise(st, "fqb_comm_attach")


def attach_host(engine, group=None) -> None:
    """Attach the host reduction backend (fqb_comm_attach_host): every reduction point of
    the engine becomes a torch.distributed all-reduce of a CPU tensor (gloo), so the row-
    sharded loop runs with any process group -- several ranks may even share one GPU, as
    no kernel waits on another rank.  Collective call."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from . import _native
    from .rsvd import _raise

    def cb(_user, buf, count):
        try:
            t = torch.from_numpy(np.ctypeslib.as_array(buf, (int(count),)))
            dist.all_reduce(t, group=group)
            # every rank must take the same decisions from the same bits: rank 0's sum wins
            dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
            return 0
        except Exception:  # noqa: BLE001 - reported through the status
            return 1

    fn = _native.HOST_ALLREDUCE_FN(cb)
    engine._host_ar_fn = fn          # kept alive as long as the engine uses it
    st = _native.lib().fqb_comm_attach_host(engine._h, fn, None, dist.get_world_size(group), dist.get_rank(group))
    if st:
        _raise(st, "fqb_comm_attach_host")
