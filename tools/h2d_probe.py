"""H2D rate of C4's 16 GB A from pinned host memory: one copy vs column chunks spread over
1, 2 or 4 streams (is the PCIe link the limit, or the single copy?)."""
import time

import torch

n_bytes = 100000 * 20000 * 8
h = torch.empty(n_bytes // 8, dtype=torch.float64, pin_memory=True)
h.fill_(1.0)
d = torch.empty_like(h, device="cuda")
torch.cuda.synchronize()


def run(nstreams, chunk):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    off, i = 0, 0
    n = h.numel()
    while off < n:
        e = min(n, off + chunk)
        with torch.cuda.stream(streams[i % nstreams]):
            d[off:e].copy_(h[off:e], non_blocking=True)
        off, i = e, i + 1
    torch.cuda.synchronize()
    return n_bytes / (time.perf_counter() - t0) / 1e9


for ns, ch in [(1, h.numel()), (1, 1 << 27), (2, 1 << 27), (4, 1 << 27), (2, 1 << 25), (4, 1 << 25), (1, h.numel())]:
    print(f"streams {ns} chunk {ch * 8 / 2**20:.0f} MiB: {run(ns, ch):.1f} GB/s", flush=True)
