"""Does splitting one 512 MB pinned H2D copy over several streams raise PCIe throughput?"""
import time

import torch

x = torch.empty(512 * 1024 * 1024 // 8, dtype=torch.float64).pin_memory()
y = torch.empty_like(x, device="cuda")
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = x.numel() // ns
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                y[i * chunk:(i + 1) * chunk].copy_(x[i * chunk:(i + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"{ns} stream(s): {dt * 1e3:.2f} ms = {0.536870912 / dt:.1f} GB/s")
