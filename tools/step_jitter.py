"""Per-step device time of the bench step (C4 run_fixed_precision + SVD) next to the SM
clock / power / throttle reasons sampled (NVML, 10 ms) during that step.

    python tools/step_jitter.py [steps]
"""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_03859_b200 as fqb  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
pynvml.nvmlInit()
hd = pynvml.nvmlDeviceGetHandleByIndex(0)
samples = []
stop = False


def poll():
    while not stop:
        samples.append((time.perf_counter(), pynvml.nvmlDeviceGetClockInfo(hd, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(hd) / 1000.0,
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(hd)))
        time.sleep(0.01)


eng = fqb.Engine(0)
a = bench.make_matrix(eng)
cfg = bench.config()
for _ in range(2):
    eng.run_fixed_precision(a, cfg, output="device", svd=True)
torch.cuda.synchronize()
t = threading.Thread(target=poll, daemon=True)
t.start()
for i in range(steps):
    t0 = time.perf_counter()
    r = eng.run_fixed_precision(a, cfg, output="device", svd=True)
    t1 = time.perf_counter()
    ms = r.elapsed_ms
    r = None
    win = [s for s in samples if t0 <= s[0] <= t1]
    clk = sum(s[1] for s in win) / max(1, len(win))
    pw = max((s[2] for s in win), default=0)
    rs = 0
    for s in win:
        rs |= s[3]
    print(f"step {i}: device {ms:8.1f} ms  wall {1e3 * (t1 - t0):8.1f} ms  sm {clk:6.0f} MHz  "
          f"power max {pw:6.0f} W  reasons 0x{rs:x}", flush=True)
stop = True
