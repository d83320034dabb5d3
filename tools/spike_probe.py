"""Per-step device times of repeated C2 runs under different conditions (spike hunt)."""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_03859_b200 as fqb  # noqa: E402

eng = fqb.Engine(0)
st = torch.cuda.Stream()
eng.set_stream(st.cuda_stream)
a = bench.make_matrix(torch.device("cuda:0"))
torch.cuda.synchronize()
cfg = bench.config()
for mode in ("none", "device-keep", "device-drop"):
    keep = []
    ts = []
    for i in range(12):
        r = eng.run_fixed_precision(a, cfg, output="none" if mode == "none" else "device")
        ts.append(round(r.elapsed_ms, 2))
        if mode == "device-keep":
            keep.append(r)
    print(mode, ts, flush=True)
proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv", "-lms", "50"],
                        stdout=subprocess.DEVNULL)
time.sleep(0.3)
ts = [round(eng.run_fixed_precision(a, cfg, output="none").elapsed_ms, 2) for _ in range(12)]
proc.terminate()
print("with nvidia-smi polling", ts, flush=True)
