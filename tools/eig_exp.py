import os, sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2506_03859_b200 as fqb
eng = fqb.default_engine(0)
n = 2000
rng = np.random.default_rng(0)
q, _ = np.linalg.qr(rng.standard_normal((n, n)))
m = (q * 10.0 ** (-6 * np.arange(n) / n)) @ q.T
m = torch.from_numpy(np.asfortranarray(0.5 * (m + m.T))).cuda()
def t(fn, reps=5):
    for _ in range(2): fn()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps * 1e3
for mode in ["syevd", "syevj", "large"]:
    os.environ["FQB_EIG"] = mode
    try:
        print(mode, f"{t(lambda: eng.sym_eig(m)):.2f} ms", flush=True)
    except Exception as e:
        print(mode, "error", e)
print("torch.linalg.eigh", f"{t(lambda: torch.linalg.eigh(m)):.2f} ms")
print("torch.linalg.eigvalsh", f"{t(lambda: torch.linalg.eigvalsh(m)):.2f} ms")
mm = m.float()
print("torch.linalg.eigh fp32", f"{t(lambda: torch.linalg.eigh(mm)):.2f} ms")
