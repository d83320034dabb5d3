import sys, torch
sys.path.insert(0, "/root/repo")
import paper_2506_03859_b200 as fqb
eng = fqb.Engine(0)
for (m, n) in [(8000, 8000), (100000, 1000), (8000, 125000), (100000, 2000), (4096, 1000), (4097, 1000), (8192, 1000), (12288, 1000), (16384, 1000)]:
    a = torch.ones(n, m, dtype=torch.float64, device="cuda").t()
    got = eng.frob_norm_sq(a.data_ptr(), m, n, m)
    print(m, n, m * n, got, got / (m * n), flush=True)
    del a; torch.cuda.empty_cache()
