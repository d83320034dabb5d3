import torch, time
torch.backends.cuda.matmul.allow_tf32 = False
for (M, N, K) in [(8192, 8192, 8192), (8000, 50, 8000), (20000, 64, 20000), (100000, 100, 20000)]:
    a = torch.randn(M, K, dtype=torch.float64, device="cuda")
    b = torch.randn(K, N, dtype=torch.float64, device="cuda")
    for _ in range(3): c = a @ b
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): c = a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"cublas dgemm NN {M}x{N}x{K}: {ms:.3f} ms {2*M*N*K/ms/1e9:.2f} TFLOP/s")
    at = a.t()  # TN shape: (K x M)^T...
    a2 = torch.randn(K, M, dtype=torch.float64, device="cuda")
    bb = torch.randn(K, N, dtype=torch.float64, device="cuda")
    for _ in range(3): c = a2.t() @ bb
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10): c = a2.t() @ bb
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"cublas dgemm TN {M}x{N}x{K}: {ms:.3f} ms {2*M*N*K/ms/1e9:.2f} TFLOP/s")
    del a, b, a2, bb, c
    torch.cuda.empty_cache()
