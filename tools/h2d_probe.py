import torch, time
x = torch.empty(512*1024*1024//8, dtype=torch.float64).pin_memory()
y = torch.empty_like(x, device="cuda")
for i in range(3):
    torch.cuda.synchronize(); t=time.perf_counter(); y.copy_(x, non_blocking=True); torch.cuda.synchronize(); dt=time.perf_counter()-t
    print(f"H2D pinned 512MB: {dt*1e3:.2f} ms = {0.512/dt:.1f} GB/s")
z = torch.empty(51*1024*1024//8, dtype=torch.float64)  # pageable
w = torch.empty_like(z, device="cuda")
for i in range(2):
    torch.cuda.synchronize(); t=time.perf_counter(); z.copy_(w); torch.cuda.synchronize(); dt=time.perf_counter()-t
    print(f"D2H pageable 51MB: {dt*1e3:.2f} ms = {0.051/dt:.1f} GB/s")
zp = z.pin_memory()
for i in range(2):
    torch.cuda.synchronize(); t=time.perf_counter(); zp.copy_(w, non_blocking=True); torch.cuda.synchronize(); dt=time.perf_counter()-t
    print(f"D2H pinned 51MB: {dt*1e3:.2f} ms = {0.051/dt:.1f} GB/s")
