import time, numpy as np, torch
n = 112 * 1024 * 1024 // 8
a = np.random.rand(n)
b = np.empty_like(a)
for _ in range(2): np.copyto(b, a)
t = time.perf_counter(); 
for _ in range(5): np.copyto(b, a)
dt = (time.perf_counter() - t) / 5
print(f"host memcpy 1 thread: {a.nbytes/dt/1e9:.1f} GB/s ({dt*1e3:.2f} ms)")
p = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
for _ in range(3): d.copy_(p, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5): d.copy_(p, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 5
print(f"H2D pinned: {a.nbytes/dt/1e9:.1f} GB/s ({dt*1e3:.2f} ms)")
src = torch.from_numpy(a)
t = time.perf_counter()
for _ in range(3): d.copy_(src)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 3
print(f"H2D pageable: {a.nbytes/dt/1e9:.1f} GB/s ({dt*1e3:.2f} ms)")
