"""Host-side copy bandwidth on the GPU box (design probe for the e2e result copy): pinned -> pinned
torch copies of 1 GiB with 1..N threads, and D2H DMA of the same size."""
import os
import time

import torch

n = 1 << 27  # 1 GiB of float64
a = torch.empty(n, dtype=torch.float64, pin_memory=True).fill_(1.0)
b = torch.empty(n, dtype=torch.float64, pin_memory=True)
print("cpu count", os.cpu_count())
for t in (1, 4, 8, 16, 32, os.cpu_count()):
    torch.set_num_threads(t)
    b.copy_(a)
    t0 = time.perf_counter()
    for _ in range(3):
        b.copy_(a)
    dt = (time.perf_counter() - t0) / 3
    print(f"threads {t}: {8 * n / dt / 1e9:.1f} GB/s")
d = torch.empty(n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
for _ in range(2):
    t0 = time.perf_counter()
    b.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    print(f"D2H DMA: {8 * n / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
    t0 = time.perf_counter()
    d.copy_(a, non_blocking=True)
    torch.cuda.synchronize()
    print(f"H2D DMA: {8 * n / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
