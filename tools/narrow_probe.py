"""Host-side narrowing throughput probe: int64 -> int32 on the host threads
(torch CPU copy with dtype conversion) against the pinned H2D copy rate."""
import os
import time

import torch

n = (1 << 30)  # 1 G elements = 8 GiB int64
src = torch.randint(0, 1 << 26, (n,), dtype=torch.int64).pin_memory()
dst32 = torch.empty(n, dtype=torch.int32).pin_memory()
dev64 = torch.empty(n, dtype=torch.int64, device="cuda")
dev32 = torch.empty(n, dtype=torch.int32, device="cuda")
print("cpus", os.cpu_count(), "torch threads", torch.get_num_threads())
for th in (1, 4, 8, 16):
    torch.set_num_threads(th)
    c = 1 << 27
    t0 = time.perf_counter()
    dst32[:c].copy_(src[:c])
    dt = time.perf_counter() - t0
    t0 = time.perf_counter()
    dst32.copy_(src)
    dt2 = time.perf_counter() - t0
    print(f"narrow threads={th}: {8 * c / dt / 1e9:.1f} GB/s (1 GiB chunk), {8 * n / dt2 / 1e9:.1f} GB/s (8 GiB)")
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev64.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    t0 = time.perf_counter()
    dev32.copy_(dst32, non_blocking=True)
    torch.cuda.synchronize()
    dt2 = time.perf_counter() - t0
    print(f"H2D int64 {8 * n / dt / 1e9:.1f} GB/s, int32 {4 * n / dt2 / 1e9:.1f} GB/s")
