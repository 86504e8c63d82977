"""PCIe host->device bandwidth for the triplet-stream upload (1.38 GB of
values, pinned), split over 1 / 2 / 4 concurrent copy streams."""
import time

import torch

n = 1_380_000_000 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
for k in (1, 2, 4, 1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(k)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    step = (n + k - 1) // k
    for i, s in enumerate(streams):
        with torch.cuda.stream(s):
            d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{k} stream(s): {n * 8 / dt / 1e9:.1f} GB/s", flush=True)
