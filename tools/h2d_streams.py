"""Host->device bandwidth from pinned memory with 1, 2 and 4 concurrent copy streams (16 GB)."""
import time

import torch

n = 16 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h.fill_(3)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for k in (1, 2, 4, 1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(k)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    step = n // k
    for i, st in enumerate(streams):
        with torch.cuda.stream(st):
            d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{k} stream(s): {n / dt / 1e9:.1f} GB/s", flush=True)
# chunked on one stream (many 256 MB copies)
torch.cuda.synchronize()
t0 = time.perf_counter()
c = 256 << 20
for i in range(0, n, c):
    d[i:i + c].copy_(h[i:i + c], non_blocking=True)
torch.cuda.synchronize()
print(f"256 MB pieces: {n / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
