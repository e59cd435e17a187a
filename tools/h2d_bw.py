"""Pinned H2D bandwidth with 1, 2 and 4 concurrent copy streams (diagnostics)."""
import time

import torch

N = 64 * 1024 * 1024  # doubles per buffer (512 MB)
h = torch.empty(N, dtype=torch.float64, pin_memory=True)
h.fill_(1.0)
d = torch.empty(N, dtype=torch.float64, device="cuda")
for ns in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = N // ns
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[k * chunk:(k + 1) * chunk].copy_(h[k * chunk:(k + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"{ns} streams: {N * 8 / dt / 1e9:.1f} GB/s")
