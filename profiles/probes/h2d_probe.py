"""Probe: host->device bandwidth of pinned copies by size and stream count."""
import time

import torch

for mb in (1, 6.5, 26, 105, 420):
    n = int(mb * 1024 * 1024) // 8
    h = torch.empty(n, dtype=torch.int64, pin_memory=True)
    d = torch.empty(n, dtype=torch.int64, device="cuda")
    for k in (1, 2, 4):
        ss = [torch.cuda.Stream() for _ in range(k)]
        for _ in range(3):
            for i, s in enumerate(ss):
                with torch.cuda.stream(s):
                    d[i * n // k:(i + 1) * n // k].copy_(h[i * n // k:(i + 1) * n // k], non_blocking=True)
        torch.cuda.synchronize()
        reps = 20 if mb < 100 else 5
        t0 = time.perf_counter()
        for _ in range(reps):
            for i, s in enumerate(ss):
                with torch.cuda.stream(s):
                    d[i * n // k:(i + 1) * n // k].copy_(h[i * n // k:(i + 1) * n // k], non_blocking=True)
            torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / reps
        print("%6.1f MB  streams %d: %.1f us  %.1f GB/s" % (mb, k, dt * 1e6, n * 8 / dt / 1e9))
