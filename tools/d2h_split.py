"""D2H of a 4K visibility buffer (66 MB) into pinned memory: one copy vs the
buffer split over 2 / 4 streams (copy engines), CUDA-event / wall timed."""
import time

import torch

n = 3840 * 2160
d = torch.full((n,), -1, dtype=torch.int64, device="cuda")
p = torch.empty(n, dtype=torch.int64, pin_memory=True)
torch.cuda.synchronize()
for parts in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(parts)]
    best = 1e9
    for rep in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        step = (n + parts - 1) // parts
        for i, s in enumerate(streams):
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                p[i * step:(i + 1) * step].copy_(d[i * step:(i + 1) * step], non_blocking=True)
        for s in streams:
            s.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(f"parts {parts}: {best * 1e3:.3f} ms  {n * 8 / best / 1e9:.1f} GB/s", flush=True)
