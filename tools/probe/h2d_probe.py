"""H2D bandwidth probe: one 4.29 GB pinned->device copy vs. split copies on
several streams (the e2e leg of bench.py is bound by this copy)."""
import time
import torch

n = (1 << 29)  # doubles = 4.29 GB
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
h.fill_(1.0)
d = torch.empty(n, dtype=torch.float64, device="cuda")
for parts in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(parts)]
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        step = n // parts
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
    print(f"parts={parts} {8 * n / el / 1e9:.1f} GB/s", flush=True)
