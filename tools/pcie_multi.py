"""H2D throughput (pinned) with 1, 2 and 4 concurrent copy streams, 2 GiB total."""
import time

import torch

N = 1 << 28
h = torch.empty(N, dtype=torch.float64).pin_memory()
d = torch.empty(N, dtype=torch.float64, device="cuda")
for ns in (1, 2, 4, 1, 2):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = N // ns
    def go():
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
    go()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        go()
    torch.cuda.synchronize()
    print(f"{ns} stream(s): {3 * 8 * N / (time.perf_counter() - t) / 1e9:.1f} GB/s", flush=True)
