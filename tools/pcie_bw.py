"""Raw host<->device copy bandwidth on the box (pinned), for the e2e roofline."""
import time
import torch

N = 1 << 28  # 2 GiB of float64
h = torch.empty(N, dtype=torch.float64).pin_memory()
h2 = torch.empty(N, dtype=torch.float64).pin_memory()
d = torch.empty(N, dtype=torch.float64, device="cuda")
d2 = torch.empty(N, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d.copy_(h, non_blocking=True); h.copy_(d, non_blocking=True)
torch.cuda.synchronize()
def bw(f, nbytes, reps=3):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize(); return nbytes * reps / (time.perf_counter() - t) / 1e9
print("H2D GB/s", bw(lambda: d.copy_(h, non_blocking=True), 8 * N))
print("D2H GB/s", bw(lambda: h.copy_(d, non_blocking=True), 8 * N))
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
print("H2D+D2H concurrent GB/s (sum)", bw(both, 16 * N))
