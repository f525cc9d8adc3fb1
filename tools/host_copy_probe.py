"""Host memcpy bandwidth on the GPU box (pageable -> pinned, T threads) and the
driver's own pageable H2D / D2H rates: the inputs of the staging design in
csrc/host_stage.hpp."""
import threading
import time

import numpy as np
import torch

N = 1 << 28  # 2 GiB
src = np.random.default_rng(0).random(N)
pin = torch.empty(N, dtype=torch.float64).pin_memory().numpy()
dev = torch.empty(N, dtype=torch.float64, device="cuda")


def par_copy(dst, s, T):
    ths = []
    for t in range(T):
        lo, hi = N * t // T, N * (t + 1) // T
        ths.append(threading.Thread(target=np.copyto, args=(dst[lo:hi], s[lo:hi])))
    t0 = time.perf_counter()
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    return 8 * N / (time.perf_counter() - t0) / 1e9


for T in (1, 2, 4, 8, 12, 16):
    par_copy(pin, src, T)
    print(f"memcpy pageable->pinned T={T:2d}: {max(par_copy(pin, src, T) for _ in range(3)):6.1f} GB/s")
    print(f"memcpy pinned->pageable T={T:2d}: {max(par_copy(src, pin, T) for _ in range(3)):6.1f} GB/s")
t = torch.from_numpy(src)
for name, f in (("driver pageable H2D", lambda: dev.copy_(t)), ("driver pageable D2H", lambda: t.copy_(dev))):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f()
    torch.cuda.synchronize()
    print(f"{name}: {8 * N / (time.perf_counter() - t0) / 1e9:6.1f} GB/s")
