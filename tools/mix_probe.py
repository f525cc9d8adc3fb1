#!/usr/bin/env python
"""Would mixing the L2-heavy first batch with the MMA-heavy second batch across SMs
help?  Runs C3's batch 0 and batch 1 (OZMM_ONLY_BATCH, timing only) back to back
and concurrently on two streams, and prints the times (ms)."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_13313_b200 import ozmm  # noqa: E402

n = 16384
k = 8
dev = torch.device("cuda", 0)
A = torch.from_numpy(ozmm.gen_phi_block(n, n, 0.5, ozmm.counter_hash(0, 1))).to(dev)
B = torch.from_numpy(ozmm.gen_phi_block(n, n, 0.5, ozmm.counter_hash(0, 2))).to(dev)
sa = ozmm.split_rn_const_shift(A, k, "L")
sb = ozmm.split_rn_const_shift(B, k, "R")
C1 = torch.zeros((n, n), dtype=torch.float64, device=dev)
C2 = torch.zeros((n, n), dtype=torch.float64, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h1, h2 = ozmm.Handle(0), ozmm.Handle(0)


def launch(h, st, C, batch):
    os.environ["OZMM_ONLY_BATCH"] = str(batch)
    h.set_stream(st.cuda_stream)
    h.check(ozmm.lib.ozmm_gemm_slices(h.h, n, n, n, k, sa.beta, 0, sa.slices.data_ptr(),
                                      sa.slices.shape[-1], sa.shift.data_ptr(), sb.slices.data_ptr(),
                                      sb.slices.shape[-1], sb.shift.data_ptr(), 1.0, 0.0,
                                      C.data_ptr(), n, None))


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


print("batch0 alone", timed(lambda: launch(h1, s1, C1, 0)))
print("batch1 alone", timed(lambda: launch(h2, s2, C2, 1)))
print("serial b0+b1", timed(lambda: (launch(h1, s1, C1, 0), launch(h1, s1, C2, 1))))
print("concurrent b0|b1", timed(lambda: (launch(h1, s1, C1, 0), launch(h2, s2, C2, 1))))
os.environ.pop("OZMM_ONLY_BATCH")
print("full kernel", timed(lambda: launch(h1, s1, C1, -1)))
