"""Bit-exactness of explicit batch sets (diag OZMM_SCHED_SETS) vs the reference build:
m = p = 256, n = 16384 (r = 8) and n = 8192 (r = 16)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle  # checker
from paper_2409_13313_b200 import ozmm

for n, k, sets in [(16384, 9, "0.1.2.9/3.4.5/6.7.8"), (16384, 9, "0.1.2.3/4.5.6.9/7.8"),
                   (8192, 9, "0.1.2.8/3.4.5/6.7"), (8192, 10, "0.1/2.3.4/5.6.7/8.9")]:
    m = p = 256
    A = ozmm.gen_phi_matrix(m, n, 0.5, ozmm.counter_hash(3, 1))
    B = ozmm.gen_phi_matrix(n, p, 0.5, ozmm.counter_hash(3, 2))
    C = ozmm.gen_phi_matrix(m, p, 0.5, ozmm.counter_hash(3, 3))
    os.environ["OZMM_SCHED_SETS"] = sets
    d = lambda x: torch.tensor(x, device="cuda")  # noqa: E731
    got = ozmm.ozaki_gemm(1.5, d(A), d(B), 0.5, d(C), ozmm.config_for("ozIMMU_H", k)).cpu().numpy()
    del os.environ["OZMM_SCHED_SETS"]
    want = oracle.best().gemm(1.5, A, B, 0.5, C, k=k)
    bad = int((got.view(np.uint64) != want.view(np.uint64)).sum())
    print(f"sets n={n} k={k} {sets}: {bad} of {got.size} differ")
