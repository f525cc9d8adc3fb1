"""Bit-exactness of batch cuts with chunk pieces (diag OZMM_SCHED_SETS c:s0-s1) vs the
reference build, incl. INT32 chunk dumps: n = 16384 (r = 8) and n = 8192 (r = 16)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle  # checker
from paper_2409_13313_b200 import ozmm

CASES = [(16384, 9, "0.1.2.8:1-1/3.4.5/6.7.8:2-8.9"), (16384, 9, "0.1.8:1-1/2.3.4.5/6.7.8:2-8.9"),
         (8192, 9, "0.1.2.8:1-1/3.4.5/6.7.8:2-9"), (8192, 10, "0.1.2.9:1-2/3.4.5.8:1-1/6.7.8:2-9.9:3-10"),
         (8192, 9, "8:1-3.0.1/2.3.4.8:4-5/5.6.7.8:6-9")]
for n, k, sets in CASES:
    m, p = 256, 384
    A = ozmm.gen_phi_matrix(m, n, 0.5, ozmm.counter_hash(4, 1))
    B = ozmm.gen_phi_matrix(n, p, 0.5, ozmm.counter_hash(4, 2))
    C = ozmm.gen_phi_matrix(m, p, 0.5, ozmm.counter_hash(4, 3))
    d = lambda x: torch.tensor(x, device="cuda")  # noqa: E731
    ch = oracle.RefLib().groupwise_chunks(A, B, k)
    for signed in (False, True):
        os.environ["OZMM_SCHED_SETS"] = sets
        dump = torch.zeros((ch.acc.shape[0], m, p), dtype=torch.int32, device="cuda")
        got = ozmm.ozaki_gemm(1.5, d(A), d(B), 0.5, d(C), ozmm.config_for("ozIMMU_H", k), chunk_dump=dump,
                              signed_slices=signed).cpu().numpy()
        got2 = ozmm.ozaki_gemm(1.5, d(A), d(B), 0.5, d(C), ozmm.config_for("ozIMMU_H", k),
                               signed_slices=signed).cpu().numpy()
        del os.environ["OZMM_SCHED_SETS"]
        want = oracle.best().gemm(1.5, A, B, 0.5, C, k=k)
        bad = int((got.view(np.uint64) != want.view(np.uint64)).sum())
        bad2 = int((got2.view(np.uint64) != want.view(np.uint64)).sum())
        dbad = int((dump.cpu().numpy() != ch.acc).sum())
        print(f"pieces n={n} k={k} signed={signed} {sets}: C {bad}+{bad2} of {got.size} differ, dumps {dbad} differ")
