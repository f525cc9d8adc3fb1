#!/usr/bin/env python
"""The Python drop-in at C3 on numpy arrays: ozaki_gemm_ex (host path: a new
result matrix, C read-only, ozmm_dgemm_host_out) per-call wall time, and what the
round-1/2 path added on top (a full copy of C before the call)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_13313_b200 import ozmm  # noqa: E402

m = n = p = int(os.environ.get("N", 16384))
rng = np.random.default_rng(0)
A = (rng.random((m, n)) - 0.5) * np.exp(0.5 * rng.standard_normal((m, n)))
B = (rng.random((n, p)) - 0.5) * np.exp(0.5 * rng.standard_normal((n, p)))
C = np.zeros((m, p))
cfg = ozmm.config_for(ozmm.Method.ozIMMU_H, 8)
ms = []
for _ in range(4):
    t0 = time.perf_counter()
    D = ozmm.ozaki_gemm(1.0, A, B, 0.0, C, cfg)
    ms.append(round((time.perf_counter() - t0) * 1e3, 2))
t0 = time.perf_counter()
C2 = C.copy()
copy_ms = (time.perf_counter() - t0) * 1e3
print(json.dumps({"ozaki_gemm_ms": ms, "c_copy_ms_saved": round(copy_ms, 2),
                  "tflops_best": round(2.0 * m * n * p / min(ms[1:]) / 1e9, 2)}))
