#!/usr/bin/env python
"""Per-call times of ozmm_dgemm_host at C3 (pinned host buffers, like bench.py's e2e):
    python tools/e2e_jitter.py [--calls 12]
Prints each call's wall time, to separate run-to-run jitter from the mean."""
import argparse
import ctypes
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--calls", type=int, default=12)
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--pageable", action="store_true", help="plain numpy (pageable) buffers")
    ap.add_argument("--staging", type=int, default=0, help="ozmm_options_t.host_staging")
    ap.add_argument("--col-split", type=int, default=0, help="ozmm_options_t.col_split")
    args = ap.parse_args()
    from paper_2409_13313_b200 import ozmm
    n = args.n
    hA = torch.from_numpy(ozmm.gen_phi_block(n, n, 0.5, ozmm.counter_hash(0, 1))).pin_memory()
    hB = torch.from_numpy(ozmm.gen_phi_block(n, n, 0.5, ozmm.counter_hash(0, 2))).pin_memory()
    hC = torch.zeros((n, n), dtype=torch.float64).pin_memory()
    h = ozmm.Handle(0)
    opt, cnt = ozmm.Options(), ozmm.Counts()
    if hasattr(opt, "host_staging"):
        opt.host_staging = args.staging
    if hasattr(opt, "col_split"):
        opt.col_split = args.col_split
    a, b, c = hA.numpy(), hB.numpy(), hC.numpy()
    if args.pageable:
        import numpy as np
        a, b, c = np.array(a), np.array(b), np.array(c)
    ts = []
    for _ in range(args.calls):
        t0 = time.perf_counter()
        h.check(ozmm.lib.ozmm_dgemm_host(h.h, b"N", b"N", n, n, n, 1.0, a.ctypes.data, n,
                                         b.ctypes.data, n, 0.0, c.ctypes.data, n, 8,
                                         ctypes.byref(opt), ctypes.byref(cnt), None))
        ts.append(round((time.perf_counter() - t0) * 1e3, 2))
    print(json.dumps({"ms": ts, "cores": os.cpu_count()}))


if __name__ == "__main__":
    main()
