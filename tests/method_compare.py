#!/usr/bin/env python
"""Method comparison on B200 (the paper's Figs. 8-10 claims):
ozIMMU (bitmask + per-product), ozIMMU_RN, ozIMMU_EF and ozIMMU_H at the same
shape / k, device-timed, with max_rel_err vs the reference's exact oracle on a
sampled block.  Test infrastructure (the oracle is the checker).

    python tests/method_compare.py --n 16384 --k 8 --phi 0.5 --out profiles/r1/methods.csv
"""
from __future__ import annotations

import argparse
import csv
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--k", default="8")
    ap.add_argument("--phi", type=float, default=0.5)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--sample", type=int, default=48)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import torch

    from oracle import oracle
    from paper_2409_13313_b200 import ozmm
    chk = oracle.best()
    n = a.n
    A = ozmm.gen_phi_matrix(n, n, a.phi, ozmm.counter_hash(0, 1))
    B = ozmm.gen_phi_matrix(n, n, a.phi, ozmm.counter_hash(0, 2))
    rng = np.random.default_rng(7)
    I = np.sort(rng.choice(n, a.sample, replace=False))
    J = np.sort(rng.choice(n, a.sample, replace=False))
    exact = chk.exact_gemm(np.ascontiguousarray(A[I]), np.ascontiguousarray(B[:, J]))
    dA, dB = torch.tensor(A, device="cuda"), torch.tensor(B, device="cuda")
    C = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    rows = []
    for k in [int(x) for x in a.k.split(",")]:
        base = None
        for meth in ("ozIMMU", "ozIMMU_RN", "ozIMMU_EF", "ozIMMU_H"):
            cfg = ozmm.config_for(meth, k)
            ozmm.ozaki_gemm_ex(1.0, dA, dB, 0.0, C, cfg, out=C)  # warm-up
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            gemm_ms = 0.0
            for _ in range(a.reps):
                res = ozmm.ozaki_gemm_ex(1.0, dA, dB, 0.0, C, cfg, out=C)
                gemm_ms += res.timings.int_gemm * 1e3
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.reps
            err = chk.max_rel_err(C.cpu().numpy()[np.ix_(I, J)], exact)
            if meth == "ozIMMU":
                base = ms
            row = dict(n=n, k=k, phi=a.phi, method=meth, ms=ms, gemm_ms=gemm_ms / a.reps,
                       tflops=2.0 * n ** 3 / (ms * 1e-3) / 1e12, speedup_vs_ozIMMU=base / ms,
                       fp64_flushes=res.counts.fp64_flushes, max_rel_err=err)
            rows.append(row)
            print(" ".join(f"{k_}={v:.4g}" if isinstance(v, float) else f"{k_}={v}"
                           for k_, v in row.items()), flush=True)
    if a.out:
        os.makedirs(os.path.dirname(os.path.abspath(a.out)), exist_ok=True)
        with open(a.out, "w", newline="") as f:
            w = csv.DictWriter(f, fieldnames=list(rows[0]))
            w.writeheader()
            w.writerows(rows)


if __name__ == "__main__":
    main()
