#!/usr/bin/env python
"""Section-5 error bounds on GPU results at scale.

verify_bounds (proj/src/harness.cpp:137-187) on the B200 path: for each
(phi, k, method), D = ozaki_mm(A, B) on the GPU at full size; on a sampled
block I x J the reference's own total_bound (analysis.cpp:73-100, |A||B| from
exact_gemm_oracle) is evaluated and max |D - exact| / bound must be <= 1.
Bounds are entry-local (g_i, f_j, n, k, beta, r, w), so the block check is exact.
`--inject-error` corrupts D[I0, J0] first (the reference's negative control,
harness.cpp:154-155) and must fail.  Test infrastructure (oracle = checker).
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(n, phis, ks, methods, sample, inject=False, seed=0, verbose=True):
    import torch

    from oracle import oracle
    from paper_2409_13313_b200 import ozmm
    ref = oracle.RefLib()
    rng = np.random.default_rng(seed)
    I = np.sort(rng.choice(n, min(sample, n), replace=False))
    J = np.sort(rng.choice(n, min(sample, n), replace=False))
    ok, cells = True, []
    for phi in phis:
        A = ozmm.gen_phi_matrix(n, n, phi, ozmm.counter_hash(seed, 1))
        B = ozmm.gen_phi_matrix(n, n, phi, ozmm.counter_hash(seed, 2))
        Ab, Bb = np.ascontiguousarray(A[I]), np.ascontiguousarray(B[:, J])
        exact = ref.exact_gemm(Ab, Bb)
        dA, dB = torch.tensor(A, device="cuda"), torch.tensor(B, device="cuda")
        for k in ks:
            for meth in methods:
                d = ozmm.ozaki_mm(dA, dB, ozmm.config_for(meth, k)).d.cpu().numpy()[np.ix_(I, J)]
                if inject:
                    d[0, 0] += abs(d[0, 0]) * 2.0 ** -20 + 1.0
                bound = ref.total_bound(Ab, Bb, k, meth)
                err = np.abs(d - exact)
                bad_zero = ((bound == 0) & (err != 0)).any()
                ratio = np.where(bound > 0, err / np.where(bound > 0, bound, 1), 0).max()
                cell_ok = (not bad_zero) and ratio <= 1.0
                ok &= cell_ok
                cells.append((phi, k, meth, float(ratio), cell_ok))
                if verbose:
                    print(f"n={n} phi={phi} k={k:2d} {meth:10s} max err/bound = {ratio:.3e} "
                          f"{'ok' if cell_ok else 'FAIL'}", flush=True)
    return ok, cells


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--phi", default="0.5,2")
    ap.add_argument("--k", default="3,6,8,10")
    ap.add_argument("--methods", default="ozIMMU,ozIMMU_RN,ozIMMU_EF,ozIMMU_H")
    ap.add_argument("--sample", type=int, default=32)
    ap.add_argument("--inject-error", action="store_true")
    a = ap.parse_args()
    ok, _ = run(a.n, [float(x) for x in a.phi.split(",")], [int(x) for x in a.k.split(",")],
                a.methods.split(","), a.sample, a.inject_error)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
