#!/usr/bin/env python
"""Accuracy sweep of the B200 ozIMMU_H path (paper Fig. 4).

For each (n, phi, seed): A = gen_phi_matrix(n, n, phi, counter_hash(seed, 1)),
B = gen_phi_matrix(n, n, phi, counter_hash(seed, 2)) exactly as the reference
harness (proj/src/harness.cpp:19-24).  D = ozaki_mm(A, B) runs on the GPU for
each k; native cuBLAS DGEMM (torch.matmul, FP64) is the comparator.  Errors are
max_rel_err (proj/src/oracle.cpp:321-335) against the correctly rounded
exact_gemm_oracle (oracle.cpp:276) of the reference build, evaluated on a
sampled block of rows I x columns J (exact oracle on full 8192^3 would take
hours on the CPU); the sample is stated in the CSV.

Writes the reference's sweep CSV schema (harness.cpp:40-42), one row per
(n, phi, k, method, seed), with methods "ozIMMU_H" (GPU), "cuBLAS_DGEMM" and
"FP64" (the reference's plain triple loop on the same block).

    python tests/accuracy_sweep.py --n 8192 --k 6-14 --phi 0.5,1,2,4 --seeds 1 \
        --out profiles/r1/accuracy_n8192.csv
Test infrastructure (imports the oracle as the checker).
"""
from __future__ import annotations

import argparse
import csv
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

HEADER = ("n,phi,k,method,seed,max_rel_err,int8_gemms,fp64_flushes,r,w,kprime_max,"
          "t_split_a,t_split_b,t_int_gemm,t_accum,t_copy").split(",")


def kprime_max(n: int, beta: int) -> int:
    """analysis.cpp:57-63."""
    if beta < 3:
        return 1
    budget = 51 - (int(n).bit_length() - 1)
    return max(1, budget // beta - 1)


def parse_list(s, typ):
    out = []
    for part in s.split(","):
        if "-" in part and typ is int:
            a, b = part.split("-")
            out += list(range(int(a), int(b) + 1))
        else:
            out.append(typ(part))
    return out


def run(ns, ks, phis, seeds, sample, out_path, verbose=True):
    import torch

    from oracle import oracle
    from paper_2409_13313_b200 import ozmm

    chk = oracle.best()
    rows = []
    rng = np.random.default_rng(12345)
    for n in ns:
        I = np.sort(rng.choice(n, min(sample, n), replace=False))
        J = np.sort(rng.choice(n, min(sample, n), replace=False))
        beta = ozmm.compute_beta(n)
        for phi in phis:
            for seed in seeds:
                A = ozmm.gen_phi_matrix(n, n, phi, ozmm.counter_hash(seed, 1))
                B = ozmm.gen_phi_matrix(n, n, phi, ozmm.counter_hash(seed, 2))
                Ab, Bb = np.ascontiguousarray(A[I, :]), np.ascontiguousarray(B[:, J])
                exact = chk.exact_gemm(Ab, Bb)
                dA = torch.tensor(A, device="cuda")
                dB = torch.tensor(B, device="cuda")
                # comparators on the same block
                cub = torch.matmul(dA, dB)
                torch.cuda.synchronize()
                e_cub = chk.max_rel_err(cub.cpu().numpy()[np.ix_(I, J)], exact)
                e_fp = chk.max_rel_err(chk.fp64_gemm(Ab, Bb), exact)
                for meth, e in (("cuBLAS_DGEMM", e_cub), ("FP64", e_fp)):
                    rows.append([n, phi, 0, meth, seed, e, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0])
                for k in ks:
                    res = ozmm.ozaki_mm(dA, dB, ozmm.config_for("ozIMMU_H", k))
                    d = res.d.cpu().numpy()
                    e = chk.max_rel_err(d[np.ix_(I, J)], exact)
                    t = res.timings
                    rows.append([n, phi, k, "ozIMMU_H", seed, e, res.counts.int8_gemms,
                                 res.counts.fp64_flushes, res.counts.r, res.counts.w,
                                 kprime_max(n, beta), t.split_a, t.split_b, t.int_gemm,
                                 t.accum_fp64, t.copy])
                    if verbose:
                        print(f"n={n} phi={phi} seed={seed} k={k:2d}: ozIMMU_H {e:.3e}  "
                              f"cuBLAS {e_cub:.3e}  FP64 {e_fp:.3e}  "
                              f"gemm {t.int_gemm * 1e3:.1f} ms", flush=True)
                del dA, dB
    if out_path:
        os.makedirs(os.path.dirname(os.path.abspath(out_path)), exist_ok=True)
        with open(out_path, "w", newline="") as f:
            f.write(f"# sampled block: |I| = |J| = {sample} rows/cols (seeded), exact = "
                    f"reference exact_gemm_oracle ({chk.kind} build); t_* from CUDA events\n")
            w = csv.writer(f)
            w.writerow(HEADER)
            for r in rows:
                w.writerow([f"{x:.17g}" if isinstance(x, float) else x for x in r])
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", default="8192")
    ap.add_argument("--k", default="6-14")
    ap.add_argument("--phi", default="0.5,1,2,4")
    ap.add_argument("--seeds", default="0")
    ap.add_argument("--sample", type=int, default=96)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    t0 = time.time()
    run(parse_list(a.n, int), parse_list(a.k, int), parse_list(a.phi, float),
        parse_list(a.seeds, int), a.sample, a.out)
    print(f"done in {time.time() - t0:.1f} s")


if __name__ == "__main__":
    main()
