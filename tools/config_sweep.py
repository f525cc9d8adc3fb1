#!/usr/bin/env python
"""Per-config throughput of the B200 ozIMMU_H path on every BASELINE.json config.

    python tools/config_sweep.py [--only C2,C4,C5] [--out profiles/r1/configs.csv]

For each config: inputs from the reference phi generator on the host, uploaded
once; the device path (ozaki_gemm_ex through ozmm_dgemm_ex, C overwritten in
place) is warmed up twice and timed over `--reps` back-to-back calls with CUDA
events on the launching stream (inputs are 0.5-17 GB, far above the 126 MB L2).
cuBLAS DGEMM (torch.matmul, FP64) is timed the same way on the same device
buffers.  max_rel_err (oracle.cpp:321-335) against the reference's exact oracle
is evaluated on a sampled block (|I| = |J| = --sample) for both -- the oracle is
the checker here, never the thing timed.

Configs (BASELINE.json):
  C2  m=n=p=8192, k = 6..14, phi = 0.5 / 1 / 2
  C3  m=n=p=16384, k = 8 (the headline; bench.py measures it too)
  C4  m=p=8192, n=65536, k = 8 (r = 2: INT32-overflow-safe inner chunks, w = 20)
  C5  m=n=p=16384, transa = transb = 'T', alpha = 1.5, beta = 0.5, phi = 4, k = 10/12/14
"""
from __future__ import annotations

import argparse
import csv
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

HEADER = ["config", "m", "n", "p", "k", "phi", "transa", "transb", "alpha", "beta",
          "r", "w", "int8_gemms", "ms", "emulated_tflops", "int8_tops", "cublas_dgemm_ms",
          "cublas_dgemm_tflops", "speedup_vs_dgemm", "max_rel_err", "dgemm_max_rel_err",
          "sample"]


def configs(only):
    out = []
    if "C2" in only:
        for phi in (0.5, 1.0, 2.0):
            for k in range(6, 15):
                out.append(("C2", 8192, 8192, 8192, k, phi, False, False, 1.0, 0.0))
    if "C3" in only:
        out.append(("C3", 16384, 16384, 16384, 8, 0.5, False, False, 1.0, 0.0))
    if "C4" in only:
        out.append(("C4", 8192, 65536, 8192, 8, 0.5, False, False, 1.0, 0.0))
    if "C5" in only:
        for k in (10, 12, 14):
            out.append(("C5", 16384, 16384, 16384, k, 4.0, True, True, 1.5, 0.5))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="C2,C3,C4,C5")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--sample", type=int, default=32)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1", "configs.csv"))
    args = ap.parse_args()

    import torch

    from oracle import oracle  # checker only
    from paper_2409_13313_b200 import ozmm

    chk = oracle.best()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    rng = np.random.default_rng(7)
    rows = []
    cache = {}
    for (name, m, n, p, k, phi, ta, tb, alpha, beta) in configs(args.only.split(",")):
        key = (m, n, p, phi, ta, tb)
        if key not in cache:
            cache.clear()
            torch.cuda.empty_cache()
            # stored shapes: A n x m when transa, B p x n when transb
            A = ozmm.gen_phi_matrix(*((n, m) if ta else (m, n)), phi, ozmm.counter_hash(0, 1))
            B = ozmm.gen_phi_matrix(*((p, n) if tb else (n, p)), phi, ozmm.counter_hash(0, 2))
            C = ozmm.gen_phi_matrix(m, p, phi, ozmm.counter_hash(0, 3))
            I = np.sort(rng.choice(m, args.sample, replace=False))
            J = np.sort(rng.choice(p, args.sample, replace=False))
            Aop, Bop = (A.T if ta else A), (B.T if tb else B)
            Ab, Bb = np.ascontiguousarray(Aop[I, :]), np.ascontiguousarray(Bop[:, J])
            exact_d = chk.exact_gemm(Ab, Bb)
            cache[key] = dict(dA=torch.tensor(A, device=dev), dB=torch.tensor(B, device=dev),
                              dC=torch.tensor(C, device=dev), C=C, I=I, J=J, exact_d=exact_d)
            del A, B
        e = cache[key]
        cfg = ozmm.config_for(ozmm.Method.ozIMMU_H, k)
        out = e["dC"].clone()

        def call():  # in place (C <- alpha*D + beta*C), no extra copy in the timed loop
            return ozmm.ozaki_gemm_ex(alpha, e["dA"], e["dB"], beta, out, cfg, transa=ta,
                                      transb=tb, out=out, timings=False)

        for _ in range(2):
            call()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.reps):
            call()
        e1.record(stream)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / args.reps
        out.copy_(e["dC"])
        res = call()  # the checked result, from the original C
        # exact reference value of alpha*A*B + beta*C on the block (C enters exactly)
        I, J = e["I"], e["J"]
        want = alpha * e["exact_d"] + beta * e["C"][np.ix_(I, J)]
        got = out.cpu().numpy()[np.ix_(I, J)]
        err = chk.max_rel_err(np.ascontiguousarray(got), np.ascontiguousarray(want))
        # cuBLAS DGEMM on the same buffers (op() via transposed views)
        opA = e["dA"].t() if ta else e["dA"]
        opB = e["dB"].t() if tb else e["dB"]
        cb = torch.empty_like(out)

        def dgemm():
            torch.addmm(e["dC"], opA, opB, beta=beta, alpha=alpha, out=cb)

        for _ in range(2):
            dgemm()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.reps):
            dgemm()
        e1.record(stream)
        torch.cuda.synchronize()
        tc = e0.elapsed_time(e1) / args.reps
        errc = chk.max_rel_err(np.ascontiguousarray(cb.cpu().numpy()[np.ix_(I, J)]),
                               np.ascontiguousarray(want))
        flops = 2.0 * m * n * p
        c = res.counts
        row = [name, m, n, p, k, phi, int(ta), int(tb), alpha, beta, c.r, c.w, c.int8_gemms,
               round(t, 3), round(flops / t / 1e9, 2),
               round(c.int8_gemms * flops / t / 1e9, 1), round(tc, 3),
               round(flops / tc / 1e9, 2), round(tc / t, 3), f"{err:.3e}", f"{errc:.3e}",
               f"{args.sample}x{args.sample}"]
        rows.append(row)
        print(",".join(str(x) for x in row), flush=True)
        del out, cb
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w", newline="") as f:
        f.write("# tools/config_sweep.py on one B200: device-resident inputs, CUDA events, "
                f"{args.reps} timed calls after 2 warm-ups; max_rel_err vs the reference exact "
                "oracle of alpha*A*B + beta*C on a sampled block\n")
        w = csv.writer(f)
        w.writerow(HEADER)
        w.writerows(rows)


if __name__ == "__main__":
    main()
