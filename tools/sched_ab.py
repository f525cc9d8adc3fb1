#!/usr/bin/env python
"""A/B of GEMM schedules (K2+K3 only, pre-split slices) on one B200.

    python tools/sched_ab.py --cases 8192:9,16384:12 --variants greedy,dp --rounds 3

Each variant is a set of environment overrides read by the launcher per call
(OZMM_SCHED, OZMM_SCHED_BATCH, OZMM_SCHED_FILL).  Variants are interleaved round
by round so clock/power drift hits all of them alike; the median per-call time
of each is reported (CUDA events, 3 calls per sample after a warm-up).
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

VARIANTS = {
    "greedy": {"OZMM_SCHED": "greedy"},
    "dp": {},
    "dp_b100": {"OZMM_SCHED_BATCH": "100"},
    "dp_b300": {"OZMM_SCHED_BATCH": "300"},
    "dp_f075": {"OZMM_SCHED_FILL": "0.75"},
    "dp_f125": {"OZMM_SCHED_FILL": "1.25"},
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="8192:9,8192:12,8192:13,16384:8,16384:12,16384:14")
    ap.add_argument("--variants", default="greedy,dp")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--n-inner", type=int, default=0, help="inner dimension (default = n)")
    args = ap.parse_args()
    import torch
    from paper_2409_13313_b200 import ozmm
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream(dev)
    for case in args.cases.split(","):
        parts = [int(x) for x in case.split(":")]
        n, k = parts[0], parts[1]
        inner = parts[2] if len(parts) > 2 else n
        A = torch.tensor(ozmm.gen_phi_matrix(n, inner, 1.0, 1), device=dev)
        B = torch.tensor(ozmm.gen_phi_matrix(inner, n, 1.0, 2), device=dev)
        sa = ozmm.split_rn_const_shift(A, k, "L")
        sb = ozmm.split_rn_const_shift(B, k, "R")
        del A, B
        C = torch.zeros((n, n), dtype=torch.float64, device=dev)
        times = {v: [] for v in args.variants.split(",")}
        ops = k * (k + 1) / 2 * 2.0 * n * inner * n
        for _ in range(args.rounds):
            for v in times:
                saved = {kk: os.environ.get(kk) for kk in ("OZMM_SCHED", "OZMM_SCHED_BATCH",
                                                           "OZMM_SCHED_FILL")}
                for kk in saved:
                    os.environ.pop(kk, None)
                os.environ.update(VARIANTS[v])
                ozmm.gemm_slices(sa, sb, 1.0, 0.0, C)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                for _ in range(3):
                    ozmm.gemm_slices(sa, sb, 1.0, 0.0, C)
                e1.record(st)
                torch.cuda.synchronize()
                times[v].append(e0.elapsed_time(e1) / 3)
                for kk, val in saved.items():
                    if val is None:
                        os.environ.pop(kk, None)
                    else:
                        os.environ[kk] = val
        line = [f"n={n} inner={inner} k={k}"]
        for v, ts in times.items():
            t = statistics.median(ts)
            line.append(f"{v}: {t:.3f} ms {ops / t / 1e9:.0f} TOPS")
        print(" | ".join(line), flush=True)
        del sa, sb, C
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
