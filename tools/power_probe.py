#!/usr/bin/env python
"""Data-dependence of the fused GEMM's speed under the 1 kW power cap.

    python tools/power_probe.py [--n 16384] [--k 8] [--secs 3]

Runs the fused ozIMMU_H GEMM (ozmm_gemm_slices, the K2+K3 kernel alone) back
to back on synthetic slice planes with different value distributions and
reports ms per call plus the median SM clock while it runs.  The INT8 work is
identical in every case; only the operand bits differ, so any difference is
the power draw of the tensor datapath / operand movement.  Used to decide
whether an operand-offset encoding (unsigned slices + exact rank-1
correction) could buy clock.  Not a bench number.
"""
from __future__ import annotations

import argparse
import os
import subprocess
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def clocks(stop, out):
    while not stop.is_set():
        try:
            r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw",
                                "--format=csv,noheader,nounits", "-i", "0"],
                               capture_output=True, text=True, timeout=5)
            a, b = r.stdout.strip().split(",")
            out.append((float(a), float(b)))
        except Exception:
            pass
        time.sleep(0.1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--secs", type=float, default=3.0)
    ap.add_argument("--phi", type=float, default=0.5)
    ap.add_argument("--real", action="store_true")
    args = ap.parse_args()
    from paper_2409_13313_b200 import ozmm
    dev = torch.device("cuda", 0)
    m = n = p = args.n
    k = args.k
    lds = ozmm.slice_ld(n)
    h = ozmm.Handle(0)
    h.set_stream(torch.cuda.current_stream(dev).cuda_stream)
    beta_bits = ozmm.compute_beta(n)
    mu = torch.ones(m, dtype=torch.float64, device=dev)
    nu = torch.ones(p, dtype=torch.float64, device=dev)
    C = torch.zeros((m, p), dtype=torch.float64, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(0)

    def rnd(lo, hi, rows):
        return torch.randint(lo, hi + 1, (k, rows, lds), dtype=torch.int8, device=dev, generator=g)

    cases = {
        "signed [-64,64]": lambda: (rnd(-64, 64, m), rnd(-64, 64, p)),
        "A unsigned [0,127], B signed": lambda: (rnd(0, 127, m), rnd(-64, 64, p)),
        "both [0,127]": lambda: (rnd(0, 127, m), rnd(0, 127, p)),
        "both [0,64]": lambda: (rnd(0, 64, m), rnd(0, 64, p)),
        "signed [-8,8]": lambda: (rnd(-8, 8, m), rnd(-8, 8, p)),
        "zeros": lambda: (torch.zeros((k, m, lds), dtype=torch.int8, device=dev),
                          torch.zeros((k, p, lds), dtype=torch.int8, device=dev)),
        "signed [-64,64] again": lambda: (rnd(-64, 64, m), rnd(-64, 64, p)),
    }
    if args.real:
        # real slices of the bench inputs (phi generator, GPU slicer), signed, and
        # biased to unsigned (slice 1 + (2^beta - 1), slices >= 2 + 2^(beta-1));
        # the biased ones run with the MMA's operand types flipped to u8 x u8
        # (OZMM_IDESC_XOR=0x480), which is what an offset encoding would execute
        A64 = torch.from_numpy(ozmm.gen_phi_block(m, n, args.phi, ozmm.counter_hash(0, 1))).to(dev)
        sa = ozmm.split_rn_const_shift(A64, k, "L")
        del A64
        B64 = torch.from_numpy(ozmm.gen_phi_block(n, p, args.phi, ozmm.counter_hash(0, 2))).to(dev)
        sb = ozmm.split_rn_const_shift(B64, k, "R")
        del B64
        torch.cuda.empty_cache()
        off = torch.tensor([2 ** beta_bits - 1] + [2 ** (beta_bits - 1)] * (k - 1), device=dev,
                           dtype=torch.int16).view(k, 1, 1)

        def biased(x):
            return (x.to(torch.int16) + off).to(torch.uint8).view(torch.int8)
        for s in range(k):
            a, b = sa.slices[s].float(), sb.slices[s].float()
            print(f"slice {s + 1}: A mean|x| {a.abs().mean():.1f} max {a.abs().max():.0f}; "
                  f"B mean|x| {b.abs().mean():.1f} max {b.abs().max():.0f}", flush=True)
        cases = {"real signed": lambda: (sa.slices, sb.slices),
                 "real biased u8 (xor)": lambda: (biased(sa.slices), biased(sb.slices)),
                 "real signed again": lambda: (sa.slices, sb.slices)}
    for name, make in cases.items():
        A, B = make()
        if "xor" in name:
            os.environ["OZMM_IDESC_XOR"] = "0x480"
        else:
            os.environ.pop("OZMM_IDESC_XOR", None)

        def call():
            h.check(ozmm.lib.ozmm_gemm_slices(h.h, m, n, p, k, beta_bits, 0, A.data_ptr(), lds,
                                              mu.data_ptr(), B.data_ptr(), lds, nu.data_ptr(),
                                              1.0, 0.0, C.data_ptr(), p, None))
        for _ in range(3):
            call()
        torch.cuda.synchronize()
        stop, smp = threading.Event(), []
        th = threading.Thread(target=clocks, args=(stop, smp))
        th.start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 0
        e0.record()
        t0 = time.time()
        while time.time() - t0 < args.secs:
            call()
            reps += 1
            if reps % 4 == 0:
                torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
        stop.set()
        th.join()
        ms = e0.elapsed_time(e1) / reps
        sm = sorted(c for c, _ in smp)
        pw = sorted(w for _, w in smp)
        med = lambda v: v[len(v) // 2] if v else None  # noqa: E731
        ops = k * (k + 1) / 2 * 2.0 * m * n * p
        print(f"{name:32s} {ms:8.2f} ms  {ops / ms / 1e9:7.0f} TOPS  sm {med(sm)} MHz  "
              f"power {med(pw)} W  ({reps} calls)", flush=True)
        del A, B
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
