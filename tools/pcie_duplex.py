#!/usr/bin/env python
"""PCIe H2D and D2H alone and at the same time (pinned host buffers, 1 GB each).
    python tools/pcie_duplex.py [--gb 1]"""
import argparse
import json

import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gb", type=float, default=1.0)
    args = ap.parse_args()
    n = int(args.gb * 2**30) // 8
    h_in = torch.ones(n, dtype=torch.float64).pin_memory()
    h_out = torch.empty(n, dtype=torch.float64).pin_memory()
    d_in = torch.empty(n, dtype=torch.float64, device="cuda")
    d_out = torch.ones(n, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def run(h2d, d2h):
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e[0].record(s1)
        e[2].record(s2)
        if h2d:
            with torch.cuda.stream(s1):
                d_in.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h_out.copy_(d_out, non_blocking=True)
        e[1].record(s1)
        e[3].record(s2)
        torch.cuda.synchronize()
        return e[0].elapsed_time(e[1]), e[2].elapsed_time(e[3])
    gb = n * 8 / 1e9
    for name, a, b in (("h2d", 1, 0), ("d2h", 0, 1), ("both", 1, 1)) * 2:
        t1, t2 = run(a, b)
        out = {"case": name}
        if a:
            out["h2d_gbs"] = round(gb / t1 * 1e3, 1)
        if b:
            out["d2h_gbs"] = round(gb / t2 * 1e3, 1)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
