#!/usr/bin/env python
"""Device-path timing of the fused GEMM over configs x kernel options (round-2 probe).

    python tools/probe_r2.py --cfg C2:9,C4,C3:8 --opt "pair:cta_pair=2" --opt "quad:cta_pair=3"

Inputs are (rand - 0.5) * exp(phi * randn) generated ON THE DEVICE with torch
(same distribution as the reference generator, different stream: timing only,
no parity claim).  Each (config, option) is warmed up once and timed over
--reps calls with CUDA events on the launching stream; prints ms, emulated
TFLOPS, INT8 TOPS (k(k+1)/2 * 2mnp / t) and the median SM clock sampled by
nvidia-smi during the timed calls.  Options alternate per rep round so clock
drift hits every option alike.
"""
from __future__ import annotations

import argparse
import os
import subprocess
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = {"C2": (8192, 8192, 8192, 8, 0.5, False, False, 1.0, 0.0),
          "C3": (16384, 16384, 16384, 8, 0.5, False, False, 1.0, 0.0),
          "C4": (8192, 65536, 8192, 8, 0.5, False, False, 1.0, 0.0),
          "C5": (16384, 16384, 16384, 12, 4.0, True, True, 1.5, 0.5)}


class Clock:
    def __init__(self):
        self.samples, self.stop = [], threading.Event()

    def run(self):
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.split()
                self.samples.append(float(out[0]))
            except Exception:
                pass
            self.stop.wait(0.2)


def parse_opt(s):
    """name:key=v,... -- ozaki_gemm_ex kwargs; env.NAME=v sets a (diag-build)
    environment variable for that option's calls only."""
    name, _, rest = s.partition(":")
    kw = {}
    for item in filter(None, rest.replace("+", ",").split(",")):
        k, v = item.split("=")
        kw[k] = v if k.startswith("env.") else int(v)
    return name, kw


def split_env(kw):
    env = {k[4:]: v for k, v in kw.items() if k.startswith("env.")}
    return env, {k: v for k, v in kw.items() if not k.startswith("env.")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="C2:8,C2:9")
    ap.add_argument("--opt", action="append", default=[])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--rounds", type=int, default=2)
    args = ap.parse_args()
    import torch
    from paper_2409_13313_b200 import ozmm as oz
    opts = [parse_opt(o) for o in (args.opt or ["default:"])]
    dev = torch.device("cuda:0")
    for spec in args.cfg.split(","):
        name, _, kk = spec.partition(":")
        m, n, p, k, phi, ta, tb, alpha, beta = SHAPES[name]
        if kk:
            k = int(kk)
        g = torch.Generator(device=dev).manual_seed(1)

        def gen(r, c):
            x = (torch.rand(r, c, device=dev, dtype=torch.float64, generator=g) - 0.5)
            return x * torch.exp(phi * torch.randn(r, c, device=dev, dtype=torch.float64, generator=g))
        A = gen(n, m) if ta else gen(m, n)
        B = gen(p, n) if tb else gen(n, p)
        C = gen(m, p)
        cfg = oz.config_for(oz.Method.ozIMMU_H, k)
        ops = k * (k + 1) / 2 * 2.0 * m * n * p
        res = {o[0]: [] for o in opts}
        clk = {o[0]: [] for o in opts}
        for _ in range(args.rounds):
            for oname, kw_all in opts:
                env, kw = split_env(kw_all)
                for key in list(os.environ):
                    if key.startswith("OZMM_") and key not in env:
                        os.environ.pop(key)
                os.environ.update(env)
                call = lambda: oz.ozaki_gemm_ex(alpha, A, B, beta, C, cfg, transa=ta, transb=tb,  # noqa: E731
                                                out=C, timings=False, **kw)
                call()
                torch.cuda.synchronize()
                st = torch.cuda.current_stream()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ck = Clock()
                th = threading.Thread(target=ck.run)
                th.start()
                e0.record(st)
                for _ in range(args.reps):
                    call()
                e1.record(st)
                torch.cuda.synchronize()
                ck.stop.set()
                th.join()
                res[oname].append(e0.elapsed_time(e1) / args.reps)
                clk[oname] += ck.samples
        for oname, _ in opts:
            ms = min(res[oname])
            cs = sorted(clk[oname])
            mhz = cs[len(cs) // 2] if cs else float("nan")
            print(f"{name} k={k} {oname:>12}: {ms:8.3f} ms  {2.0*m*n*p/ms/1e9:7.2f} TFLOPS  "
                  f"{ops/ms/1e9:7.1f} INT8 TOPS  {mhz:.0f} MHz  (all: {[round(x, 2) for x in res[oname]]})",
                  flush=True)
        del A, B, C
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
