#!/usr/bin/env python
"""Per-rank step time of the 2-D grid partition, measured on ONE B200.

    python tools/rank_timing.py [--m 16384 --n 16384 --p 16384 --k 8] [--worlds 1,2,4,8]

The gpurun pool exposes one GPU, so the N-GPU strong-scaling run cannot be
executed here.  This tool runs the exact per-rank work of grid2d.Grid2DGemm
for rank 0 of a world-W grid (its own row/column slicing, the three strip
launches G1/G2/G3 on the gathered panel views) with the NCCL all-gather
replaced by an emulated one: the peer parts are written into the panel by a
device copy on a high-priority side stream, optionally followed by a
``torch.cuda._sleep`` that models the NVLink transfer time of the bytes the
rank would receive (--nvlink-gbs, default 700 GB/s per direction).  The
strip GEMMs, their stream overlap and the gather->GEMM dependencies are the
real ones; only the wire is modelled.

Printed per W: rank step time (CUDA events, median of --reps after warm-up),
the 1-GPU step time of the whole problem, and the implied strong-scaling
efficiency T1 / (W * T_rank).  All ranks of a grid do the same amount of
work, so rank 0 stands for the max over ranks up to NVLink/NCCL jitter.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=16384)
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--p", type=int, default=16384)
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--phi", type=float, default=0.5)
    ap.add_argument("--worlds", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--nvlink-gbs", type=float, default=700.0)
    ap.add_argument("--clock-ghz", type=float, default=1.4, help="for the _sleep cycle count")
    ap.add_argument("--no-side", action="store_true", help="G1 on the main stream (old order)")
    ap.add_argument("--native", action="store_true",
                    help="also time the native C-ABI grid entry (ozmm_dgemm_2d) with the same "
                         "emulated all-gather as a hook")
    ap.add_argument("--a-panels", type=int, default=0,
                    help="--e2e: A row panels per rank (0: bench.py's rule, ms/8 rows, >= 512)")
    ap.add_argument("--e2e", action="store_true",
                    help="also time the rank's end-to-end step (pinned H2D of its shard, step, "
                         "D2H of its C block): C rows streamed back per strip (c_host) against "
                         "one copy after the step")
    args = ap.parse_args()

    from paper_2409_13313_b200 import ozmm
    from paper_2409_13313_b200.grid2d import Backend, Grid2DGemm, make_layout

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    m, n, p, k, phi = args.m, args.n, args.p, args.k, args.phi
    seeds = [ozmm.counter_hash(0, i) for i in (1, 2, 3)]
    comm = torch.cuda.Stream(dev, priority=-1)
    out = []

    def timed(fn, reps):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        return ts[len(ts) // 2]

    t1 = None
    for world in [int(w) for w in args.worlds.split(",")]:
        L = make_layout(m, n, p, world, 0)
        wire_ns = [0.0]

        class Work:
            def __init__(self, ev):
                self.ev = ev

            def wait(self):
                torch.cuda.current_stream(dev).wait_event(self.ev)

        def all_gather(out_t, inp, group):
            nr = len(group)
            comm.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(comm):
                parts = out_t.view(nr, *inp.shape)
                for i in range(nr):
                    parts[i].copy_(inp)
                recv = inp.numel() * inp.element_size() * (nr - 1)
                ns = recv / (args.nvlink_gbs * 1e9) * 1e9
                wire_ns[0] += ns
                if ns > 0:
                    torch.cuda._sleep(int(ns * args.clock_ghz))
                ev = torch.cuda.Event()
                ev.record(comm)
            return Work(ev)

        be = Backend(0)
        if args.no_side:
            be.side_stream = None  # noqa: attribute shadow -> grid2d falls back to one stream
        G = Grid2DGemm(m, n, p, k, world=world, rank=0, backend=be,
                       group_factory=lambda ranks: tuple(ranks), all_gather=all_gather)
        A = torch.from_numpy(ozmm.gen_phi_block(m, n, phi, seeds[0], L.a_row0, L.ms, 0, n)).to(dev)
        B = torch.from_numpy(ozmm.gen_phi_block(n, p, phi, seeds[1], 0, n, L.b_col0, L.ps)).to(dev)
        C = torch.zeros((L.mr, L.pcols), dtype=torch.float64, device=dev)
        if world == 1:
            # the single-process path bench.py times at N=1 (ozaki_gemm_ex, 4 launches)
            h = ozmm.Handle(0)
            h.set_stream(torch.cuda.current_stream(dev).cuda_stream)
            cfg = ozmm.config_for(ozmm.Method.ozIMMU_H, k)
            t = timed(lambda: ozmm.ozaki_gemm_ex(1.0, A, B, 0.0, C, cfg, handle=h, out=C), args.reps)
            t1 = t
        else:
            wire_ns[0] = 0.0
            t = timed(lambda: G.step(A, B, C, 1.0, 0.0), args.reps)
        native = None
        if args.native and world > 1:
            import ctypes
            from paper_2409_13313_b200.grid2d import NativeGrid2D
            cudart = ctypes.CDLL("libcudart.so.12")
            cudart.cudaMemcpyAsync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                               ctypes.c_int, ctypes.c_void_p]
            Lw = L

            def hook(ctx, group, send, recv, nbytes, stream):
                # this rank's part into every peer slot (stand-in for the peers' data),
                # then the modelled wire time of the bytes received, on `stream`
                nr = Lw.pc if group == 0 else Lw.pr
                idx = Lw.gc if group == 0 else Lw.gr
                for i in range(nr):
                    if i != idx:
                        cudart.cudaMemcpyAsync(recv + i * nbytes, send, nbytes, 3, stream)
                ns = nbytes * (nr - 1) / (args.nvlink_gbs * 1e9) * 1e9
                if ns > 0:
                    with torch.cuda.stream(torch.cuda.ExternalStream(stream)):
                        torch.cuda._sleep(int(ns * args.clock_ghz))
                return 0
            cb = ozmm.ALLGATHER_FN(hook)
            NG = NativeGrid2D(m, n, p, k, world=world, rank=0, hook=cb)
            native = timed(lambda: NG.step(A, B, C, 1.0, 0.0), args.reps)
            NG.close()
        e2e = {}
        if args.e2e and world > 1:
            hA, hB = A.cpu().pin_memory(), B.cpu().pin_memory()
            hC = torch.empty(tuple(C.shape), dtype=torch.float64).pin_memory()
            s_in = torch.cuda.Stream(dev)
            ev = {key: torch.cuda.Event() for key in "abc"}
            # B first, then A in row panels: B's split and gather, and the first
            # strip of each A panel, run while the rest of A is still crossing PCIe
            psz = max(256, L.ms // args.a_panels) if args.a_panels else max(512, L.ms // 8)
            a_pieces = [(lo, min(lo + psz, L.ms)) for lo in range(0, L.ms, psz)]
            a_ev = [torch.cuda.Event() for _ in a_pieces]
            ev["a"] = [(lo, hi, e) for (lo, hi), e in zip(a_pieces, a_ev)]

            ev1 = torch.cuda.Event()

            def e2e_call(mode):
                # after: A then B whole, one D2H after the step; streamed: C rows go
                # back per strip (c_host); panels: + B first, then A panel by panel
                with torch.cuda.stream(s_in):
                    if mode == "panels":
                        B.copy_(hB, non_blocking=True)
                        ev["b"].record(s_in)
                        for (lo, hi), e in zip(a_pieces, a_ev):
                            A[lo:hi].copy_(hA[lo:hi], non_blocking=True)
                            e.record(s_in)
                    else:
                        A.copy_(hA, non_blocking=True)
                        ev1.record(s_in)
                        B.copy_(hB, non_blocking=True)
                        ev["b"].record(s_in)
                    ev["c"].record(s_in)
                rd = dict(ev, a=ev["a"] if mode == "panels" else ev1)
                G.step(A, B, C, 1.0, 0.0, ready=rd, c_write_only=True,
                       c_host=None if mode == "after" else hC)
                if mode == "after":
                    hC.copy_(C, non_blocking=True)
            for mode in ("after", "streamed", "panels") * 2:
                e2e.setdefault(mode, []).append(round(timed(lambda: e2e_call(mode), args.reps), 3))
        row = {"world": world, "grid": f"{L.pr}x{L.pc}", "rank_ms": round(t, 3),
               "c_block": [L.mr, L.pcols],
               "modelled_wire_ms_per_step": round(wire_ns[0] / 1e6 / (args.reps + 3), 3)
               if world > 1 else 0.0}
        if native is not None:
            row["native_rank_ms"] = round(native, 3)
        if e2e:
            row["e2e_ms"] = e2e
        if t1:
            row["t1_ms"] = round(t1, 3)
            row["efficiency"] = round(t1 / (world * t), 4)
        out.append(row)
        print(json.dumps(row), flush=True)
        del G, A, B, C
        torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    main()
