"""Column-split variants at C3 (diag build: OZMM_COLS_TWO_PASS, OZMM_PANEL_MB): time of one
ozmm_split_offset of B (16384 x 16384, columns, k = 8, offset planes) per
variant, algorithmic GB/s (8 n p read + k p lds written), and a bitwise check
that every variant writes the same planes, shifts and column sums as the
first variant (the two-pass path).  Also times the row split of A for reference.
    python tools/cols_probe.py [--n 16384] [--p 16384] [--k 8]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--p", type=int, default=16384)
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--variants", default="default:OZMM_NONE=0")
    ap.add_argument("--row-variants", default="default:OZMM_NONE=0",
                    help="env settings for the row split timing, e.g. cta256:OZMM_ROW_CTA=256")
    a = ap.parse_args()
    from paper_2409_13313_b200 import ozmm
    n, p, k = a.n, a.p, a.k
    lds = (n + 15) // 16 * 16
    g = torch.Generator(device="cuda").manual_seed(1)
    B = ((torch.rand((n, p), device="cuda", dtype=torch.float64, generator=g) - 0.5) *
         torch.exp(0.5 * torch.randn((n, p), device="cuda", dtype=torch.float64, generator=g)))
    h = ozmm.Handle(0)
    st = torch.cuda.current_stream()
    h.set_stream(st.cuda_stream)
    res = {}
    first = None
    for spec in a.variants.split(","):
        v, kv = spec.split(":")
        for key in ("OZMM_COLS_TWO_PASS", "OZMM_PANEL_MB", "OZMM_PANEL_LAG"):
            os.environ.pop(key, None)
        for assign in kv.split("+"):
            key, val = assign.split("=")
            os.environ[key] = val
        first = first or v
        S = torch.zeros((k, p, lds), dtype=torch.int8, device="cuda")
        sh = torch.zeros(p, dtype=torch.float64, device="cuda")
        ls = torch.zeros((k, p), dtype=torch.int32, device="cuda")

        def call():
            ls.zero_()
            h.check(ozmm.lib.ozmm_split_offset(h.h, b"R", b"N", p, n, B.data_ptr(), p, k, 0,
                                               S.data_ptr(), lds, sh.data_ptr(), ls.data_ptr(), p, 1))
        call()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(a.reps):
            e0.record(st)
            call()
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = sorted(ts)[len(ts) // 2]
        gbs = (8.0 * n * p + k * p * lds) / (t * 1e-3) / 1e9
        res[v] = (S.clone(), sh.clone(), ls.clone())
        same = "" if v == first else (
            f" same as {first}" if all(torch.equal(x, y) for x, y in zip(res[first], res[v]))
            else f" DIFFERS from {first}")
        print(f"{v}: {t:.3f} ms (median of {a.reps}, incl. a {4 * k * p / 1e6:.1f} MB lsum memset) "
              f"{gbs:.0f} GB/s algorithmic{same}", flush=True)
    for key in ("OZMM_COLS_TWO_PASS", "OZMM_PANEL_MB", "OZMM_PANEL_LAG"):
        os.environ.pop(key, None)
    # row split of A (same shape), per row variant
    if p < n:
        return
    for spec in a.row_variants.split(","):
        v, kv = spec.split(":")
        for assign in kv.split("+"):
            key, val = assign.split("=")
            os.environ[key] = val
        S = torch.zeros((k, n, lds), dtype=torch.int8, device="cuda")
        sh = torch.zeros(n, dtype=torch.float64, device="cuda")
        ls = torch.zeros((k, n), dtype=torch.int32, device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(a.reps):
            e0.record(st)
            ls.zero_()
            h.check(ozmm.lib.ozmm_split_offset(h.h, b"L", b"N", min(n, p), n, B.data_ptr(), p, k, 0,
                                               S.data_ptr(), lds, sh.data_ptr(), ls.data_ptr(), n, 1))
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = sorted(ts)[len(ts) // 2]
        print(f"row split (A) {v}: {t:.3f} ms {(8.0 * n * p + k * n * lds) / (t * 1e-3) / 1e9:.0f} GB/s")
        for assign in kv.split("+"):
            os.environ.pop(assign.split("=")[0], None)


if __name__ == "__main__":
    main()
