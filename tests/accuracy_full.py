#!/usr/bin/env python
"""FULL-matrix accuracy sweep of the B200 ozIMMU_H path (paper Fig. 4 shape,
SURVEY.md 8f rank 1; the reference's run_sweep, proj/src/harness.cpp:44-105).

For each (n, phi, seed): A = gen_phi_matrix(n, n, phi, counter_hash(seed, 1)),
B = gen_phi_matrix(n, n, phi, counter_hash(seed, 2)) as the reference harness
generates them (harness.cpp:19-24).  The accuracy reference is a
double-double GEMM on the GPU over EVERY entry (tests/ddref/dd_gemm.cu, Dot2),
instead of the reference's exact_gemm_oracle (oracle.cpp:276), which needs
hours on the CPU at n = 8192.  Before any number is reported the dd reference
is pinned: on a seeded sample of entries its rounded value hi must equal the
reference's correctly rounded exact oracle (the reference build itself when
present, else the C port); the count of differing entries is written to the CSV
header (0 expected).

max_rel_err follows oracle.cpp:321-335 (|t - r| / |r|, or |t| / max|r| where
r = 0), with r = hi + lo evaluated in double-double.  Methods: "ozIMMU_H"
(GPU, device path) for every k, and "cuBLAS_DGEMM" (native FP64 on the same
GPU) as the comparator.  Same CSV schema as the reference sweep
(harness.cpp:40-42); t_* columns are the GPU phase timings (CUDA events).

    python tests/accuracy_full.py --n 8192 --k 6-14 --phi 0.5,1,2,4 \
        --out profiles/r2/accuracy_full_n8192.csv

Test infrastructure: imports the oracle (checker) and the dd reference.
"""
from __future__ import annotations

import argparse
import csv
import ctypes
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

DD_DIR = os.path.join(ROOT, "tests", "ddref")
DD_SRC = os.path.join(DD_DIR, "dd_gemm.cu")
DD_SO = os.path.join(DD_DIR, "libddref.so")

from tests.accuracy_sweep import HEADER, kprime_max, parse_list  # noqa: E402


def build_dd(force: bool = False) -> str:
    """nvcc the dd reference (sm_100a, no FMA contraction)."""
    if not force and os.path.exists(DD_SO) and os.path.getmtime(DD_SO) >= os.path.getmtime(DD_SRC):
        return DD_SO
    nvcc = "/usr/local/cuda/bin/nvcc" if os.path.exists("/usr/local/cuda/bin/nvcc") else "nvcc"
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "--fmad=false",
           "-shared", "-Xcompiler", "-fPIC", "-o", DD_SO, DD_SRC]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("dd reference build failed:\n" + res.stdout + res.stderr)
    return DD_SO


_dd = None


def dd_gemm(dA, dB):
    """(hi, lo) of A B on the GPU, double-double (Dot2 per entry)."""
    import torch
    global _dd
    if _dd is None:
        _dd = ctypes.CDLL(build_dd())
        _dd.dd_gemm.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int64] * 3 + [ctypes.c_void_p]
        _dd.dd_gemm.restype = ctypes.c_int
    m, n = dA.shape
    p = dB.shape[1]
    hi = torch.empty((m, p), dtype=torch.float64, device=dA.device)
    lo = torch.empty_like(hi)
    rc = _dd.dd_gemm(dA.data_ptr(), dB.data_ptr(), hi.data_ptr(), lo.data_ptr(), m, n, p,
                     torch.cuda.current_stream(dA.device).cuda_stream)
    if rc != 0:
        raise RuntimeError(f"dd_gemm failed ({rc})")
    return hi, lo


def max_rel_err_dd(t, hi, lo) -> float:
    """oracle.cpp:321-335 with the reference r = hi + lo (double-double):
    t - r = TwoSum(t, -hi) - lo, so the difference is resolved below one ulp."""
    import torch
    s = t - hi
    bb = s - t
    e = (t - (s - bb)) + (-hi - bb)  # TwoSum(t, -hi) = s + e exactly
    diff = (s + (e - lo)).abs()
    r = (hi + lo).abs()
    rmax = r.max()
    rel = torch.where(r != 0, diff / torch.where(r != 0, r, torch.ones_like(r)), t.abs() / rmax)
    return float(rel.max())


def pin_dd(chk, A, B, hi, lo, sample: int, rng) -> dict:
    """dd hi vs the reference's exact oracle on a seeded sample of entries."""
    n_rows, n_cols = A.shape[0], B.shape[1]
    I = np.sort(rng.choice(n_rows, min(sample, n_rows), replace=False))
    J = np.sort(rng.choice(n_cols, min(sample, n_cols), replace=False))
    exact = chk.exact_gemm(np.ascontiguousarray(A[I, :]), np.ascontiguousarray(B[:, J]))
    h = hi.cpu().numpy()[np.ix_(I, J)]
    lo_s = lo.cpu().numpy()[np.ix_(I, J)]
    # dd value rounded to double: hi unless lo carries it past a rounding boundary
    rounded = h + lo_s
    diff = int((rounded.view(np.uint64) != exact.view(np.uint64)).sum())
    with np.errstate(divide="ignore", invalid="ignore"):
        rel = np.where(exact != 0, np.abs(rounded - exact) / np.abs(exact), 0.0)
    return {"entries": int(exact.size), "differ": diff, "max_rel": float(rel.max())}


def run(ns, ks, phis, seeds, pin_sample, out_path, verbose=True):
    import torch

    from oracle import oracle
    from paper_2409_13313_b200 import ozmm

    chk = oracle.best()
    rows, pins = [], []
    rng = np.random.default_rng(2409)
    for n in ns:
        beta = ozmm.compute_beta(n)
        for phi in phis:
            for seed in seeds:
                A = ozmm.gen_phi_matrix(n, n, phi, ozmm.counter_hash(seed, 1))
                B = ozmm.gen_phi_matrix(n, n, phi, ozmm.counter_hash(seed, 2))
                dA = torch.tensor(A, device="cuda")
                dB = torch.tensor(B, device="cuda")
                t0 = time.perf_counter()
                hi, lo = dd_gemm(dA, dB)
                torch.cuda.synchronize()
                t_dd = time.perf_counter() - t0
                pin = pin_dd(chk, A, B, hi, lo, pin_sample, rng)
                pin.update({"n": n, "phi": phi, "seed": seed, "dd_s": round(t_dd, 3)})
                pins.append(pin)
                cub = torch.matmul(dA, dB)
                e_cub = max_rel_err_dd(cub, hi, lo)
                del cub
                rows.append([n, phi, 0, "cuBLAS_DGEMM", seed, e_cub, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0])
                for k in ks:
                    res = ozmm.ozaki_mm(dA, dB, ozmm.config_for("ozIMMU_H", k))
                    e = max_rel_err_dd(res.d, hi, lo)
                    t = res.timings
                    rows.append([n, phi, k, "ozIMMU_H", seed, e, res.counts.int8_gemms,
                                 res.counts.fp64_flushes, res.counts.r, res.counts.w,
                                 kprime_max(n, beta), t.split_a, t.split_b, t.int_gemm,
                                 t.accum_fp64, t.copy])
                    if verbose:
                        print(f"n={n} phi={phi} seed={seed} k={k:2d}: ozIMMU_H {e:.3e}  "
                              f"cuBLAS {e_cub:.3e}  gemm {t.int_gemm * 1e3:.1f} ms", flush=True)
                    del res
                if verbose:
                    print(f"n={n} phi={phi}: dd reference {t_dd:.2f} s, pinned vs exact oracle on "
                          f"{pin['entries']} entries: {pin['differ']} differ "
                          f"(max rel {pin['max_rel']:.1e})", flush=True)
                del dA, dB, hi, lo
                torch.cuda.empty_cache()
    if out_path:
        os.makedirs(os.path.dirname(os.path.abspath(out_path)), exist_ok=True)
        with open(out_path, "w", newline="") as f:
            f.write("# max_rel_err over EVERY entry of the n x n product (oracle.cpp:321-335) "
                    "against a GPU double-double reference (tests/ddref/dd_gemm.cu, Dot2)\n")
            for pn in pins:
                f.write(f"# dd pin n={pn['n']} phi={pn['phi']} seed={pn['seed']}: "
                        f"{pn['differ']} of {pn['entries']} sampled entries differ from the "
                        f"reference exact_gemm_oracle ({chk.kind} build) after rounding; "
                        f"max rel {pn['max_rel']:.2e}; dd GEMM {pn['dd_s']} s\n")
            w = csv.writer(f)
            w.writerow(HEADER)
            for r in rows:
                w.writerow([f"{x:.17g}" if isinstance(x, float) else x for x in r])
    return rows, pins


def summary(rows) -> list[str]:
    """Per (n, phi): the smallest k whose ozIMMU_H error is at or below cuBLAS DGEMM's."""
    out = []
    keys = sorted({(r[0], r[1]) for r in rows})
    for n, phi in keys:
        cub = [r[5] for r in rows if (r[0], r[1], r[3]) == (n, phi, "cuBLAS_DGEMM")]
        oz = sorted((r[2], r[5]) for r in rows if (r[0], r[1], r[3]) == (n, phi, "ozIMMU_H"))
        kmin = next((k for k, e in oz if cub and e <= max(cub)), None)
        out.append(f"n={n} phi={phi}: cuBLAS {max(cub):.2e}; ozIMMU_H " +
                   " ".join(f"k{k}={e:.1e}" for k, e in oz) + f"; first k <= DGEMM: {kmin}")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", default="8192")
    ap.add_argument("--k", default="6-14")
    ap.add_argument("--phi", default="0.5,1,2,4")
    ap.add_argument("--seeds", default="0")
    ap.add_argument("--pin-sample", type=int, default=48)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    t0 = time.time()
    rows, _ = run(parse_list(a.n, int), parse_list(a.k, int), parse_list(a.phi, float),
                  parse_list(a.seeds, int), a.pin_sample, a.out)
    for line in summary(rows):
        print(line)
    print(f"done in {time.time() - t0:.1f} s")


if __name__ == "__main__":
    main()
