"""Generate the golden fixtures under tests/golden from the REFERENCE itself.

Run in the build container (where /root/reference exists):

    make -C oracle && python tests/golden/make_golden.py

Every array in ``golden.npz`` comes out of ``oracle/_ref/libozmm_ref.so``: the
unmodified reference sources (/root/reference/proj/src) compiled against the
in-repo Eigen shim.  The fixtures pin both CPU checkers (tests/test_oracle.py)
and the CUDA library (tests/test_gpu_*.py) without needing /root/reference at
run time -- it does not exist on the GPU box.

Cases cover: the C1-style random phi matrices (small), the SPEC known answers
(split of 351 at beta=3), zero rows/columns, power-of-two
rows, rows that trigger the rounding "bump" (split.cpp:126-129), tiny
(near-underflow / subnormal) and huge (2^900) rows, forced r (chunked
groups, scheme.cpp:91), forced beta, n=1 and ragged shapes.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import RefLib  # noqa: E402


def special_matrix(ref: RefLib, rows: int, cols: int, seed: int) -> np.ndarray:
    """phi=1 matrix with hand-made edge rows/columns mixed in."""
    a = ref.gen_phi_matrix(rows, cols, 1.0, seed)
    if rows > 6 and cols > 6:
        a[0, :] = 0.0                                   # zero row
        a[1, :] = np.ldexp(1.0, np.arange(cols) % 5 - 3)  # power-of-two row
        a[1, ::3] *= -1
        a[2, :] *= 1e-300                               # tiny but normal
        a[2, 0] = 5e-324                                # subnormal entry
        a[3, :] *= 2.0 ** 400                           # huge (products stay finite)
        # bump row: max = (2 - 2^-8) * 2^3 rounds past 2^beta grid units
        a[4, :] = 0.001 * a[4, :]
        a[4, 2] = (2.0 - 2.0 ** -8) * 8.0
        a[5, :] = -0.0                                  # negative zeros
        a[:, 0] = a[:, 0] * 0.0                         # zero column (signs kept)
    return a


CASES = [
    # name, m, n, p, phi, k, alpha, beta, force_beta, force_r, special
    ("phi05_k8", 24, 300, 20, 0.5, 8, 1.0, 0.0, 0, 0, False),
    ("phi1_k9_ab", 17, 513, 33, 1.0, 9, 1.5, 0.5, 0, 0, False),
    ("phi4_k14_r3", 16, 257, 16, 4.0, 14, -2.0, 0.25, 0, 3, False),
    ("phi2_k8_r2", 9, 1000, 11, 2.0, 8, 1.0, 1.0, 0, 2, False),
    ("special_k8", 12, 64, 10, 1.0, 8, 1.0, -1.0, 0, 0, True),
    ("special_k12_r5", 12, 96, 12, 1.0, 12, 0.75, 0.5, 0, 5, True),
    ("beta3_k5", 8, 40, 8, 0.5, 5, 1.0, 0.0, 3, 0, False),
    ("n1", 5, 1, 7, 0.5, 4, 1.0, 0.0, 0, 0, False),
    ("m1p1", 1, 200, 1, 2.0, 8, 1.0, 0.0, 0, 0, False),
]


def main() -> None:
    ref = RefLib()
    out: dict[str, np.ndarray] = {}
    for (name, m, n, p, phi, k, alpha, beta, fb, fr, special) in CASES:
        seed = sum(map(ord, name))
        if special:
            a = special_matrix(ref, m, n, seed)
            b = special_matrix(ref, p, n, seed + 1).T.copy()   # special columns of B
        else:
            a = ref.gen_phi_matrix(m, n, phi, ref.counter_hash(seed, 1))
            b = ref.gen_phi_matrix(n, p, phi, ref.counter_hash(seed, 2))
        c = ref.gen_phi_matrix(m, p, phi, ref.counter_hash(seed, 3))
        d, info = ref.gemm(alpha, a, b, beta, c, k=k, force_beta=fb, force_r=fr,
                           with_info=True)
        sa = ref.split(a, k, "left", force_beta=fb)
        sb = ref.split(b, k, "right", force_beta=fb)
        ch = ref.groupwise_chunks(a, b, k, force_beta=fb, force_r=fr)
        pre = f"{name}/"
        out[pre + "params"] = np.array([m, n, p, k, fb, fr], np.int64)
        out[pre + "scalars"] = np.array([phi, alpha, beta], np.float64)
        out[pre + "A"], out[pre + "B"], out[pre + "C"] = a, b, c
        out[pre + "out"] = d
        out[pre + "counts"] = np.array([info["int8_gemms"], info["fp64_flushes"], info["r"],
                                        info["w"]], np.int64)
        out[pre + "sliceA"], out[pre + "shiftA"] = sa.slices, sa.shift
        out[pre + "sliceB"], out[pre + "shiftB"] = sb.slices, sb.shift
        out[pre + "beta_underflow"] = np.array([sa.beta, int(sa.underflow), int(sb.underflow)])
        out[pre + "chunk_acc"] = ch.acc
        out[pre + "chunk_gs"] = np.stack([ch.g, ch.s0, ch.s1])
    # comparison methods (config_for presets, scheme.cpp:137-159) on three cases
    for name in ("phi1_k9_ab", "special_k8", "phi2_k8_r2"):
        pre = f"{name}/"
        m, n, p, k, fb, fr = (int(v) for v in out[pre + "params"])
        phi, alpha, beta = (float(v) for v in out[pre + "scalars"])
        a, b, c = out[pre + "A"], out[pre + "B"], out[pre + "C"]
        for meth in ("ozIMMU", "ozIMMU_RN", "ozIMMU_EF"):
            d, info = ref.gemm(alpha, a, b, beta, c, k=k, method=meth, force_beta=fb,
                               force_r=fr, with_info=True)
            out[pre + meth + "/out"] = d
            out[pre + meth + "/counts"] = np.array(
                [info["int8_gemms"], info["fp64_flushes"], info["r"], info["w"]], np.int64)
        for strat in ("bitmask", "rn_per_slice"):
            sa, ua = ref.split_any(a, k, strat, "left", force_beta=fb)
            sb, ub = ref.split_any(b, k, strat, "right", force_beta=fb)
            out[pre + strat + "/sliceA"], out[pre + strat + "/outA"] = sa, ua
            out[pre + strat + "/sliceB"], out[pre + strat + "/outB"] = sb, ub
    # SPEC known answer: 351 = (101011111)_2, beta forced to 3
    s = ref.split(np.array([[351.0]]), 3, "left", force_beta=3, residual=True)
    out["spec351/slices"] = s.slices.ravel()
    out["spec351/shift"] = s.shift
    sl, sh = ref.split_any(np.array([[351.0]]), 3, "bitmask", "left", force_beta=3)
    out["spec351/bitmask_slices"] = sl.ravel()  # [5, 3, 7]
    sl, un = ref.split_any(np.array([[351.0]]), 3, "rn_per_slice", "left", force_beta=3)
    out["spec351/rnps_slices"] = sl.ravel()
    out["spec351/rnps_units"] = un.ravel()
    # closed forms (AC4)
    ns = np.array([1, 2, 3, 1000, 1024, 1025, 8192, 16384, 65536, 2 ** 17, 2 ** 17 + 1,
                   2 ** 18, 2 ** 29], np.int64)
    out["closed/n"] = ns
    out["closed/beta"] = np.array([ref.compute_beta(int(x)) for x in ns], np.int64)
    out["closed/r"] = np.array([ref.compute_r(int(x), ref.compute_beta(int(x))) for x in ns],
                               np.int64)
    kr = [(k, r) for k in range(1, 21) for r in (1, 2, 3, 5, 8, 16, 128)]
    out["closed/kr"] = np.array(kr, np.int64)
    out["closed/w"] = np.array([ref.op_counts_with_r(k, r)["w"] for k, r in kr], np.int64)
    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
