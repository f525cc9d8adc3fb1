"""BASELINE.json's named configurations on the GPU, bit-exact against the
reference (oracle/_ref, the unmodified reference build; the C port pinned to it
where _ref is absent).

* C1  m=n=p=1024, phi=0.5, k=8: the WHOLE matrix, like the reference's own
      sweep, which compares full matrices (harness.cpp:44-105).
* C2  m=n=p=8192, k=6..14 x phi in {0.5, 1, 2}: a 64x64 block per run, rows and
      columns spread over every tile row / column (sub-block locality, SURVEY.md
      Appendix A.4: entry (i, j) depends only on row i of op(A), column j of
      op(B) and n).
* C3  m=n=p=16384, k=8, phi=0.5: the benchmarked shape and launch (bench.py
      checks a sample of its own timed output the same way).
* C4  m=p=8192, n=65536 (r = 2, w = 20 INT32 chunks).
* C5  m=n=p=16384, phi=4, k=12, transa/transb, alpha=1.5, beta=0.5.
Plus the kernel's tuning knobs (K-block pairs, A-ring depth), which must never
change a bit.

Inputs are the reference generator's phi matrices (generate.cpp:11-29) with
the bench's seeds: counter_hash(0, 1..3).
"""
import os

import numpy as np
import pytest

from tests.helpers import assert_bitwise

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def oz():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2409_13313_b200 import ozmm
    return ozmm


@pytest.fixture(scope="module")
def checker():
    from oracle import oracle
    if not os.path.exists(oracle.PORT_SO):
        oracle.build()
    return oracle.best()


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda")


def spread(total, count, rng, tile):
    """`count` sorted distinct indices in [0, total): one per stratum, so every
    tile row / column is hit when count >= total / tile; first and last included."""
    edges = np.linspace(0, total, count + 1).astype(np.int64)
    idx = np.array([rng.integers(lo, hi) for lo, hi in zip(edges[:-1], edges[1:])])
    idx[0], idx[-1] = 0, total - 1
    assert len(np.unique(idx)) == count
    if count * tile >= total:
        assert len(np.unique(idx // tile)) == -(-total // tile), "a tile row/column is unsampled"
    return idx


def check_block(checker, A, B, C, got, k, alpha, beta, rows, cols, ta=False, tb=False):
    """got[rows, cols] == the reference's ozaki_gemm_ex on A(I,:), B(:,J), C(I,J)."""
    Aop = A[:, rows].T if ta else A[rows, :]
    Bop = B[cols, :].T if tb else B[:, cols]
    want = checker.gemm(alpha, np.ascontiguousarray(Aop), np.ascontiguousarray(Bop), beta,
                        np.ascontiguousarray(C[np.ix_(rows, cols)]), k=k)
    assert_bitwise(got, want)


def test_c1_full_matrix(oz, checker):
    """C1: 1024^3, phi=0.5, k=8, every entry (device path and host entry)."""
    m = n = p = 1024
    A = oz.gen_phi_matrix(m, n, 0.5, oz.counter_hash(0, 1))
    B = oz.gen_phi_matrix(n, p, 0.5, oz.counter_hash(0, 2))
    C = oz.gen_phi_matrix(m, p, 0.5, oz.counter_hash(0, 3))
    cfg = oz.config_for("ozIMMU_H", 8)
    want, info = checker.gemm(1.0, A, B, 0.0, np.zeros((m, p)), k=8, with_info=True)
    res = oz.ozaki_gemm_ex(1.0, dev(A), dev(B), 0.0, torch.zeros((m, p), dtype=torch.float64,
                                                                  device="cuda"), cfg)
    assert_bitwise(res.d.cpu().numpy(), want, "C1 device path")
    assert (res.counts.int8_gemms, res.counts.fp64_flushes, res.counts.r, res.counts.w) == \
        (info["int8_gemms"], info["fp64_flushes"], info["r"], info["w"]) == (36, 8, 128, 8)
    assert_bitwise(oz.ozaki_gemm(1.0, A, B, 0.0, np.zeros((m, p)), cfg), want, "C1 host entry")
    # alpha / beta epilogue on the whole matrix too
    want2 = checker.gemm(1.5, A, B, 0.5, C, k=8)
    assert_bitwise(oz.ozaki_gemm(1.5, dev(A), dev(B), 0.5, dev(C), cfg).cpu().numpy(), want2,
                   "C1 alpha=1.5 beta=0.5")


@pytest.fixture(scope="module")
def c2_inputs(oz):
    cache = {}

    def get(phi):
        if phi not in cache:
            cache.clear()
            n = 8192
            A = oz.gen_phi_matrix(n, n, phi, oz.counter_hash(0, 1))
            B = oz.gen_phi_matrix(n, n, phi, oz.counter_hash(0, 2))
            cache[phi] = (A, B, dev(A), dev(B))
        return cache[phi]
    return get


@pytest.mark.slow
@pytest.mark.parametrize("phi", [0.5, 1.0, 2.0])
@pytest.mark.parametrize("k", list(range(6, 15)))
def test_c2_sweep_sampled(oz, checker, c2_inputs, phi, k):
    """C2: n=8192, every k of the paper's sweep at phi 0.5 / 1 / 2."""
    n = 8192
    A, B, dA, dB = c2_inputs(phi)
    out = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    res = oz.ozaki_gemm_ex(1.0, dA, dB, 0.0, out, oz.config_for("ozIMMU_H", k), out=out)
    rng = np.random.default_rng(1000 * k + int(4 * phi))
    rows, cols = spread(n, 64, rng, 256), spread(n, 64, rng, 128)
    got = out[torch.from_numpy(rows).cuda()][:, torch.from_numpy(cols).cuda()].cpu().numpy()
    check_block(checker, A, B, np.zeros((n, n)), got, k, 1.0, 0.0, rows, cols)
    assert res.counts.int8_gemms == k * (k + 1) // 2
    assert res.counts.r == 16 and res.counts.w == oz.op_counts_with_r(k, 16).w


@pytest.mark.slow
def test_c3_benchmarked_shape_sampled(oz, checker):
    """C3: the bench's exact launch (16384^3, k=8, phi=0.5, alpha=1, beta=0),
    128x128 entries covering every 256-row pair tile row and every 128-column tile."""
    n = 16384
    A = oz.gen_phi_block(n, n, 0.5, oz.counter_hash(0, 1))
    B = oz.gen_phi_block(n, n, 0.5, oz.counter_hash(0, 2))
    out = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    oz.ozaki_gemm_ex(1.0, dev(A), dev(B), 0.0, out, oz.config_for("ozIMMU_H", 8), out=out)
    rng = np.random.default_rng(3)
    rows, cols = spread(n, 128, rng, 256), spread(n, 128, rng, 128)
    got = out[torch.from_numpy(rows).cuda()][:, torch.from_numpy(cols).cuda()].cpu().numpy()
    del out
    check_block(checker, A, B, np.zeros((n, n)), got, 8, 1.0, 0.0, rows, cols)


@pytest.mark.slow
def test_c4_inner_split_sampled(oz, checker):
    """C4: m=p=8192, n=65536 -- r = 2, 20 INT32 chunks (the overflow-safe inner split)."""
    m, n, p = 8192, 65536, 8192
    A = oz.gen_phi_block(m, n, 0.5, oz.counter_hash(0, 1))
    B = oz.gen_phi_block(n, p, 0.5, oz.counter_hash(0, 2))
    out = torch.zeros((m, p), dtype=torch.float64, device="cuda")
    res = oz.ozaki_gemm_ex(1.0, dev(A), dev(B), 0.0, out, oz.config_for("ozIMMU_H", 8), out=out)
    assert (res.counts.r, res.counts.w, res.counts.fp64_flushes) == (2, 20, 20)
    rng = np.random.default_rng(4)
    rows, cols = spread(m, 64, rng, 256), spread(p, 64, rng, 128)
    got = out[torch.from_numpy(rows).cuda()][:, torch.from_numpy(cols).cuda()].cpu().numpy()
    del out
    check_block(checker, A, B, np.zeros((m, p)), got, 8, 1.0, 0.0, rows, cols)


@pytest.mark.slow
def test_c5_wide_range_transposed_sampled(oz, checker):
    """C5: 16384^3, phi=4, k=12, transa=transb='T', alpha=1.5, beta=0.5."""
    n = 16384
    A = oz.gen_phi_block(n, n, 4.0, oz.counter_hash(0, 1))    # stored n x m
    B = oz.gen_phi_block(n, n, 4.0, oz.counter_hash(0, 2))    # stored p x n
    C = oz.gen_phi_block(n, n, 4.0, oz.counter_hash(0, 3))
    out = dev(C)
    oz.ozaki_gemm_ex(1.5, dev(A), dev(B), 0.5, out, oz.config_for("ozIMMU_H", 12), out=out,
                     transa=True, transb=True)
    rng = np.random.default_rng(5)
    rows, cols = spread(n, 64, rng, 256), spread(n, 64, rng, 128)
    got = out[torch.from_numpy(rows).cuda()][:, torch.from_numpy(cols).cuda()].cpu().numpy()
    del out
    check_block(checker, A, B, C, got, 12, 1.5, 0.5, rows, cols, ta=True, tb=True)


@pytest.mark.parametrize("m,n,p,k,phi", [
    (512, 1000, 384, 8, 0.5),      # n_kb = 8 (even): K-pair passes possible
    (600, 1100, 520, 9, 1.0),      # n_kb = 9 (odd): K-pair falls back per pass
    (256, 4096, 300, 12, 4.0),     # multi-window schedule (> 8 B slices)
    (384, 2048, 256, 14, 2.0),
])
@pytest.mark.parametrize("kpair", [1, 2])
@pytest.mark.parametrize("stages", [3, 4, 5])
def test_tuning_knobs_bit_exact(oz, checker, m, n, p, k, phi, kpair, stages):
    """K-block pairs off/on x A-ring depths 3/4/5 (odd rings with K-pair included):
    tuning only, results identical to the reference."""
    A = oz.gen_phi_matrix(m, n, phi, 91)
    B = oz.gen_phi_matrix(n, p, phi, 92)
    C = oz.gen_phi_matrix(m, p, phi, 93)
    want = checker.gemm(1.5, A, B, 0.5, C, k=k)
    got = oz.ozaki_gemm(1.5, dev(A), dev(B), 0.5, dev(C), oz.config_for("ozIMMU_H", k),
                        kpair=kpair, stages=stages).cpu().numpy()
    assert_bitwise(got, want, f"kpair={kpair} stages={stages}")
    # the host entry's strips carry the whole problem's shape into the same choice
    got_h = oz.ozaki_gemm(1.5, A, B, 0.5, C, oz.config_for("ozIMMU_H", k), kpair=kpair,
                          stages=stages, host_panels=3)
    assert_bitwise(got_h, want, f"host kpair={kpair} stages={stages}")


@pytest.mark.parametrize("m,n,p,k,phi,ta,tb", [
    (200, 400, 77, 8, 0.5, False, False),     # columns <= 512: one CTA per strip
    (256, 1000, 130, 9, 1.0, False, False),   # one 1024-row CTA, ragged strip of 2 columns
    (300, 4111, 261, 12, 4.0, False, False),  # a 5-CTA cluster, rows past n zero-filled
    (130, 17000, 96, 8, 2.0, False, False),   # 1536 rows per CTA, 12-CTA cluster
    (97, 30000, 64, 7, 0.5, False, False),    # too long for one pass: the two-pass path
    (160, 2500, 200, 10, 1.0, True, True),    # op(A) columns (transa), op(B) rows (transb)
])
@pytest.mark.parametrize("col_split", [1, 2])
def test_one_pass_column_split_bit_exact(oz, checker, m, n, p, k, phi, ta, tb, col_split):
    """The one-pass column split (TMA-fed cluster kernel, op(B) read from HBM once)
    against the two-pass colmax + slice_cols path: both must give the reference's
    bits, through the device entry (offset and signed planes) and the host entry."""
    A = oz.gen_phi_matrix(n if ta else m, m if ta else n, phi, 111)
    B = oz.gen_phi_matrix(p if tb else n, n if tb else p, phi, 112)
    C = oz.gen_phi_matrix(m, p, phi, 113)
    Ar = np.ascontiguousarray(A.T) if ta else A
    Br = np.ascontiguousarray(B.T) if tb else B
    want = checker.gemm(1.5, Ar, Br, 0.5, C, k=k)
    cfg = oz.config_for("ozIMMU_H", k)
    for signed in (False, True):
        got = oz.ozaki_gemm(1.5, dev(A), dev(B), 0.5, dev(C), cfg, transa=ta, transb=tb,
                            col_split=col_split, signed_slices=signed).cpu().numpy()
        assert_bitwise(got, want, f"device col_split={col_split} signed={signed}")
    got_h = oz.ozaki_gemm(1.5, A, B, 0.5, C, cfg, transa=ta, transb=tb, col_split=col_split,
                          host_panels=3)
    assert_bitwise(got_h, want, f"host col_split={col_split}")


@pytest.mark.parametrize("k,phi,r,method", [(23, 4.0, 0, "ozIMMU_H"), (28, 2.0, 0, "ozIMMU_H"),
                                            (32, 4.0, 0, "ozIMMU_H"), (26, 1.0, 1, "ozIMMU_H"),
                                            (24, 2.0, 0, "ozIMMU_EF"), (25, 2.0, 0, "ozIMMU")])
def test_large_k_bit_exact(oz, checker, k, phi, r, method):
    """k beyond 22 (up to 32): 253..528 slice products, chunk counts up to 528 with
    r = 1; the device and host entries match the reference bit for bit."""
    m, n, p = 150, 700, 130
    A = oz.gen_phi_matrix(m, n, phi, 121)
    B = oz.gen_phi_matrix(n, p, phi, 122)
    C = oz.gen_phi_matrix(m, p, phi, 123)
    cfg = oz.config_for(method, k)
    if r:
        cfg.force_r = r
    want = checker.gemm(1.5, A, B, 0.5, C, k=k, method=method, force_r=r)
    got = oz.ozaki_gemm(1.5, dev(A), dev(B), 0.5, dev(C), cfg).cpu().numpy()
    assert_bitwise(got, want, f"device k={k}")
    assert_bitwise(oz.ozaki_gemm(1.5, A, B, 0.5, C, cfg), want, f"host k={k}")


@pytest.mark.parametrize("k,r,signed", [(8, 2, False), (9, 2, False), (12, 2, False), (8, 1, False),
                                        (7, 3, False), (14, 4, False), (12, 8, False), (14, 8, False),
                                        (10, 8, True), (8, 2, True)])
def test_parked_schedules_bit_exact(oz, checker, k, r, signed):
    """Schedules that batch chunks by shared A slices and park the ones ahead of
    their turn (schedule.hpp make_schedule_free; taken for small r and split
    groups): INT32 chunk sums (the dump, flushed from TMEM or from the park slot)
    and the final C equal the reference's, device and host entries, with the
    FP64 flushes in the reference's order (scheme.cpp:91-94)."""
    m, n, p = 300, 1500, 260
    A = oz.gen_phi_matrix(m, n, 1.0, 131)
    B = oz.gen_phi_matrix(n, p, 1.0, 132)
    C = oz.gen_phi_matrix(m, p, 1.0, 133)
    cfg = oz.config_for("ozIMMU_H", k)
    cfg.force_r = r
    cfg.overflow = oz.OverflowMode.Wrapping  # forced r: no Checked verification pass needed
    want = checker.gemm(1.5, A, B, 0.5, C, k=k, force_r=r)
    from oracle import oracle
    if os.path.exists(oracle.REF_SO):
        ch = oracle.RefLib().groupwise_chunks(A, B, k, force_r=r)
        dump = torch.zeros((ch.acc.shape[0], m, p), dtype=torch.int32, device="cuda")
        got = oz.ozaki_gemm(1.5, dev(A), dev(B), 0.5, dev(C), cfg, chunk_dump=dump,
                            signed_slices=signed)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(dump.cpu().numpy(), ch.acc)
        assert_bitwise(got.cpu().numpy(), want, f"device (dump) k={k} r={r}")
    got = oz.ozaki_gemm(1.5, dev(A), dev(B), 0.5, dev(C), cfg, signed_slices=signed).cpu().numpy()
    assert_bitwise(got, want, f"device k={k} r={r}")
    assert_bitwise(oz.ozaki_gemm(1.5, A, B, 0.5, C, cfg), want, f"host k={k} r={r}")


def test_parked_schedule_c4_shape(oz, checker):
    """n = 65536 (r = 2 without forcing, C4's inner dimension): the parked schedule
    on a 256 x 65536 x 384 problem, against the reference."""
    m, n, p, k = 256, 65536, 384, 8
    A = oz.gen_phi_matrix(m, n, 0.5, 141)
    B = oz.gen_phi_matrix(n, p, 0.5, 142)
    C = oz.gen_phi_matrix(m, p, 0.5, 143)
    want = checker.gemm(1.0, A, B, 0.0, C, k=k)
    cfg = oz.config_for("ozIMMU_H", k)
    got = oz.ozaki_gemm(1.0, dev(A), dev(B), 0.0, dev(C), cfg).cpu().numpy()
    assert_bitwise(got, want, "C4-shaped device")
    assert oz.ozaki_gemm_ex(1.0, dev(A), dev(B), 0.0, dev(C), cfg).counts.r == 2


@pytest.mark.parametrize("k,r", [(8, 2), (12, 8)])
def test_parked_schedules_quad_bit_exact(oz, checker, k, r):
    """The 4-CTA variant (cta_pair=3, A multicast) with parked schedules."""
    m, n, p = 512, 1200, 384
    A = oz.gen_phi_matrix(m, n, 2.0, 151)
    B = oz.gen_phi_matrix(n, p, 2.0, 152)
    C = oz.gen_phi_matrix(m, p, 2.0, 153)
    cfg = oz.config_for("ozIMMU_H", k)
    cfg.force_r = r
    cfg.overflow = oz.OverflowMode.Wrapping
    want = checker.gemm(-0.5, A, B, 1.5, C, k=k, force_r=r)
    got = oz.ozaki_gemm(-0.5, dev(A), dev(B), 1.5, dev(C), cfg, cta_pair=3).cpu().numpy()
    assert_bitwise(got, want, f"quad k={k} r={r}")


@pytest.mark.parametrize("k,r,panels", [(8, 2, 8), (12, 8, 6), (10, 3, 16)])
def test_parked_schedules_pipelined_host_strips(oz, checker, k, r, panels):
    """The host entry's pipelined strips (several strip GEMMs in flight on the
    handle's streams) with parked schedules: every strip's CTAs park into the
    per-SM-id scratch at its fixed stride; C equals the reference's for
    in-place and separate-output calls."""
    m, n, p = 1536, 2048, 1280
    A = oz.gen_phi_matrix(m, n, 1.0, 161)
    B = oz.gen_phi_matrix(n, p, 1.0, 162)
    C = oz.gen_phi_matrix(m, p, 1.0, 163)
    cfg = oz.config_for("ozIMMU_H", k)
    cfg.force_r = r
    cfg.overflow = oz.OverflowMode.Wrapping
    want = checker.gemm(1.5, A, B, 0.5, C, k=k, force_r=r)
    got = oz.ozaki_gemm(1.5, A, B, 0.5, C, cfg, host_panels=panels)
    assert_bitwise(got, want, f"host strips k={k} r={r} panels={panels}")
