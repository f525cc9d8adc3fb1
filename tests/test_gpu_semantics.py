"""Error semantics of the drop-in boundary on the GPU, against the reference's.

* Range errors (row max >= 2^921): the reference throws std::overflow_error
  from the split, before anything is written (split.cpp:124-125).  The device
  path raises by default too (sync_check), the deferred mode keeps the flag
  for Handle.sync_status(), and a pending flag is never blamed on a later call
  on the same handle (include/ozmm_b200.h, ozmm_sync_status).
* INT32 chunk overflow in OverflowMode::Checked: the reference's gemm_wide
  checks every running chunk sum (int_gemm.cpp:37-59) -- reachable only with
  force_r / force_beta.  The GPU verifies exactly and raises
  Int32OverflowError before C is written; in Wrapping mode both sides wrap mod
  2^32 and agree bit for bit.  (The reference's own Checked throw escapes an
  OpenMP parallel region and terminates the process, so Checked is compared
  with the C port, which returns the error, and Wrapping with the reference.)
"""
import ctypes
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
    return torch.tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")


def inputs(oz, m, n, p, seed, phi=1.0):
    return (oz.gen_phi_matrix(m, n, phi, seed), oz.gen_phi_matrix(n, p, phi, seed + 1),
            oz.gen_phi_matrix(m, p, phi, seed + 2))


def test_device_range_error_raises_and_next_host_call_is_clean(oz, checker):
    """The ADVICE scenario: a device-path range error on the shared default handle
    must raise there (C untouched) and must not leak into the next host call."""
    m, n, p = 300, 700, 200
    A, B, C = inputs(oz, m, n, p, 11)
    bad = A.copy()
    bad[123, 45] = 2.0 ** 950
    cfg = oz.config_for("ozIMMU_H", 8)
    c_dev = dev(C)
    with pytest.raises(OverflowError):
        oz.ozaki_gemm(1.0, dev(bad), dev(B), 0.5, c_dev, cfg, out=c_dev)
    assert_bitwise(c_dev.cpu().numpy(), C, "C after a device range error")
    # same (default) handle: host entry, then device entry, both bit-exact
    want = checker.gemm(1.0, A, B, 0.5, C, k=8)
    assert_bitwise(oz.ozaki_gemm(1.0, A, B, 0.5, C, cfg), want, "host call after the error")
    assert_bitwise(oz.ozaki_gemm(1.0, dev(A), dev(B), 0.5, dev(C), cfg).cpu().numpy(), want,
                   "device call after the error")
    assert oz.default_handle(0).sync_status() in (False, True)   # nothing pending: no raise


def test_deferred_range_error_stays_pending(oz, checker):
    """sync_check=False: stream-ordered, no raise; later calls on the handle report
    only their own status; Handle.sync_status() returns the pending error once."""
    m, n, p = 256, 500, 192
    A, B, C = inputs(oz, m, n, p, 21)
    bad = A.copy()
    bad[0, 0] = -(2.0 ** 921)
    cfg = oz.config_for("ozIMMU_H", 8)
    h = oz.Handle(0)
    oz.ozaki_gemm(1.0, dev(bad), dev(B), 0.0, dev(C), cfg, handle=h, sync_check=False)
    want = checker.gemm(1.0, A, B, 0.0, C, k=8)
    got = oz.ozaki_gemm(1.0, dev(A), dev(B), 0.0, dev(C), cfg, handle=h)   # sync_check on
    assert_bitwise(got.cpu().numpy(), want, "clean device call after a deferred error")
    assert_bitwise(oz.ozaki_gemm(1.0, A, B, 0.0, C, cfg, handle=h), want,
                   "clean host call after a deferred error")
    with pytest.raises(OverflowError):
        h.sync_status()
    h.sync_status()   # reported once, then clear
    h.close()


def _overflow_inputs(m, n, p):
    # slices 127, 63, 63, ... (all positive): the products of a group add up
    v = (127 + 63 / 127) / 64
    return np.full((m, n), v), np.full((n, p), v), np.zeros((m, p))


@pytest.mark.parametrize("path", ["device", "host"])
def test_checked_overflow_raises_like_the_reference(oz, path):
    from oracle import oracle
    port = oracle.PortLib()
    m, n, p, k = 64, 65536, 48, 14
    A, B, C = _overflow_inputs(m, n, p)
    with pytest.raises(oracle.OracleError) as e:             # the reference semantics
        port.gemm(1.0, A, B, 0.0, C, k=k, force_r=14)
    assert e.value.code == oracle.ERR_OVERFLOW
    cfg = oz.config_for("ozIMMU_H", k)
    cfg.force_r = 14
    if path == "device":
        out = dev(np.full((m, p), 7.0))
        with pytest.raises(oz.Int32OverflowError, match="INT32 overflow at"):
            oz.ozaki_gemm(1.0, dev(A), dev(B), 0.0, dev(C), cfg, out=out)
        assert bool((out == 7.0).all()), "C written despite the overflow"
    else:
        out = np.full((m, p), 7.0)
        with pytest.raises(oz.Int32OverflowError):
            oz.ozaki_gemm(1.0, A, B, 0.0, C, cfg, out=out)
        assert (out == 7.0).all()


@pytest.mark.parametrize("path", ["device", "host"])
def test_wrapping_overflow_bit_exact(oz, checker, path):
    """OverflowMode::Wrapping: the reference wraps each running sum mod 2^32
    (int_gemm.cpp:50-51), so does the tensor core."""
    m, n, p, k = 64, 65536, 48, 14
    A, B, C = _overflow_inputs(m, n, p)
    want = checker.gemm(1.0, A, B, 0.0, C, k=k, force_r=14, wrapping=True)
    cfg = oz.config_for("ozIMMU_H", k)
    cfg.force_r, cfg.overflow = 14, oz.OverflowMode.Wrapping
    got = oz.ozaki_gemm(1.0, dev(A), dev(B), 0.0, dev(C), cfg).cpu().numpy() \
        if path == "device" else oz.ozaki_gemm(1.0, A, B, 0.0, C, cfg)
    assert_bitwise(got, want)
    # and the wrapped result differs from the unforced (r = 2) one: overflow happened
    assert not np.array_equal(got, checker.gemm(1.0, A, B, 0.0, C, k=k))


def test_checked_no_overflow_with_forced_r_is_bit_exact(oz, checker):
    """Forced r whose chunks could overflow but do not (random data): the verification
    passes and the result is the reference's."""
    m, n, p, k = 200, 40000, 150, 12
    A, B, C = inputs(oz, m, n, p, 31, phi=0.5)
    cfg = oz.config_for("ozIMMU_H", k)
    cfg.force_r = 12
    want = checker.gemm(1.25, A, B, 0.5, C, k=k, force_r=12)
    assert_bitwise(oz.ozaki_gemm(1.25, dev(A), dev(B), 0.5, dev(C), cfg).cpu().numpy(), want)
    assert_bitwise(oz.ozaki_gemm(1.25, A, B, 0.5, C, cfg), want)


def test_c_write_only_needs_positive_alpha(oz):
    """c_write_only drops fl(beta*c); with alpha <= 0 the sign of a zero would come
    from it (-0 + +0 = +0), so the slice-level entry rejects it."""
    m, n, p, k = 64, 64, 64, 2
    lds = oz.slice_ld(n)
    s = torch.zeros((k, m, lds), dtype=torch.int8, device="cuda")
    sh = torch.ones(m, dtype=torch.float64, device="cuda")
    c = torch.zeros((m, p), dtype=torch.float64, device="cuda")
    h = oz.default_handle(0)
    for alpha, ok in ((-1.0, False), (0.0, False), (-0.0, False), (2.0, True)):
        opt = oz.Options()
        opt.c_write_only = 1
        rc = oz.lib.ozmm_gemm_slices(h.h, m, n, p, k, 7, 0, s.data_ptr(), lds, sh.data_ptr(),
                                     s.data_ptr(), lds, sh.data_ptr(), alpha, 0.0, c.data_ptr(),
                                     p, ctypes.byref(opt))
        assert (rc == oz.OZMM_OK) == ok, (alpha, rc)
    torch.cuda.synchronize()


@pytest.mark.parametrize("method", ["ozIMMU", "ozIMMU_RN", "ozIMMU_EF", "ozIMMU_H"])
def test_methods_through_host_entry(oz, checker, method):
    m, n, p, k = 200, 1500, 170, 9
    A, B, C = inputs(oz, m, n, p, 41, phi=2.0)
    want = checker.gemm(1.5, A, B, 0.5, C, k=k, method=method)
    assert_bitwise(oz.ozaki_gemm(1.5, A, B, 0.5, C, oz.config_for(method, k)), want, method)


def test_groupwise_simple_bitmask(oz, checker):
    """(BitMask, GroupwiseSimple): valid in the reference when r >= k."""
    m, n, p, k = 128, 1024, 96, 8
    A, B, C = inputs(oz, m, n, p, 51)
    cfg = oz.config_for("ozIMMU_EF", k)
    cfg.accumulation = oz.Accumulation.GroupwiseSimple
    want = checker.gemm(1.0, A, B, 0.0, C, k=k, method="ozIMMU_EF")   # r = 128 >= k: same chunks
    assert_bitwise(oz.ozaki_gemm(1.0, dev(A), dev(B), 0.0, dev(C), cfg).cpu().numpy(), want)


def _host_call(oz, ta, tb, m, n, p, alpha, A, B, beta, C, k, **opt_kw):
    """ozmm_dgemm_host straight through the C ABI on the caller's own buffers
    (lda / ldb / ldc from the arrays' row strides)."""
    h = oz.default_handle(0)
    h.set_stream(None)
    opt = oz.Options()
    for key, v in opt_kw.items():
        setattr(opt, key, v)
    return oz.lib.ozmm_dgemm_host(h.h, b"T" if ta else b"N", b"T" if tb else b"N", m, n, p, alpha,
                                  A.ctypes.data, A.strides[0] // 8, B.ctypes.data,
                                  B.strides[0] // 8, beta, C.ctypes.data, C.strides[0] // 8, k,
                                  ctypes.byref(opt), None, None)


def _pinned_like(x):
    t = torch.empty(x.shape, dtype=torch.float64).pin_memory()
    a = t.numpy()
    a[...] = x
    return a, t


@pytest.mark.parametrize("staging", [0, 1, 2])
@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("case", [
    # (transa, transb, m, n, p, alpha, beta, pad)
    (False, False, 700, 1100, 530, 1.0, 0.0, 0),
    (True, False, 512, 900, 384, 1.5, 0.5, 3),
    (False, True, 333, 640, 257, -2.0, 0.0, 5),
])
def test_host_entry_staging_bit_exact(oz, checker, staging, pinned, case):
    """Pageable caller buffers go through the pinned slot rings (host_stage.hpp);
    pinned ones are copied directly; the driver-copy mode stays available.
    Every combination must give the reference's bits, with strided leading
    dimensions, transposes, beta != 0 (C read) and beta = 0 (C write-only)."""
    ta, tb, m, n, p, alpha, beta, pad = case
    k = 8
    A0, B0, C0 = inputs(oz, m, n, p, 61, phi=1.0)
    # non-finite C entries: beta = 0 still forms fl(beta*c) (scheme.cpp:287)
    C0[3, 5], C0[m - 1, p - 2], C0[m // 2, 0] = np.inf, np.nan, -np.inf
    want = checker.gemm(alpha, A0, B0, beta, C0, k=k)
    sa = np.ascontiguousarray(A0.T) if ta else A0
    sb = np.ascontiguousarray(B0.T) if tb else B0

    def padded(x):  # leading dimension cols + pad, pad columns poisoned
        y = np.full((x.shape[0], x.shape[1] + pad), np.nan)
        y[:, :x.shape[1]] = x
        return y

    keep = []
    bufs = []
    for x in (padded(sa), padded(sb), padded(C0)):
        if pinned:
            a, t = _pinned_like(x)
            keep.append(t)
            bufs.append(a)
        else:
            bufs.append(x.copy())
    A, B, C = bufs
    rc = _host_call(oz, ta, tb, m, n, p, alpha, A[:, :sa.shape[1]], B[:, :sb.shape[1]], beta,
                    C[:, :p], k, host_staging=staging, host_panels=3, sync_check=1)
    assert rc == oz.OZMM_OK, oz.lib.ozmm_last_error(oz.default_handle(0).h)
    assert_bitwise(C[:, :p], want, f"staging={staging} pinned={pinned}")
    if pad:
        assert np.isnan(C[:, p:]).all(), "padding columns of C were written"


@pytest.mark.parametrize("staging", [0, 2])
def test_host_entry_staged_range_error_leaves_c(oz, staging):
    """Range error with staged (pageable) buffers: OZMM_ERR_RANGE, C untouched,
    then a clean call on the same handle."""
    m, n, p, k = 600, 800, 300, 8
    A, B, C = inputs(oz, m, n, p, 71)
    bad = A.copy()
    bad[m - 5, 17] = 2.0 ** 950
    for beta in (0.0, 0.5):
        c = C.copy()
        rc = _host_call(oz, False, False, m, n, p, 1.0, bad, B, beta, c, k, host_staging=staging,
                        host_panels=4)
        assert rc == oz.OZMM_ERR_RANGE
        assert_bitwise(c, C, "C must be untouched on a range error")
    c = C.copy()
    assert _host_call(oz, False, False, m, n, p, 1.0, A, B, 0.0, c, k,
                      host_staging=staging) == oz.OZMM_OK


def test_host_entry_staging_options_checked(oz):
    A, B, C = inputs(oz, 64, 64, 64, 81)
    assert _host_call(oz, False, False, 64, 64, 64, 1.0, A, B, 0.0, C.copy(), 8,
                      host_staging=3) == oz.OZMM_ERR_ARG
    assert _host_call(oz, False, False, 64, 64, 64, 1.0, A, B, 0.0, C.copy(), 8,
                      host_threads=-1) == oz.OZMM_ERR_ARG
    for nt in (1, 3):
        c = C.copy()
        assert _host_call(oz, False, False, 64, 64, 64, 1.0, A, B, 0.0, c, 8, host_staging=2,
                          host_threads=nt) == oz.OZMM_OK


def test_host_entry_staging_slots_grow_with_the_operands(oz, checker):
    """Slots are sized by the operands and re-allocated when a later pageable call
    on the same handle is larger: small, large, small again -- all bit-exact."""
    h = oz.Handle(0)
    try:
        for (m, n, p) in [(64, 96, 80), (1536, 2048, 1280), (100, 130, 70)]:
            A, B, C = inputs(oz, m, n, p, 101)
            want = checker.gemm(1.0, A, B, 0.0, C, k=8)
            c = C.copy()
            opt = oz.Options()
            h.set_stream(None)
            rc = oz.lib.ozmm_dgemm_host(h.h, b"N", b"N", m, n, p, 1.0, A.ctypes.data, n,
                                        B.ctypes.data, p, 0.0, c.ctypes.data, p, 8,
                                        ctypes.byref(opt), None, None)
            assert rc == oz.OZMM_OK
            assert_bitwise(c, want, f"{m}x{n}x{p}")
    finally:
        h.close()


@pytest.fixture(scope="module")
def ref():
    from oracle import oracle
    if not os.path.exists(oracle.REF_SO):
        pytest.skip("oracle/_ref not built")
    return oracle.RefLib()


@pytest.mark.parametrize("strategy", ["rn_const", "bitmask", "rn_per_slice"])
@pytest.mark.parametrize("side", ["L", "R"])
def test_split_dump_matches_reference_split(oz, ref, strategy, side):
    """split_dump (ozmm_split_host) against the reference's split_any on the same
    matrix: slices, shift or per-slice units and the residual, bit for bit
    (split.cpp:182-198, dump_split :254-270), with zero, -0, power-of-two,
    tiny (underflowing grid) and ragged-magnitude lines."""
    rng = np.random.default_rng(11)
    a = (rng.random((37, 301)) - 0.5) * np.exp(2.0 * rng.standard_normal((37, 301)))
    a[3] = 0.0
    a[4] = -0.0
    a[5] = 2.0 ** rng.integers(-20, 20, 301)
    a[6] *= 2.0 ** -1060
    a[:, 7] = 0.0
    a[:, 8] = 2.0 ** 40
    if side == "R":
        a = np.ascontiguousarray(a.T)
    k = 9
    strat = {"rn_const": oz.SliceStrategy.RoundNearestConstShift, "bitmask": oz.SliceStrategy.BitMask,
             "rn_per_slice": oz.SliceStrategy.RoundNearestPerSlice}[strategy]
    sl, out, res = oz.split_dump(a, k, side, strat)
    want_sl, want_out, want_res = ref.split_any(a, k, strategy, "left" if side == "L" else "right",
                                                residual=True)
    np.testing.assert_array_equal(sl, want_sl)
    assert_bitwise(out, want_out, "shift / units")
    assert_bitwise(res, want_res, "residual")


def test_split_dump_argument_errors(oz):
    a = np.ones((4, 8))
    with pytest.raises(ValueError):
        oz.split_dump(a, 0)
    with pytest.raises(ValueError):
        oz.split_dump(a, 33)  # kMaxK = 32 (csrc/ozimmu_gemm.cuh)
    with pytest.raises(OverflowError):
        oz.split_dump(np.full((4, 8), 2.0 ** 950), 4)


def _host_out_call(oz, ta, tb, m, n, p, alpha, A, B, beta, C, D, k, **opt_kw):
    """ozmm_dgemm_host_out: C read-only, the result in D (ldd from D's row stride)."""
    h = oz.default_handle(0)
    h.set_stream(None)
    opt = oz.Options()
    for key, v in opt_kw.items():
        setattr(opt, key, v)
    return oz.lib.ozmm_dgemm_host_out(h.h, b"T" if ta else b"N", b"T" if tb else b"N", m, n, p,
                                      alpha, A.ctypes.data, A.strides[0] // 8, B.ctypes.data,
                                      B.strides[0] // 8, beta, C.ctypes.data, C.strides[0] // 8,
                                      D.ctypes.data, D.strides[0] // 8, k, ctypes.byref(opt),
                                      None, None)


@pytest.mark.parametrize("staging", [0, 1, 2])
@pytest.mark.parametrize("pinned_out", [False, True])
@pytest.mark.parametrize("case", [
    # (transa, transb, m, n, p, alpha, beta, method)
    (False, False, 700, 1100, 530, 1.0, 0.0, 0),   # beta = 0: C not uploaded, patch from C
    (True, False, 512, 900, 384, 1.5, 0.5, 0),     # beta != 0: C uploaded
    (False, True, 333, 640, 257, -2.0, 0.0, 0),    # alpha < 0: C uploaded
    (False, False, 300, 700, 260, 1.0, 0.25, 1),   # ozIMMU: the copy-in / copy-out route
])
def test_host_out_entry_matches_in_place(oz, checker, staging, pinned_out, case):
    """ozmm_dgemm_host_out (the reference's new-matrix semantics, scheme.cpp:281,
    :289): the result equals the in-place ozmm_dgemm_host bit for bit, C is not
    written (not even its padding), and D's padding columns stay untouched."""
    ta, tb, m, n, p, alpha, beta, method = case
    k = 8
    A0, B0, C0 = inputs(oz, m, n, p, 81, phi=1.0)
    C0[3, 5], C0[m - 1, p - 2], C0[m // 2, 0] = np.inf, np.nan, -np.inf
    sa = np.ascontiguousarray(A0.T) if ta else A0
    sb = np.ascontiguousarray(B0.T) if tb else B0
    cfg_kw = dict(host_staging=staging, host_panels=3, sync_check=1, method=method)
    Cin = np.full((m, p + 3), -5.0)
    Cin[:, :p] = C0
    want = Cin.copy()
    assert _host_call(oz, ta, tb, m, n, p, alpha, sa, sb, beta, want[:, :p], k, **cfg_kw) == 0
    keep = []
    if pinned_out:
        D, t = _pinned_like(np.full((m, p + 2), 7.0))
        keep.append(t)
    else:
        D = np.full((m, p + 2), 7.0)
    before = Cin.copy()
    rc = _host_out_call(oz, ta, tb, m, n, p, alpha, sa, sb, beta, Cin[:, :p], D[:, :p], k, **cfg_kw)
    assert rc == oz.OZMM_OK, oz.lib.ozmm_last_error(oz.default_handle(0).h)
    assert_bitwise(D[:, :p], want[:, :p], f"staging={staging} pinned_out={pinned_out}")
    assert (D[:, p:] == 7.0).all(), "padding columns of D were written"
    assert before.tobytes() == Cin.tobytes(), "C was written"


def test_host_out_entry_errors(oz):
    """Overlapping D and C is refused; a range error leaves C untouched."""
    m, n, p, k = 256, 512, 128, 8
    A, B, C = inputs(oz, m, n, p, 91)
    big = np.zeros((m, p + 8))
    rc = _host_out_call(oz, False, False, m, n, p, 1.0, A, B, 0.5, big[:, :p], big[:, 8:], k)
    assert rc == oz.OZMM_ERR_ARG
    A2 = A.copy()
    A2[7, 3] = 2.0 ** 950
    D = np.zeros((m, p))
    before = C.copy()
    rc = _host_out_call(oz, False, False, m, n, p, 1.0, A2, B, 0.0, C, D, k)
    assert rc == oz.OZMM_ERR_RANGE
    assert before.tobytes() == C.tobytes()
    # the same handle is clean afterwards
    rc = _host_out_call(oz, False, False, m, n, p, 1.0, A, B, 0.0, C, D, k)
    assert rc == oz.OZMM_OK
