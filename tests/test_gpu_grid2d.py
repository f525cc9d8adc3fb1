"""GPU: the 2-D partition's CUDA backend (grid2d.Backend) through
torch.distributed/NCCL with world size 1 (the pod exposes one GPU), checked
bit-exactly against the single-call path.  Multi-rank gather logic is covered
on CPU by tests/test_grid2d_gloo.py."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def test_grid2d_cuda_world1():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.distributed as dist
    from paper_2409_13313_b200 import ozmm
    from paper_2409_13313_b200.grid2d import Backend, Grid2DGemm
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        m, n, p, k = 512, 3000, 384, 8
        A = torch.tensor(ozmm.gen_phi_matrix(m, n, 1.0, 1), device="cuda")
        B = torch.tensor(ozmm.gen_phi_matrix(n, p, 1.0, 2), device="cuda")
        C = torch.tensor(ozmm.gen_phi_matrix(m, p, 1.0, 3), device="cuda")
        G = Grid2DGemm(m, n, p, k, backend=Backend(0))
        got = C.clone()
        G.step(A, B, got, 1.5, 0.5)
        want = ozmm.ozaki_gemm(1.5, A, B, 0.5, C, ozmm.config_for("ozIMMU_H", k))
        assert torch.equal(got.view(torch.int64), want.view(torch.int64))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,trans,host", [(2, False, False), (4, False, False),
                                              (8, False, False), (4, True, False),
                                              (8, True, False), (2, False, True),
                                              (4, False, True), (8, True, True),
                                              (2, False, "panels"), (4, False, "panels"),
                                              (8, False, "panels")])
def test_grid2d_cuda_emulated_ranks(world, trans, host):
    """All ranks of a Pr x Pc grid as threads on the one GPU, with an in-process
    all-gather: the CUDA backend's strip launches (G1/G2/G3 on row/column ranges of
    the gathered panels, ozmm_gemm_slices_strided) must tile C exactly like the
    single call, bit for bit.  host: the C rows stream back into a pinned host
    block piece by piece (step's c_host), which must hold the same result;
    "panels": A also arrives in row panels with one ready event each, split and
    multiplied panel by panel."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import threading
    from paper_2409_13313_b200 import ozmm
    from paper_2409_13313_b200.grid2d import Backend, Grid2DGemm, make_layout

    m, n, p, k, alpha, beta = 1024, 2500, 768, 8, 1.25, -0.5
    A = ozmm.gen_phi_matrix(m, n, 1.0, 11)
    B = ozmm.gen_phi_matrix(n, p, 1.0, 12)
    C = ozmm.gen_phi_matrix(m, p, 1.0, 13)
    dev = lambda x: torch.tensor(np.ascontiguousarray(x), device="cuda")  # noqa: E731
    want = ozmm.ozaki_gemm(alpha, dev(A), dev(B), beta, dev(C),
                           ozmm.config_for("ozIMMU_H", k)).cpu().numpy()
    # transa / transb: each rank holds its shard of the stored transposes
    At, Bt = np.ascontiguousarray(A.T), np.ascontiguousarray(B.T)

    barriers, pool, lock = {}, {}, threading.Lock()

    class Done:
        def wait(self):
            pass

    def all_gather(out, inp, group):
        ranks = tuple(group)
        me = threading.current_thread().rank
        with lock:
            bar = barriers.setdefault(ranks, threading.Barrier(len(ranks)))
            seq = threading.current_thread().seq.setdefault(ranks, 0)
            threading.current_thread().seq[ranks] = seq + 1
        torch.cuda.synchronize()
        with lock:
            pool[(ranks, seq, me)] = inp
        bar.wait()
        parts = [pool[(ranks, seq, r)] for r in ranks]
        out.copy_(torch.cat([x.reshape(-1) for x in parts]).view_as(out))
        torch.cuda.synchronize()
        bar.wait()
        return Done()

    got = np.full((m, p), np.nan)
    errors = []

    def run(rank):
        try:
            th = threading.current_thread()
            th.rank, th.seq = rank, {}
            L = make_layout(m, n, p, world, rank)
            G = Grid2DGemm(m, n, p, k, world=world, rank=rank, backend=Backend(0),
                           group_factory=lambda ranks: tuple(ranks), all_gather=all_gather,
                           transa=trans, transb=trans)
            if trans:
                a = dev(At[:, L.a_row0:L.a_row0 + L.ms])
                b = dev(Bt[L.b_col0:L.b_col0 + L.ps])
            else:
                a = dev(A[L.a_row0:L.a_row0 + L.ms])
                b = dev(B[:, L.b_col0:L.b_col0 + L.ps])
            c = dev(C[L.c_row0:L.c_row0 + L.mr, L.c_col0:L.c_col0 + L.pcols])
            hc = torch.full(tuple(c.shape), float("nan"), dtype=torch.float64).pin_memory() \
                if host else None
            ready = None
            if host == "panels":
                cuts = sorted({0, L.ms, *(int(x) for x in np.random.default_rng(rank).integers(
                    1, L.ms, 2))})
                ready = {"a": []}
                for lo, hi in zip(cuts[:-1], cuts[1:]):
                    e = torch.cuda.Event()
                    e.record()
                    ready["a"].append((lo, hi, e))
            G.step(a, b, c, alpha, beta, c_host=hc, ready=ready)
            torch.cuda.synchronize()
            got[L.c_row0:L.c_row0 + L.mr, L.c_col0:L.c_col0 + L.pcols] = \
                (hc if host else c.cpu()).numpy()
        except BaseException as ex:  # surfaced below
            errors.append(ex)
            for bar in list(barriers.values()):
                bar.abort()

    threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=300)
    assert not errors, errors
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_gemm_slices_c_write_only():
    """c_write_only (beta = 0, finite C): C is not read, the result equals the
    reference's fl(alpha*D) + fl(0*c); with beta != 0 the option is rejected."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2409_13313_b200 import ozmm
    from paper_2409_13313_b200.grid2d import Backend
    m, n, p, k = 300, 1100, 260, 8
    A = torch.tensor(ozmm.gen_phi_matrix(m, n, 1.0, 21), device="cuda")
    B = torch.tensor(ozmm.gen_phi_matrix(n, p, 1.0, 22), device="cuda")
    C0 = torch.tensor(ozmm.gen_phi_matrix(m, p, 1.0, 23), device="cuda")
    want = ozmm.ozaki_gemm(1.25, A, B, 0.0, C0, ozmm.config_for("ozIMMU_H", k))
    be = Backend(0)
    beta_bits, lds = ozmm.compute_beta(n), ozmm.slice_ld(n)
    sa = torch.empty((k, m, lds), dtype=torch.int8, device="cuda")
    sb = torch.empty((k, p, lds), dtype=torch.int8, device="cuda")
    mu = torch.empty(m, dtype=torch.float64, device="cuda")
    nu = torch.empty(p, dtype=torch.float64, device="cuda")
    la = torch.empty((m, k), dtype=torch.int32, device="cuda")
    lb = torch.empty((p, k), dtype=torch.int32, device="cuda")
    be.split(A, k, "L", False, beta_bits, sa, mu, lsum=la)
    be.split(B, k, "R", False, beta_bits, sb, nu, lsum=lb)
    got = torch.full((m, p), float("nan"), dtype=torch.float64, device="cuda")  # never read
    be.gemm(m, n, p, k, beta_bits, sa, mu, sb, nu, 1.25, 0.0, got, lsa=la, lsb=lb,
            c_write_only=True)
    torch.cuda.synchronize()
    assert torch.equal(got.view(torch.int64), want.view(torch.int64))
    with pytest.raises(ValueError):
        be.gemm(m, n, p, k, beta_bits, sa, mu, sb, nu, 1.25, 0.5, got, lsa=la, lsb=lb,
                c_write_only=True)


def _native_case(trans, k=8, n=2500):
    from paper_2409_13313_b200 import ozmm
    m, p, alpha, beta = 1024, 768, 1.25, -0.5
    A = ozmm.gen_phi_matrix(m, n, 1.0, 21)
    B = ozmm.gen_phi_matrix(n, p, 1.0, 22)
    C = ozmm.gen_phi_matrix(m, p, 1.0, 23)
    dev = lambda x: torch.tensor(np.ascontiguousarray(x), device="cuda")  # noqa: E731
    want = ozmm.ozaki_gemm(alpha, dev(A), dev(B), beta, dev(C),
                           ozmm.config_for("ozIMMU_H", k)).cpu().numpy()

    def shard(L):
        if trans:
            a = dev(np.ascontiguousarray(A.T)[:, L.a_row0:L.a_row0 + L.ms])
            b = dev(np.ascontiguousarray(B.T)[L.b_col0:L.b_col0 + L.ps])
        else:
            a = dev(A[L.a_row0:L.a_row0 + L.ms])
            b = dev(B[:, L.b_col0:L.b_col0 + L.ps])
        c = dev(C[L.c_row0:L.c_row0 + L.mr, L.c_col0:L.c_col0 + L.pcols])
        return a, b, c
    return (m, n, p, k, alpha, beta), want, shard


@pytest.mark.parametrize("trans", [False, True])
def test_native_grid_world1(trans):
    """ozmm_dgemm_2d on a 1x1 grid (no collective) equals the single call."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2409_13313_b200.grid2d import NativeGrid2D
    (m, n, p, k, alpha, beta), want, shard = _native_case(trans)
    G = NativeGrid2D(m, n, p, k, world=1, rank=0, transa=trans, transb=trans)
    a, b, c = shard(G.L)
    G.step(a, b, c, alpha, beta)
    torch.cuda.synchronize()
    assert np.array_equal(c.cpu().numpy().view(np.uint64), want.view(np.uint64))
    G.close()


def test_native_grid_nccl_init():
    """The NCCL plumbing of the native grid: unique id, ncclCommInitRank and the
    two ncclCommSplit calls on a one-rank world, then a bit-exact step."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import ctypes
    from paper_2409_13313_b200 import ozmm
    (m, n, p, k, alpha, beta), want, shard = _native_case(False)
    from paper_2409_13313_b200.grid2d import make_layout
    h = ozmm.Handle(0)
    nid = (ctypes.c_char * 128)()
    assert ozmm.lib.ozmm_nccl_unique_id(nid) == 0, ozmm.lib.ozmm_grid_last_error()
    g = ctypes.c_void_p()
    rc = ozmm.lib.ozmm_grid_create(h.h, 0, 1, 0, nid, None, None, ctypes.byref(g))
    assert rc == 0, ozmm.lib.ozmm_grid_last_error()
    a, b, c = shard(make_layout(m, n, p, 1, 0))
    h.set_stream(torch.cuda.current_stream().cuda_stream)
    assert ozmm.lib.ozmm_dgemm_2d(g, b"N", b"N", m, n, p, alpha, a.data_ptr(), a.stride(0),
                                  b.data_ptr(), b.stride(0), beta, c.data_ptr(), c.stride(0),
                                  k) == 0, ozmm.lib.ozmm_grid_last_error()
    torch.cuda.synchronize()
    assert np.array_equal(c.cpu().numpy().view(np.uint64), want.view(np.uint64))
    assert ozmm.lib.ozmm_grid_destroy(g) == 0


@pytest.mark.parametrize("world,trans,k,n", [(2, False, 8, 2500), (4, False, 8, 2500),
                                             (8, False, 8, 2500), (8, True, 8, 2500),
                                             (2, True, 3, 333), (4, False, 11, 1500)])
def test_native_grid_emulated_ranks(world, trans, k, n):
    """ozmm_dgemm_2d with W ranks as threads on the one GPU: the all-gather hook
    copies the peers' parts (cudaMemcpy) between barriers.  The native split
    into panel slots, in-place gathers and strips must tile C like the single
    call, bit for bit."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import ctypes
    import threading
    from paper_2409_13313_b200 import ozmm
    from paper_2409_13313_b200.grid2d import NativeGrid2D, make_layout
    (m, n, p, k, alpha, beta), want, shard = _native_case(trans, k, n)
    cudart = ctypes.CDLL("libcudart.so.12")
    cudart.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
    barriers, pool, lock, errors = {}, {}, threading.Lock(), []

    def gather(ctx, group, send, recv, nbytes, stream):
        try:
            th = threading.current_thread()
            L = th.L
            members = tuple(L.gr * L.pc + c for c in range(L.pc)) if group == 0 else \
                tuple(r * L.pc + L.gc for r in range(L.pr))
            with lock:
                bar = barriers.setdefault(members, threading.Barrier(len(members)))
                seq = th.seq.setdefault(members, 0)
                th.seq[members] = seq + 1
            torch.cuda.synchronize()
            pool[(members, seq, th.rank)] = send
            bar.wait()
            for idx, r in enumerate(members):
                if r != th.rank:
                    assert cudart.cudaMemcpy(recv + idx * nbytes, pool[(members, seq, r)],
                                             nbytes, 3) == 0
            bar.wait()
            return 0
        except BaseException as ex:  # surfaced below
            errors.append(ex)
            for b in list(barriers.values()):
                b.abort()
            return 1
    hook = ozmm.ALLGATHER_FN(gather)
    got = np.full((m, p), np.nan)

    def run(rank):
        try:
            th = threading.current_thread()
            th.rank, th.seq = rank, {}
            th.L = L = make_layout(m, n, p, world, rank)
            G = NativeGrid2D(m, n, p, k, world=world, rank=rank, transa=trans, transb=trans,
                             hook=hook)
            a, b, c = shard(L)
            G.step(a, b, c, alpha, beta)
            torch.cuda.synchronize()
            got[L.c_row0:L.c_row0 + L.mr, L.c_col0:L.c_col0 + L.pcols] = c.cpu().numpy()
            G.close()
        except BaseException as ex:
            errors.append(ex)
            for b in list(barriers.values()):
                b.abort()

    threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=300)
    assert not errors, errors
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("world,bad", [(2, (1, "A")), (4, (2, "B")), (8, (5, "A")), (4, None)])
def test_native_grid_range_error_reaches_every_rank(world, bad):
    """ozmm_dgemm_2d: a line max >= 2^921 in ONE rank's shard makes EVERY rank
    return OZMM_ERR_RANGE (OverflowError) before any strip writes its C block --
    the grid-wide max of the range flags (row gather, then column gather).
    bad = None is the negative control (no error anywhere, bit-exact result)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import ctypes
    import threading
    from paper_2409_13313_b200 import ozmm
    from paper_2409_13313_b200.grid2d import NativeGrid2D, make_layout
    (m, n, p, k, alpha, beta), want, shard = _native_case(False, 8, 700)
    cudart = ctypes.CDLL("libcudart.so.12")
    cudart.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
    barriers, pool, lock, errors, outcome = {}, {}, threading.Lock(), [], {}

    def gather(ctx, group, send, recv, nbytes, stream):
        th = threading.current_thread()
        L = th.L
        members = tuple(L.gr * L.pc + c for c in range(L.pc)) if group == 0 else \
            tuple(r * L.pc + L.gc for r in range(L.pr))
        with lock:
            bar = barriers.setdefault(members, threading.Barrier(len(members)))
            seq = th.seq.setdefault(members, 0)
            th.seq[members] = seq + 1
        torch.cuda.synchronize()
        pool[(members, seq, th.rank)] = send
        bar.wait(timeout=120)
        for idx, r in enumerate(members):
            if r != th.rank:
                assert cudart.cudaMemcpy(recv + idx * nbytes, pool[(members, seq, r)],
                                         nbytes, 3) == 0
        bar.wait(timeout=120)
        return 0
    hook = ozmm.ALLGATHER_FN(gather)

    def run(rank):
        try:
            th = threading.current_thread()
            th.rank, th.seq = rank, {}
            th.L = L = make_layout(m, n, p, world, rank)
            G = NativeGrid2D(m, n, p, k, world=world, rank=rank, hook=hook)
            a, b, c = shard(L)
            if bad is not None and rank == bad[0]:
                (a if bad[1] == "A" else b)[3, 4] = 2.0 ** 940
            c0 = c.clone()
            try:
                G.step(a, b, c, alpha, beta)
                torch.cuda.synchronize()
                outcome[rank] = ("ok", torch.equal(c.cpu(), torch.from_numpy(
                    want[L.c_row0:L.c_row0 + L.mr, L.c_col0:L.c_col0 + L.pcols])))
            except OverflowError:
                torch.cuda.synchronize()
                outcome[rank] = ("OverflowError", torch.equal(c.view(torch.int64),
                                                              c0.view(torch.int64)))
            G.close()
        except BaseException as ex:
            errors.append(ex)
            for b_ in list(barriers.values()):
                b_.abort()

    threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=300)
    assert not errors, errors
    expect = "OverflowError" if bad is not None else "ok"
    assert outcome == {r: (expect, True) for r in range(world)}, outcome


def test_grid2d_cuda_sync_check_range_error():
    """Grid2DGemm.step(sync_check=True) on the CUDA backend: a line max >= 2^921
    raises OverflowError before any GEMM (C untouched), the flag is cleared, and
    the next clean step is bit-exact."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2409_13313_b200 import ozmm
    from paper_2409_13313_b200.grid2d import Backend, Grid2DGemm
    m, n, p, k = 512, 1000, 384, 8
    A = ozmm.gen_phi_matrix(m, n, 1.0, 31)
    B = ozmm.gen_phi_matrix(n, p, 1.0, 32)
    G = Grid2DGemm(m, n, p, k, world=1, rank=0, backend=Backend(0),
                   group_factory=lambda ranks: tuple(ranks), all_gather=None)
    bad = A.copy()
    bad[7, 11] = 2.0 ** 925
    a, b = torch.tensor(bad, device="cuda"), torch.tensor(B, device="cuda")
    c = torch.full((m, p), 7.0, dtype=torch.float64, device="cuda")
    with pytest.raises(OverflowError):
        G.step(a, b, c, 1.0, 0.0, sync_check=True)
    assert bool((c == 7.0).all())
    # A in panels (the e2e upload order): the bad line sits in the last panel
    evs = []
    for lo, hi in ((0, 256), (256, m)):
        e = torch.cuda.Event()
        e.record()
        evs.append((lo, hi, e))
    bad2 = A.copy()
    bad2[300, 5] = 2.0 ** 925
    with pytest.raises(OverflowError):
        G.step(torch.tensor(bad2, device="cuda"), b, c, 1.0, 0.0, ready={"a": evs},
               sync_check=True)
    assert bool((c == 7.0).all())
    want = ozmm.ozaki_gemm(1.0, torch.tensor(A, device="cuda"), b, 0.0, torch.zeros_like(c),
                           ozmm.config_for("ozIMMU_H", k)).cpu().numpy()
    G.step(torch.tensor(A, device="cuda"), b, c, 1.0, 0.0, sync_check=True)
    torch.cuda.synchronize()
    assert np.array_equal(c.cpu().numpy().view(np.uint64), want.view(np.uint64))


def test_native_grid_rejects_bad_shapes():
    """ozmm_dgemm_2d: m or p not divisible by Pr*Pc, and k outside 1..32, are
    argument / config errors (no launch)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import ctypes
    from paper_2409_13313_b200 import ozmm
    hook = ozmm.ALLGATHER_FN(lambda *a: 0)
    h = ozmm.Handle(0)
    g = ctypes.c_void_p()
    assert ozmm.lib.ozmm_grid_create(h.h, 0, 4, 1, None, ctypes.cast(hook, ctypes.c_void_p),
                                     None, ctypes.byref(g)) == 0
    x = torch.zeros(64, 64, dtype=torch.float64, device="cuda")
    args = lambda m, p, k: (g, b"N", b"N", m, 64, p, 1.0, x.data_ptr(), 64, x.data_ptr(),  # noqa
                            64, 0.0, x.data_ptr(), 64, k)
    assert ozmm.lib.ozmm_dgemm_2d(*args(66, 64, 8)) == ozmm.OZMM_ERR_ARG
    assert b"divisible" in ozmm.lib.ozmm_grid_last_error()
    assert ozmm.lib.ozmm_dgemm_2d(*args(64, 62, 8)) == ozmm.OZMM_ERR_ARG
    assert ozmm.lib.ozmm_dgemm_2d(*args(64, 64, 33)) == ozmm.OZMM_ERR_CONFIG
    # world > 1 without an id or a hook
    g2 = ctypes.c_void_p()
    assert ozmm.lib.ozmm_grid_create(h.h, 0, 2, 0, None, None, None,
                                     ctypes.byref(g2)) == ozmm.OZMM_ERR_ARG
    assert ozmm.lib.ozmm_grid_destroy(g) == 0
