"""CPU, multi-process: the 2-D block partition (grid2d.Grid2DGemm) under gloo.

Runs the real orchestration -- rank grid, row/column communicators, per-rank
slicing of full rows/columns, async slice-panel all-gathers overlapped with the
three strip GEMMs -- with world sizes 2, 4 and 8 (grids 2x1, 2x2, 2x4) on CPU.  The compute backend is a TEST-ONLY stand-in (the GPU kernels
need a B200): slicing by the oracle port, and the group-wise accumulation of
the gathered slice panels restated in numpy (exact int64 products, the
reference's flush order scheme.cpp:81-101 and flush arithmetic :29-41).
Each rank's C block must equal the single-process reference result bitwise.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleBackend:
    """Test stand-in for grid2d.Backend (CPU tensors)."""

    def __init__(self):
        import sys
        sys.path.insert(0, ROOT)
        from oracle.oracle import PortLib
        self.port = PortLib()

    def empty(self, shape, dtype):
        return torch.zeros(shape, dtype=dtype)

    def split(self, x, k, side, trans, beta, out_slices, out_shift):
        from oracle.oracle import OracleError
        a = x.numpy().T if trans else x.numpy()
        try:
            s = self.port.split(np.ascontiguousarray(a), k, "left" if side == "L" else "right",
                                force_beta=beta)
        except OracleError:  # line max >= 2^921: flagged like the CUDA backend's split
            self._range = 1
            out_slices.zero_()
            out_shift.zero_()
            return
        planes = s.slices if side == "L" else s.slices.transpose(0, 2, 1)  # [k][lines][n]
        out_slices.zero_()
        out_slices[:, :, : planes.shape[2]] = torch.from_numpy(np.ascontiguousarray(planes))
        out_shift.copy_(torch.from_numpy(s.shift))

    def range_error(self):
        r, self._range = getattr(self, "_range", 0), 0
        return r

    def gemm(self, m, n, p, k, beta_bits, a_slices, mu, b_slices, nu, alpha, beta, c):
        from paper_2409_13313_b200.ozmm import compute_r
        r = compute_r(n, beta_bits)
        A = a_slices.numpy()[:, :, :n].astype(np.int64)
        B = b_slices.numpy()[:, :, :n].astype(np.int64)
        mu, nu = mu.numpy(), nu.numpy()
        D = np.zeros((m, p))
        for g in range(2, k + 2):
            acc = np.zeros((m, p), np.int64)
            q = 0
            for s in range(1, g):
                q += 1
                acc += A[s - 1] @ B[g - s - 1].T
                if q == r or s == g - 1:
                    ru = np.ldexp(mu, 2 - beta_bits * g)
                    D = D + (ru[:, None] * acc.astype(np.float64)) * nu[None, :]
                    q = 0
                    acc[:] = 0
        c.copy_(torch.from_numpy(alpha * D + beta * c.numpy()))


class OffsetOracleBackend(OracleBackend):
    """Test stand-in with the CUDA backend's offset-binary contract: split()
    emits byte = slice + o_s (o_1 = 2^beta, o_s = max(2, 2^(beta-1)); padding 0) and
    the signed line sums into lsum ([lines][k]); gemm() recovers the signed
    planes from the bytes, checks the line sums that travelled through the
    gathers against them, then accumulates like OracleBackend."""

    offset_planes = True

    @staticmethod
    def _offsets(k, beta):
        return np.array([1 << beta] + [max(2, 1 << (beta - 1))] * (k - 1), np.int64)

    def split(self, x, k, side, trans, beta, out_slices, out_shift, lsum=None):
        super().split(x, k, side, trans, beta, out_slices, out_shift)
        a = x.numpy().T if trans else x.numpy()
        n = a.shape[1] if side == "L" else a.shape[0]
        sl = out_slices.numpy()[:, :, :n].astype(np.int64)
        lsum.copy_(torch.from_numpy(sl.sum(axis=2).T.astype(np.int32)))
        biased = (sl + self._offsets(k, beta)[:, None, None]).astype(np.uint8).view(np.int8)
        out_slices[:, :, :n] = torch.from_numpy(np.ascontiguousarray(biased))

    def gemm(self, m, n, p, k, beta_bits, a_slices, mu, b_slices, nu, alpha, beta, c,
             lsa=None, lsb=None):
        off = self._offsets(k, beta_bits)

        def unbias(planes, sums):
            u = planes.numpy()[:, :, :n].view(np.uint8).astype(np.int64) - off[:, None, None]
            assert np.array_equal(u.sum(axis=2).T.astype(np.int32), sums.numpy())
            out = torch.zeros_like(planes)
            out[:, :, :n] = torch.from_numpy(u.astype(np.int8))
            return out
        super().gemm(m, n, p, k, beta_bits, unbias(a_slices, lsa), mu, unbias(b_slices, lsb),
                     nu, alpha, beta, c)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, m, n, p, k, phi, alpha, beta, q, offset=False):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2409_13313_b200 import ozmm
        from paper_2409_13313_b200.grid2d import Grid2DGemm
        G = Grid2DGemm(m, n, p, k, backend=OffsetOracleBackend() if offset else OracleBackend())
        L = G.L
        sa, sb, sc = (ozmm.counter_hash(5, i) for i in (1, 2, 3))
        a_rows = torch.from_numpy(ozmm.gen_phi_block(m, n, phi, sa, L.a_row0, L.ms, 0, n))
        b_cols = torch.from_numpy(ozmm.gen_phi_block(n, p, phi, sb, 0, n, L.b_col0, L.ps))
        c_blk = torch.from_numpy(ozmm.gen_phi_block(m, p, phi, sc, L.c_row0, L.mr, L.c_col0,
                                                    L.pcols))
        G.step(a_rows, b_cols, c_blk, alpha, beta)
        q.put((rank, L.c_row0, L.c_col0, c_blk.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,offset", [(2, False), (4, False), (8, False), (4, True),
                                          (8, True)])
def test_grid2d_matches_single_process(world, offset, port):
    m, n, p, k, phi, alpha, beta = 32, 200, 48, 8, 1.0, 1.5, 0.5
    from paper_2409_13313_b200 import ozmm
    A = ozmm.gen_phi_block(m, n, phi, ozmm.counter_hash(5, 1))
    B = ozmm.gen_phi_block(n, p, phi, ozmm.counter_hash(5, 2))
    C = ozmm.gen_phi_block(m, p, phi, ozmm.counter_hash(5, 3))
    want = port.gemm(alpha, A, B, beta, C, k=k)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, PORT[(world, offset)],
                                               m, n, p, k, phi, alpha, beta, q, offset))
             for r in range(world)]
    for pr in procs:
        pr.start()
    got = np.full((m, p), np.nan)
    for _ in range(world):
        rank, r0, c0, blk = q.get(timeout=120)
        got[r0:r0 + blk.shape[0], c0:c0 + blk.shape[1]] = blk
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


PORT = {(w, o): _free_port() for w in (2, 4, 8) for o in (False, True)}


def _range_worker(rank, world, port, bad_rank, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2409_13313_b200.grid2d import Grid2DGemm
        m, n, p, k = 32, 64, 48, 4
        G = Grid2DGemm(m, n, p, k, backend=OracleBackend())
        L = G.L
        a_rows = torch.ones((L.ms, n), dtype=torch.float64)
        if rank == bad_rank:
            a_rows[1, 3] = 2.0 ** 925
        b_cols = torch.ones((n, L.ps), dtype=torch.float64)
        c_blk = torch.full((L.mr, L.pcols), 7.0, dtype=torch.float64)
        try:
            G.step(a_rows, b_cols, c_blk, 1.0, 0.0, sync_check=True)
            q.put((rank, "no error", bool((c_blk == 7.0).all())))
        except OverflowError:
            q.put((rank, "OverflowError", bool((c_blk == 7.0).all())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,bad", [(4, 3), (8, 5), (4, -1)])
def test_grid2d_range_error_reaches_every_rank(world, bad):
    """sync_check: one rank's line max >= 2^921 (the reference throws
    std::overflow_error before writing, split.cpp:124-125) makes EVERY rank of
    the grid raise OverflowError before any GEMM, with C untouched."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_range_worker, args=(r, world, port, bad, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    want = "OverflowError" if bad >= 0 else "no error"  # bad = -1: the negative control
    assert res == [(r, want, bad >= 0) for r in range(world)]
