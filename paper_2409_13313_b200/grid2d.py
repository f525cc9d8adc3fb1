"""2-D block partition of the ozIMMU_H emulated DGEMM across ranks.

One process per GPU (``torch.distributed``, backend "nccl" on GPUs).  The
ranks form a Pr x Pc grid; rank (gr, gc) owns the C block (gr, gc) of size
(m/Pr) x (p/Pc).  The reference is single-process: this
partition is new, and it is bit-identical to the 1-GPU result because every
entry of D depends only on its row of op(A) (+ mu_i), its column of op(B)
(+ nu_j) and n -- the slicer is line-local (proj/src/split.cpp:157-171) and
the group-wise accumulation is entry-local (proj/src/scheme.cpp:81-101).

Per step each rank:
  1. slices m/(Pr*Pc) FULL rows of op(A) from its row panel and p/(Pr*Pc)
     FULL columns of op(B) from its column panel (K1; row maxima are local),
  2. all-gathers the INT8 slice planes + shift vectors (+ the int32 line sums
     of the offset-binary planes the CUDA backend uses): A planes inside its
     row communicator (the Pc ranks sharing gr), B planes inside its column
     communicator (the Pr ranks sharing gc).  No reductions: NCCL only
     broadcasts slice panels, as the north star asks,
  3. runs the fused K2+K3 kernel on its C block in three strips, the first
     of which needs no communication, so the gathers overlap the GEMM (step()).
     The first strip runs on a side stream: the other two wait only on the
     gathers, so their CTAs take the SMs the first strip's last partial wave
     leaves idle (no wave-quantisation gap between strips).

The compute backend is injectable (``Backend``): the default calls the CUDA
library; tests/test_grid2d_gloo.py drives the same orchestration under gloo
on CPU with a test-only backend to check the gather/partition logic.
"""
from __future__ import annotations

import contextlib
import ctypes
import math
import os
from dataclasses import dataclass

import torch
import torch.distributed as dist


def grid_shape(world: int) -> tuple[int, int]:
    """Pr x Pc with Pr <= Pc as square as possible: 1x1, 2x1, 2x2, 2x4 ..."""
    if world == 2:
        return 2, 1
    pr = int(math.isqrt(world))
    while world % pr:
        pr -= 1
    return pr, world // pr


@dataclass
class Layout:
    m: int
    n: int
    p: int
    pr: int
    pc: int
    gr: int
    gc: int

    @property
    def mr(self):  # rows of the C block / A row panel
        return self.m // self.pr

    @property
    def pcols(self):  # cols of the C block / B column panel
        return self.p // self.pc

    @property
    def ms(self):  # A rows this rank slices
        return self.mr // self.pc

    @property
    def ps(self):  # B cols this rank slices
        return self.pcols // self.pr

    @property
    def a_row0(self):  # first global row of op(A) this rank slices
        return self.gr * self.mr + self.gc * self.ms

    @property
    def b_col0(self):  # first global column of op(B) this rank slices
        return self.gc * self.pcols + self.gr * self.ps

    @property
    def c_row0(self):
        return self.gr * self.mr

    @property
    def c_col0(self):
        return self.gc * self.pcols


def make_layout(m: int, n: int, p: int, world: int, rank: int) -> Layout:
    pr, pc = grid_shape(world)
    if m % (pr * pc) or p % (pr * pc):
        raise ValueError(f"m={m}, p={p} must be divisible by Pr*Pc={pr * pc}")
    return Layout(m, n, p, pr, pc, rank // pc, rank % pc)


class Backend:
    """CUDA backend: K1 / K2+K3 through the C ABI (no CPU fallback).

    ``offset_planes``: the slice planes are the fused GEMM's offset-binary
    format (ozmm_split_offset / ozmm_gemm_slices_offset) and travel with their
    int32 line sums, which the grid gathers alongside the shift vectors."""

    offset_planes = True

    def __init__(self, device: int):
        from . import ozmm
        self.oz = ozmm
        self.device = torch.device("cuda", device)
        self.handle = ozmm.Handle(device)

    def empty(self, shape, dtype):
        return torch.empty(shape, dtype=dtype, device=self.device)

    def side_stream(self, after_current=True):
        """Context for the communication-free strip G1: a second stream that
        starts after the current one, so G2/G3 (which wait only on the gathers)
        fill the SMs G1's last partial wave leaves idle.  join_side() puts the
        current stream back behind it."""
        if not hasattr(self, "_side"):
            self._side = torch.cuda.Stream(self.device)
        cur = torch.cuda.current_stream(self.device)
        if after_current:  # else the caller orders the side stream with events
            self._side.wait_stream(cur)
        return torch.cuda.stream(self._side)

    def split_stream(self):
        """Stream for the per-panel A splits (Grid2DGemm.step with A panels); it
        starts after the current stream."""
        if not hasattr(self, "_split"):
            self._split = torch.cuda.Stream(self.device)
        self._split.wait_stream(torch.cuda.current_stream(self.device))
        return self._split

    def range_error(self) -> int:
        """1 if a split since the last query saw a line max >= 2^921 (the
        reference's std::overflow_error, split.cpp:124-125), else 0.  Synchronises
        the device and clears the flag."""
        torch.cuda.synchronize(self.device)
        uf = ctypes.c_int()
        rc = self.oz.lib.ozmm_sync_status(self.handle.h, ctypes.byref(uf))
        if rc == self.oz.OZMM_ERR_RANGE:
            return 1
        self.handle.check(rc)
        return 0

    def copy_stream(self):
        """Stream for the D2H copies of finished C rows (Grid2DGemm.step c_host)."""
        if not hasattr(self, "_copy"):
            self._copy = torch.cuda.Stream(self.device)
        return self._copy

    def join_side(self):
        if hasattr(self, "_side"):
            torch.cuda.current_stream(self.device).wait_stream(self._side)

    def split(self, x, k: int, side: str, trans: bool, beta: int, out_slices, out_shift,
              lsum=None):
        """lsum ([lines][k] int32 view): offset-binary planes plus their line sums;
        None: the reference's signed planes."""
        oz = self.oz
        rows, cols = x.shape
        if side == "L":
            lines, n = (cols, rows) if trans else (rows, cols)
        else:
            n, lines = (cols, rows) if trans else (rows, cols)
        self.handle.set_stream(torch.cuda.current_stream(self.device).cuda_stream)
        args = (self.handle.h, side.encode(), b"T" if trans else b"N", lines, n, x.data_ptr(),
                x.stride(0), k, beta, out_slices.data_ptr(), out_slices.shape[-1],
                out_shift.data_ptr())
        if lsum is None:
            self.handle.check(oz.lib.ozmm_split(*args))
        else:  # out_slices may be a line range of a larger [k][lines][lds] array
            self.handle.check(oz.lib.ozmm_split_offset_strided(
                *args[:-1], out_slices.stride(0), args[-1], lsum.data_ptr(), lsum.stride(1),
                lsum.stride(0)))

    def gemm(self, m, n, p, k, beta_bits, a_slices, mu, b_slices, nu, alpha, beta, c,
             lsa=None, lsb=None, c_write_only=False):
        """K2+K3 on [k][m][lds] / [k][p][lds] slice views (row / column ranges of a
        panel are fine: the plane stride is passed through); lsa / lsb: the line
        sums of offset-binary planes ([m][k] / [p][k] views)."""
        oz = self.oz
        self.handle.set_stream(torch.cuda.current_stream(self.device).cuda_stream)
        opt = oz.Options()
        opt.c_write_only = int(c_write_only)
        if lsa is None:
            self.handle.check(oz.lib.ozmm_gemm_slices_strided(
                self.handle.h, m, n, p, k, beta_bits, 0, a_slices.data_ptr(), a_slices.stride(1),
                a_slices.stride(0), mu.data_ptr(), b_slices.data_ptr(), b_slices.stride(1),
                b_slices.stride(0), nu.data_ptr(), alpha, beta, c.data_ptr(), c.stride(0),
                ctypes.byref(opt)))
        else:
            self.handle.check(oz.lib.ozmm_gemm_slices_offset(
                self.handle.h, m, n, p, k, beta_bits, 0, a_slices.data_ptr(), a_slices.stride(1),
                a_slices.stride(0), mu.data_ptr(), lsa.data_ptr(), lsa.stride(1), lsa.stride(0),
                b_slices.data_ptr(), b_slices.stride(1), b_slices.stride(0), nu.data_ptr(),
                lsb.data_ptr(), lsb.stride(1), lsb.stride(0), alpha, beta, c.data_ptr(),
                c.stride(0), ctypes.byref(opt)))


def _new_group(ranks):
    """Row / column communicator.  Under NCCL its stream is high priority, so the
    gather kernels take SMs ahead of the GEMM's next CTAs as they free up."""
    if dist.get_backend() == "nccl":
        opts = dist.ProcessGroupNCCL.Options()
        opts.is_high_priority_stream = True
        return dist.new_group(ranks, pg_options=opts)
    return dist.new_group(ranks)


def _other_ranges(total: int, own0: int, own: int):
    """[0, total) minus [own0, own0 + own), as up to two (start, stop) ranges."""
    return [(a, b) for a, b in ((0, own0), (own0 + own, total)) if b > a]


def _pieces(total: int, size: int):
    """[0, total) in consecutive pieces of `size` (the last one shorter)."""
    return [(a, min(a + size, total)) for a in range(0, total, size)]


class Grid2DGemm:
    """Sharded emulated DGEMM over a Pr x Pc rank grid.

    Buffers are allocated once; ``step(a_rows, b_cols, c_block)`` runs one
    emulated GEMM on this rank's shard:
      a_rows: op(A) rows [a_row0, a_row0 + ms) -- (ms x n), or its transpose
              (n x ms) when transa;
      b_cols: op(B) columns [b_col0, b_col0 + ps) -- (n x ps), or (ps x n) when
              transb;
      c_block: C block (mr x pcols), overwritten with alpha*D + beta*C.
    """

    def __init__(self, m, n, p, k, *, world=None, rank=None, backend=None, transa=False,
                 transb=False, group_factory=None, all_gather=None):
        self.world = world if world is not None else dist.get_world_size()
        self.rank = rank if rank is not None else dist.get_rank()
        self.L = make_layout(m, n, p, self.world, self.rank)
        self.k = k
        self.transa, self.transb = transa, transb
        # all_gather(out, inp, group) -> work with .wait(); injectable for tests
        self._all_gather = all_gather or (lambda out, inp, group: dist.all_gather_into_tensor(
            out, inp, group=group, async_op=True))
        from .ozmm import compute_beta, slice_ld  # closed forms (host)
        self.beta_bits = compute_beta(n)
        self.lds = slice_ld(n)
        self.backend = backend
        L = self.L
        # every rank must create every group, in the same order
        make = group_factory or _new_group
        self.row_group = self.col_group = None
        for gr in range(L.pr):
            ranks = [gr * L.pc + gc for gc in range(L.pc)]
            g = make(ranks)
            if gr == L.gr:
                self.row_group = g
        for gc in range(L.pc):
            ranks = [gr * L.pc + gc for gr in range(L.pr)]
            g = make(ranks)
            if gc == L.gc:
                self.col_group = g
        be = backend
        self.a_loc = be.empty((k, L.ms, self.lds), torch.int8)
        self.mu_loc = be.empty((L.ms,), torch.float64)
        self.b_loc = be.empty((k, L.ps, self.lds), torch.int8)
        self.nu_loc = be.empty((L.ps,), torch.float64)
        # a rank alone in its row (column) group slices the whole panel itself
        if L.pc == 1:
            self.a_pan, self.mu_pan = self.a_loc, self.mu_loc
        else:
            self.a_pan = be.empty((k, L.mr, self.lds), torch.int8)
            self.mu_pan = be.empty((L.mr,), torch.float64)
        if L.pr == 1:
            self.b_pan, self.nu_pan = self.b_loc, self.nu_loc
        else:
            self.b_pan = be.empty((k, L.pcols, self.lds), torch.int8)
            self.nu_pan = be.empty((L.pcols,), torch.float64)
        # offset-binary planes travel with their int32 line sums, [lines][k] so that
        # one all-gather along the lines moves them
        self.offset = bool(getattr(be, "offset_planes", False))
        self.lsa_loc = self.lsa_pan = self.lsb_loc = self.lsb_pan = None
        if self.offset:
            self.lsa_loc = be.empty((L.ms, k), torch.int32)
            self.lsb_loc = be.empty((L.ps, k), torch.int32)
            self.lsa_pan = self.lsa_loc if L.pc == 1 else be.empty((L.mr, k), torch.int32)
            self.lsb_pan = self.lsb_loc if L.pr == 1 else be.empty((L.pcols, k), torch.int32)

    def _gather(self, out, inp, group, nranks):
        if nranks > 1:
            return self._all_gather(out, inp, group)
        return None

    @staticmethod
    def _wait(works):
        for w in works:
            if w is not None:
                w.wait()

    def _check_range_across_grid(self):
        L, be = self.L, self.backend
        flag = be.empty((1,), torch.int32)
        flag.fill_(be.range_error())
        for group, nr in ((self.row_group, L.pc), (self.col_group, L.pr)):
            if nr > 1:
                out = be.empty((nr,), torch.int32)
                self._wait([self._gather(out, flag, group, nr)])
                flag.fill_(int(out.max().item()))
        if int(flag.item()):
            raise OverflowError("split: a rank of the grid saw a line magnitude too large for "
                                "shift extraction (>= 2^921)")

    def step(self, a_rows, b_cols, c_block, alpha=1.0, beta=0.0, ready=None,
             c_write_only=False, c_host=None, sync_check=False):
        """One sharded emulated GEMM.  The slice-panel all-gathers run while the
        GEMM works on what is already local, in three strip launches:
          G1  own A rows x own B columns     -- needs no communication;
          G2  own A rows x the other columns -- after the B (column-group) gather;
          G3  the other rows x all columns   -- after the A (row-group) gather.
        Every C entry is still produced by exactly one fused launch from the same
        slices and shifts, so the result is bit-identical to one GPU.

        ready: optional {'a', 'b', 'c'} -> CUDA event of the copy that fills
        a_rows / b_cols / c_block, for callers that stream the inputs in: each
        split waits only for its own operand and the GEMMs for C, so the
        slicing and gathers overlap the rest of the upload.  ready['a'] may also
        be a list of (row0, row1, event) panels of a_rows (not transa): B is then
        split first, each A panel as soon as it lands, and the first strip runs
        per panel (upload B first, then A panel by panel).
        c_write_only: C is not read (beta == 0 and a finite C, where fl(beta*c)
        = 0), so the caller need not upload it.
        c_host: optional (pinned) host tensor shaped like c_block.  Each finished
        full-width row range of C goes back on the backend's copy stream as soon
        as the strips that write it are done: the own rows after G1 and G2, the
        other rows per peer piece of G3 (pieces alternate between two streams so
        one's last wave overlaps the next one's first).  Only the last piece's
        D2H trails the GEMM.  The current stream waits for the copies.
        sync_check: the reference's throw-before-write across the grid.  After the
        local splits every rank reads its range flag (a synchronisation), the
        flags are max-reduced over the grid by two tiny all-gathers (row group,
        then column group), and EVERY rank raises OverflowError before any GEMM
        when any rank saw a line max >= 2^921; C is left untouched.  Without it
        the flag stays in the backend (Backend.range_error / ozmm_sync_status)."""
        L, k = self.L, self.k
        be = self.backend
        off = self.offset
        ready = ready or {}
        # OZMM_GRID_TRACE=1 (diagnostics, CUDA only): timing events after each
        # split / strip / copy, printed after a synchronize at the end of the step
        marks = [] if os.environ.get("OZMM_GRID_TRACE") == "1" else None

        def mark(name):
            if marks is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                marks.append((name, e))
        mark("start")

        def wait(key):
            if ready.get(key) is not None:
                torch.cuda.current_stream().wait_event(ready[key])
        ls = (lambda *a: dict(lsum=a[0])) if off else (lambda *a: {})
        a_panels = ready.get("a") if isinstance(ready.get("a"), (list, tuple)) else None
        if a_panels is not None and self.transa:
            raise ValueError("A panels need row-major op(A) (transa=False)")

        def split_b():
            wait("b")
            be.split(b_cols, k, "R", self.transb, self.beta_bits, self.b_loc, self.nu_loc,
                     **ls(self.lsb_loc))
            mark("split B")
        def gather_b():  # B first: it unblocks G2; group g needs slice planes <= g-1
            wb = [self._gather(self.b_pan[s], self.b_loc[s], self.col_group, L.pr)
                  for s in range(k)]
            wb.append(self._gather(self.nu_pan, self.nu_loc, self.col_group, L.pr))
            if off:
                wb.append(self._gather(self.lsb_pan, self.lsb_loc, self.col_group, L.pr))
            return wb
        a_split = []  # per A panel: (row0, row1, event after its split) when panelled
        if a_panels is None:
            wait("a")
            be.split(a_rows, k, "L", self.transa, self.beta_bits, self.a_loc, self.mu_loc,
                     **ls(self.lsa_loc))
            mark("split A")
            split_b()
            wb = gather_b()
        else:
            split_b()
            wb = gather_b()  # before the A panels: the collective waits on this stream

        if sync_check and a_panels is None:
            self._check_range_across_grid()

        def gather_a():
            wa = [self._gather(self.a_pan[s], self.a_loc[s], self.row_group, L.pc)
                  for s in range(k)]
            wa.append(self._gather(self.mu_pan, self.mu_loc, self.row_group, L.pc))
            if off:
                wa.append(self._gather(self.lsa_pan, self.lsa_loc, self.row_group, L.pc))
            return wa
        if a_panels is None:
            wa = gather_a()
        else:
            # the A panels are split on their own stream (the strips on the main
            # and side streams wait per panel), and A's gather follows the last one
            sp = be.split_stream()
            with torch.cuda.stream(sp):
                for lo, hi, ev in a_panels:
                    sp.wait_event(ev)
                    be.split(a_rows[lo:hi], k, "L", False, self.beta_bits, self.a_loc[:, lo:hi],
                             self.mu_loc[lo:hi], **ls(self.lsa_loc[lo:hi] if off else None))
                    a_split.append((lo, hi, torch.cuda.Event()))
                    a_split[-1][2].record(sp)
                    mark(f"split A {lo}:{hi}")
                if sync_check:  # after the last panel: A's lines are checked too
                    self._check_range_across_grid()
                wa = gather_a()

        def sums(a_sl, b_sl):  # line sums of the operand rows / columns a strip reads
            kw = dict(lsa=a_sl, lsb=b_sl) if off else {}
            if c_write_only:
                kw["c_write_only"] = True
            return kw
        r0, c0 = L.gc * L.ms, L.gr * L.ps  # own rows / columns inside the C block
        g = (L.n, k, self.beta_bits)
        own_rows = c_block[r0:r0 + L.ms]
        side = getattr(be, "side_stream", None)
        if not c_write_only:
            wait("c")  # C block landed (the side stream forks from here)
        out_s = be.copy_stream() if c_host is not None else None
        cur = torch.cuda.current_stream() if out_s is not None else None
        # streaming C back: the own rows go in pieces too (G1 / G2 per piece)
        if a_split:
            own = [(lo, hi) for lo, hi, _ in a_split]
        else:
            own = [(0, L.ms)] if out_s is None else _pieces(L.ms, max(256, L.ms // 4))

        def send(lo, hi, waits):  # D2H of C rows [lo, hi) once `waits` are done
            for w in waits:
                if isinstance(w, torch.cuda.Event):
                    out_s.wait_event(w)
                else:
                    out_s.wait_stream(w)
            with torch.cuda.stream(out_s):
                c_host[lo:hi].copy_(c_block[lo:hi], non_blocking=True)
                mark(f"D2H {lo}:{hi}")

        def g1(lo, hi):  # own rows x own columns: no communication
            be.gemm(hi - lo, g[0], L.ps, k, g[2], self.a_loc[:, lo:hi], self.mu_loc[lo:hi],
                    self.b_loc, self.nu_loc, alpha, beta, own_rows[lo:hi, c0:c0 + L.ps],
                    **sums(self.lsa_loc[lo:hi] if off else None, self.lsb_loc))
            mark(f"G1 {lo}:{hi}")

        def g2(lo, hi):  # own rows x the other columns: after the B gather
            for clo, chi in _other_ranges(L.pcols, c0, L.ps):
                be.gemm(hi - lo, g[0], chi - clo, k, g[2], self.a_loc[:, lo:hi], self.mu_loc[lo:hi],
                        self.b_pan[:, clo:chi], self.nu_pan[clo:chi], alpha, beta,
                        own_rows[lo:hi, clo:chi],
                        **sums(self.lsa_loc[lo:hi] if off else None,
                               self.lsb_pan[clo:chi] if off else None))
            mark(f"G2 {lo}:{hi}")
        if side and (a_split or out_s is not None):
            # per piece of the own rows: G1 and G2 back to back, pieces alternating
            # between the main and the side stream, so the own rows finish (and go
            # back) piece by piece while the next piece's first wave fills the SMs
            forked = torch.cuda.Event()
            forked.record()  # splits, B gather and C's arrival queued on the main stream
            for i, (lo, hi) in enumerate(own):
                st = be.side_stream(after_current=False) if i % 2 else contextlib.nullcontext()
                with st:
                    if i % 2:
                        torch.cuda.current_stream().wait_event(forked)
                    if a_split:
                        torch.cuda.current_stream().wait_event(a_split[i][2])
                    g1(lo, hi)
                    self._wait(wb)
                    g2(lo, hi)
                    if out_s is not None:
                        send(r0 + lo, r0 + hi, [torch.cuda.current_stream()])
        else:
            g1_done = []
            with side() if side else contextlib.nullcontext():
                for lo, hi in own:
                    if a_split:
                        torch.cuda.current_stream().wait_event(a_split[len(g1_done)][2])
                    g1(lo, hi)
                    g1_done.append(torch.cuda.Event() if out_s is not None else None)
                    if out_s is not None:
                        g1_done[-1].record()
            self._wait(wb)
            for i, (lo, hi) in enumerate(own):
                g2(lo, hi)
                if out_s is not None:
                    send(r0 + lo, r0 + hi, [cur, g1_done[i]])
        self._wait(wa)
        gathered = torch.cuda.Event() if out_s is not None and side else None
        if gathered is not None:
            gathered.record(cur)

        def g3(lo, hi):
            be.gemm(hi - lo, g[0], L.pcols, k, g[2], self.a_pan[:, lo:hi], self.mu_pan[lo:hi],
                    self.b_pan, self.nu_pan, alpha, beta, c_block[lo:hi],
                    **sums(self.lsa_pan[lo:hi] if off else None, self.lsb_pan))
            mark(f"G3 {lo}:{hi}")
        if out_s is None:
            for lo, hi in _other_ranges(L.mr, r0, L.ms):
                g3(lo, hi)
        else:
            # half a peer's rows per piece: a shorter D2H tail (grid_g3_split.txt:
            # 2x2 41 -> 38.8 ms, 2x4 21.6 -> 21.2 ms); OZMM_GRID_G3_SPLIT overrides
            size = max(256, L.ms // int(os.environ.get("OZMM_GRID_G3_SPLIT", "2")))
            pieces = [(a, min(a + size, hi)) for lo, hi in _other_ranges(L.mr, r0, L.ms)
                      for a in range(lo, hi, size)]
            for i, (lo, hi) in enumerate(pieces):
                if i % 2 and side:
                    with be.side_stream(after_current=False):
                        sst = torch.cuda.current_stream()
                        sst.wait_event(gathered)  # gathers done, not piece i-1
                        g3(lo, hi)
                    send(lo, hi, [sst])
                else:
                    g3(lo, hi)
                    send(lo, hi, [cur])
        if side:
            be.join_side()
        if out_s is not None:
            cur.wait_stream(out_s)
        if marks is not None:
            mark("end")
            torch.cuda.synchronize()
            t0 = marks[0][1]
            print("grid trace:", ", ".join(f"{n} {t0.elapsed_time(e):.1f}" for n, e in marks),
                  flush=True)
        return c_block


class NativeGrid2D:
    """The same 2-D partition through the C ABI's native entry (ozmm_dgemm_2d,
    csrc/ozmm_grid.cpp): splits, in-place all-gathers and the three strips are
    orchestrated in C++ on the handle's stream.  The collective is NCCL -- rank 0
    makes the id (ozmm_nccl_unique_id) and torch.distributed broadcasts it -- or
    `hook`, an ozmm.ALLGATHER_FN (the single-GPU tests emulate ranks with it).
    The shard arguments of step() are those of Grid2DGemm.step."""

    def __init__(self, m: int, n: int, p: int, k: int, world: int | None = None,
                 rank: int | None = None, device: int = 0, transa: bool = False,
                 transb: bool = False, hook=None):
        from . import ozmm
        self.oz = ozmm
        if world is None:
            world = dist.get_world_size() if dist.is_initialized() else 1
        if rank is None:
            rank = dist.get_rank() if dist.is_initialized() else 0
        self.m, self.n, self.p, self.k = m, n, p, k
        self.transa, self.transb = transa, transb
        self.L = make_layout(m, n, p, world, rank)
        self.device = torch.device("cuda", device)
        self.handle = ozmm.Handle(device)
        self._hook = hook  # keep the ctypes callback alive
        nid = None
        if world > 1 and hook is None:
            buf = (ctypes.c_char * 128)()
            if rank == 0:
                self._check(ozmm.lib.ozmm_nccl_unique_id(buf))
            obj = [bytes(buf)]
            dist.broadcast_object_list(obj, src=0)
            nid = (ctypes.c_char * 128).from_buffer_copy(obj[0])
        g = ctypes.c_void_p()
        self._check(ozmm.lib.ozmm_grid_create(self.handle.h, device, world, rank, nid,
                                              ctypes.cast(hook, ctypes.c_void_p) if hook else None,
                                              None, ctypes.byref(g)))
        self.g = g

    def _check(self, rc):
        # OZMM_ERR_RANGE -> OverflowError on every rank (the grid-wide check), the
        # other codes as in ozmm
        if rc != 0:
            self.oz._raise(rc, f"ozmm grid: {self.oz.lib.ozmm_grid_last_error().decode()}")

    def step(self, a_rows, b_cols, c_block, alpha=1.0, beta=0.0):
        self.handle.set_stream(torch.cuda.current_stream(self.device).cuda_stream)
        self._check(self.oz.lib.ozmm_dgemm_2d(
            self.g, b"T" if self.transa else b"N", b"T" if self.transb else b"N",
            self.m, self.n, self.p, alpha, a_rows.data_ptr(), a_rows.stride(0),
            b_cols.data_ptr(), b_cols.stride(0), beta, c_block.data_ptr(), c_block.stride(0),
            self.k))
        return c_block

    def close(self):
        if getattr(self, "g", None):
            self.oz.lib.ozmm_grid_destroy(self.g)
            self.g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
