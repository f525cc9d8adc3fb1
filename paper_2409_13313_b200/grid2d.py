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

    def side_stream(self):
        """Context for the communication-free strip G1: a second stream that
        starts after the current one, so G2/G3 (which wait only on the gathers)
        fill the SMs G1's last partial wave leaves idle.  join_side() puts the
        current stream back behind it."""
        if not hasattr(self, "_side"):
            self._side = torch.cuda.Stream(self.device)
        cur = torch.cuda.current_stream(self.device)
        self._side.wait_stream(cur)
        return torch.cuda.stream(self._side)

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
        else:
            self.handle.check(oz.lib.ozmm_split_offset(*args, lsum.data_ptr(), lsum.stride(1),
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

    def step(self, a_rows, b_cols, c_block, alpha=1.0, beta=0.0, ready=None,
             c_write_only=False):
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
        slicing and gathers overlap the rest of the upload.
        c_write_only: C is not read (beta == 0 and a finite C, where fl(beta*c)
        = 0), so the caller need not upload it."""
        L, k = self.L, self.k
        be = self.backend
        off = self.offset
        ready = ready or {}

        def wait(key):
            if ready.get(key) is not None:
                torch.cuda.current_stream().wait_event(ready[key])
        ls = (lambda *a: dict(lsum=a[0])) if off else (lambda *a: {})
        wait("a")
        be.split(a_rows, k, "L", self.transa, self.beta_bits, self.a_loc, self.mu_loc,
                 **ls(self.lsa_loc))
        wait("b")
        be.split(b_cols, k, "R", self.transb, self.beta_bits, self.b_loc, self.nu_loc,
                 **ls(self.lsb_loc))
        # B first: it unblocks G2; group g of a GEMM needs slice planes <= g-1
        wb = [self._gather(self.b_pan[s], self.b_loc[s], self.col_group, L.pr) for s in range(k)]
        wb.append(self._gather(self.nu_pan, self.nu_loc, self.col_group, L.pr))
        wa = [self._gather(self.a_pan[s], self.a_loc[s], self.row_group, L.pc) for s in range(k)]
        wa.append(self._gather(self.mu_pan, self.mu_loc, self.row_group, L.pc))
        if off:
            wb.append(self._gather(self.lsb_pan, self.lsb_loc, self.col_group, L.pr))
            wa.append(self._gather(self.lsa_pan, self.lsa_loc, self.row_group, L.pc))

        def sums(a_sl, b_sl):  # line sums of the operand rows / columns a strip reads
            kw = dict(lsa=a_sl, lsb=b_sl) if off else {}
            if c_write_only:
                kw["c_write_only"] = True
            return kw
        r0, c0 = L.gc * L.ms, L.gr * L.ps  # own rows / columns inside the C block
        g = (L.n, k, self.beta_bits)
        own_rows = c_block[r0:r0 + L.ms]
        side = getattr(be, "side_stream", None)
        wait("c")  # C block landed (the side stream forks from here)
        with side() if side else contextlib.nullcontext():
            be.gemm(L.ms, g[0], L.ps, k, g[2], self.a_loc, self.mu_loc, self.b_loc, self.nu_loc,
                    alpha, beta, own_rows[:, c0:c0 + L.ps], **sums(self.lsa_loc, self.lsb_loc))
        self._wait(wb)
        for lo, hi in _other_ranges(L.pcols, c0, L.ps):
            be.gemm(L.ms, g[0], hi - lo, k, g[2], self.a_loc, self.mu_loc, self.b_pan[:, lo:hi],
                    self.nu_pan[lo:hi], alpha, beta, own_rows[:, lo:hi],
                    **sums(self.lsa_loc, self.lsb_pan[lo:hi] if off else None))
        self._wait(wa)
        for lo, hi in _other_ranges(L.mr, r0, L.ms):
            be.gemm(hi - lo, g[0], L.pcols, k, g[2], self.a_pan[:, lo:hi], self.mu_pan[lo:hi],
                    self.b_pan, self.nu_pan, alpha, beta, c_block[lo:hi],
                    **sums(self.lsa_pan[lo:hi] if off else None, self.lsb_pan))
        if side:
            be.join_side()
        return c_block
