"""Python mirror of the reference ``ozmm`` API over the B200 C ABI.

Same names, argument meaning and error behaviour as the reference's
operator API (/root/reference/proj/include/ozmm/scheme.hpp):

=======================  ==================================================
``ozaki_gemm``            scheme.hpp:92-95  -> ozmm_dgemm_ex / _host
``ozaki_gemm_ex``         scheme.hpp:96-98  (returns OzakiResult)
``ozaki_mm``              scheme.hpp:89-90  (alpha = 1, beta = 0)
``config_for``            scheme.cpp:137-159 (only ozIMMU_H runs on the GPU)
``compute_beta``          split.cpp:211-216
``compute_r``             int_gemm.cpp:253-258
``op_counts[_with_r]``    scheme.cpp:176-188
``split_rn_const_shift``  split.cpp:233-237 (K1 slicer on the device)
``gen_phi_matrix``        generate.cpp:11-29 (host, bit-identical)
=======================  ==================================================

Exceptions follow the reference: ``ConfigError`` (a ``ValueError``, like the
reference's ``std::invalid_argument`` subclass), ``ValueError`` for
argument errors, ``OverflowError`` for row magnitudes >= 2^921
(std::overflow_error, split.cpp:124-125) and ``Int32OverflowError`` (an
``OverflowError``) for an INT32 chunk overflow in ``OverflowMode.Checked``
(the reference's ``OverflowError``, int_gemm.hpp:15-26).  Both are raised
before C is written, on the host path and -- by default (``sync_check=True``)
-- on the device path too.

Operands may be numpy arrays (host, reference semantics: a NEW result is
returned and C is untouched) or CUDA float64 torch tensors (device path,
stream-ordered on the current torch stream; also returns a new tensor unless
``out=`` is given).  The library ``libozmm_b200.so`` is REQUIRED: there is no
CPU fallback and importing this module without it raises.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
import threading
from dataclasses import dataclass, field

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libozmm_b200.so")

OZMM_OK, OZMM_ERR_ARG, OZMM_ERR_CONFIG, OZMM_ERR_RANGE, OZMM_ERR_OVERFLOW = 0, 1, 2, 3, 4
OZMM_ERR_CUDA, OZMM_ERR_NCCL, OZMM_ERR_UNSUPPORTED = 5, 6, 7


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2409_13313_b200.build` "
            "(the emulated DGEMM has no CPU fallback)")
    return C.CDLL(LIB_PATH)


lib = _load()

_i64, _dp, _vp = C.c_int64, C.POINTER(C.c_double), C.c_void_p


class Counts(C.Structure):
    _fields_ = [("int8_gemms", C.c_int64), ("fp64_flushes", C.c_int64), ("r", C.c_int64),
                ("w", C.c_int64)]


class Timings(C.Structure):
    _fields_ = [("split_a", C.c_double), ("split_b", C.c_double), ("int_gemm", C.c_double),
                ("accum_fp64", C.c_double), ("copy", C.c_double)]


class Options(C.Structure):
    _fields_ = [("force_beta", C.c_int), ("force_r", C.c_int64), ("timings", C.c_int),
                ("sync_check", C.c_int), ("chunk_dump", C.c_void_p), ("tile_n", C.c_int),
                ("cta_pair", C.c_int), ("method", C.c_int), ("signed_slices", C.c_int),
                ("c_write_only", C.c_int), ("overflow_wrap", C.c_int), ("kpair", C.c_int),
                ("stages", C.c_int), ("host_panels", C.c_int), ("col_split", C.c_int),
                ("host_staging", C.c_int), ("host_threads", C.c_int)]


_SIG = {
    "ozmm_create": ([C.POINTER(C.c_void_p), C.c_int], C.c_int),
    "ozmm_destroy": ([_vp], C.c_int),
    "ozmm_set_stream": ([_vp, _vp], C.c_int),
    "ozmm_last_error": ([_vp], C.c_char_p),
    "ozmm_status_string": ([C.c_int], C.c_char_p),
    "ozmm_sync_status": ([_vp, C.POINTER(C.c_int)], C.c_int),
    "ozmm_workspace_bytes": ([_vp], C.c_size_t),
    "ozmm_compute_beta": ([_i64, C.POINTER(C.c_int)], C.c_int),
    "ozmm_compute_r": ([_i64, C.c_int, C.POINTER(_i64)], C.c_int),
    "ozmm_op_counts": ([C.c_int, _i64, C.POINTER(Counts)], C.c_int),
    "ozmm_dgemm": ([_vp, C.c_char, C.c_char, _i64, _i64, _i64, C.c_double, _vp, _i64, _vp, _i64,
                    C.c_double, _vp, _i64, C.c_int], C.c_int),
    "ozmm_dgemm_ex": ([_vp, C.c_char, C.c_char, _i64, _i64, _i64, C.c_double, _vp, _i64, _vp,
                       _i64, C.c_double, _vp, _i64, C.c_int, C.POINTER(Options),
                       C.POINTER(Counts), C.POINTER(Timings)], C.c_int),
    "ozmm_dgemm_host": ([_vp, C.c_char, C.c_char, _i64, _i64, _i64, C.c_double, _vp, _i64, _vp,
                         _i64, C.c_double, _vp, _i64, C.c_int, C.POINTER(Options),
                         C.POINTER(Counts), C.POINTER(Timings)], C.c_int),
    "ozmm_dgemm_host_out": ([_vp, C.c_char, C.c_char, _i64, _i64, _i64, C.c_double, _vp, _i64,
                             _vp, _i64, C.c_double, _vp, _i64, _vp, _i64, C.c_int,
                             C.POINTER(Options), C.POINTER(Counts), C.POINTER(Timings)], C.c_int),
    "ozmm_slice_ld": ([_i64], _i64),
    "ozmm_split": ([_vp, C.c_char, C.c_char, _i64, _i64, _vp, _i64, C.c_int, C.c_int, _vp, _i64,
                    _vp], C.c_int),
    "ozmm_split_ex": ([_vp, C.c_char, C.c_char, _i64, _i64, _vp, _i64, C.c_int, C.c_int, C.c_int,
                       _vp, _i64, _vp], C.c_int),
    "ozmm_split_host": ([_vp, C.c_char, C.c_char, _i64, _i64, _vp, _i64, C.c_int, C.c_int, C.c_int,
                         _vp, _vp, _vp], C.c_int),
    "ozmm_gemm_slices": ([_vp, _i64, _i64, _i64, C.c_int, C.c_int, _i64, _vp, _i64, _vp, _vp,
                          _i64, _vp, C.c_double, C.c_double, _vp, _i64, C.POINTER(Options)],
                         C.c_int),
    "ozmm_gemm_slices_strided": ([_vp, _i64, _i64, _i64, C.c_int, C.c_int, _i64, _vp, _i64, _i64,
                                  _vp, _vp, _i64, _i64, _vp, C.c_double, C.c_double, _vp, _i64,
                                  C.POINTER(Options)], C.c_int),
    "ozmm_split_offset": ([_vp, C.c_char, C.c_char, _i64, _i64, _vp, _i64, C.c_int, C.c_int,
                           _vp, _i64, _vp, _vp, _i64, _i64], C.c_int),
    "ozmm_split_offset_strided": ([_vp, C.c_char, C.c_char, _i64, _i64, _vp, _i64, C.c_int,
                                   C.c_int, _vp, _i64, _i64, _vp, _vp, _i64, _i64], C.c_int),
    "ozmm_gemm_slices_offset": ([_vp, _i64, _i64, _i64, C.c_int, C.c_int, _i64, _vp, _i64, _i64,
                                 _vp, _vp, _i64, _i64, _vp, _i64, _i64, _vp, _vp, _i64, _i64,
                                 C.c_double, C.c_double, _vp, _i64, C.POINTER(Options)], C.c_int),
    "ozmm_gen_phi_block": ([_i64, _i64, C.c_double, C.c_uint64, _i64, _i64, _i64, _i64, _vp,
                            _i64], C.c_int),
    "ozmm_counter_hash": ([C.c_uint64, C.c_uint64], C.c_uint64),
    "ozmm_get_stream": ([_vp, C.POINTER(C.c_void_p)], C.c_int),
    # 2-D grid (ozmm_dgemm_2d); the hook argument is an ALLGATHER_FN or None
    "ozmm_grid_shape": ([C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)], C.c_int),
    "ozmm_nccl_unique_id": ([_vp], C.c_int),
    "ozmm_grid_create": ([_vp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, C.POINTER(C.c_void_p)],
                         C.c_int),
    "ozmm_grid_destroy": ([_vp], C.c_int),
    "ozmm_grid_coords": ([_vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                          C.POINTER(C.c_int)], C.c_int),
    "ozmm_grid_last_error": ([], C.c_char_p),
    "ozmm_dgemm_2d": ([_vp, C.c_char, C.c_char, _i64, _i64, _i64, C.c_double, _vp, _i64, _vp,
                       _i64, C.c_double, _vp, _i64, C.c_int], C.c_int),
    "ozmm_debug_schedule": ([C.c_int, _i64, C.c_int, C.c_int, _vp, C.c_int, _vp], C.c_int),
}
for _name, (_args, _res) in _SIG.items():
    _f = getattr(lib, _name)
    _f.argtypes, _f.restype = _args, _res

EXPORTED_SYMBOLS = tuple(_SIG)

# ozmm_allgather_fn (include/ozmm_b200.h): (ctx, group, send, recv, bytes, stream) -> int
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, _vp, C.c_int, _vp, _vp, _i64, _vp)


# ---------------------------------------------------------------- errors
class ConfigError(ValueError):
    """Inconsistent scheme configuration (reference ConfigError, scheme.hpp:20-22)."""


class OzmmCudaError(RuntimeError):
    """CUDA / launch failure inside the library."""


class Int32OverflowError(OverflowError):
    """INT32 chunk overflow in OverflowMode.Checked (the reference's
    OverflowError, int_gemm.hpp:15-26); reachable only with force_beta / force_r."""


def _raise(code: int, msg: str):
    if code == OZMM_ERR_CONFIG:
        raise ConfigError(msg)
    if code == OZMM_ERR_ARG:
        raise ValueError(msg)
    if code == OZMM_ERR_RANGE:
        raise OverflowError(msg)
    if code == OZMM_ERR_OVERFLOW:
        raise Int32OverflowError(msg)
    if code == OZMM_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise OzmmCudaError(f"[{code}] {msg}")


def _check(code: int, handle=None):
    if code != OZMM_OK:
        _raise(code, (lib.ozmm_last_error(handle) or b"").decode())


# ---------------------------------------------------------- config types
class Method(enum.Enum):
    ozIMMU = "ozIMMU"
    ozIMMU_RN = "ozIMMU_RN"
    ozIMMU_EF = "ozIMMU_EF"
    ozIMMU_H = "ozIMMU_H"


class SliceStrategy(enum.Enum):
    BitMask = 0
    RoundNearestPerSlice = 1
    RoundNearestConstShift = 2


class Accumulation(enum.Enum):
    PerProduct = 0
    Groupwise = 1
    GroupwiseSimple = 2


class OverflowMode(enum.Enum):
    """int_gemm.hpp:13."""
    Checked = 0
    Wrapping = 1


@dataclass
class SchemeConfig:
    """scheme.hpp:24-31.  Defaults as the reference (k = 8)."""
    k: int = 8
    strategy: SliceStrategy = SliceStrategy.BitMask
    accumulation: Accumulation = Accumulation.PerProduct
    overflow: OverflowMode = OverflowMode.Checked
    force_beta: int = 0
    force_r: int = 0


def config_for(method: Method | str, k: int) -> SchemeConfig:
    """Method presets, scheme.cpp:137-159."""
    method = Method(method) if isinstance(method, str) else method
    strat, acc = {
        Method.ozIMMU: (SliceStrategy.BitMask, Accumulation.PerProduct),
        Method.ozIMMU_RN: (SliceStrategy.RoundNearestPerSlice, Accumulation.PerProduct),
        Method.ozIMMU_EF: (SliceStrategy.BitMask, Accumulation.Groupwise),
        Method.ozIMMU_H: (SliceStrategy.RoundNearestConstShift, Accumulation.Groupwise),
    }[method]
    return SchemeConfig(k=k, strategy=strat, accumulation=acc)


@dataclass
class OpCounts:
    int8_gemms: int = 0
    fp64_flushes: int = 0
    r: int = 0
    w: int = 0


@dataclass
class PhaseTimings:
    split_a: float = 0.0
    split_b: float = 0.0
    int_gemm: float = 0.0
    accum_fp64: float = 0.0
    copy: float = 0.0


@dataclass
class OzakiResult:
    d: object
    counts: OpCounts = field(default_factory=OpCounts)
    timings: PhaseTimings = field(default_factory=PhaseTimings)


# ------------------------------------------------------------ closed forms
def compute_beta(n: int) -> int:
    out = C.c_int()
    _check(lib.ozmm_compute_beta(n, C.byref(out)))
    return out.value


def compute_r(n: int, beta: int) -> int:
    out = _i64()
    _check(lib.ozmm_compute_r(n, beta, C.byref(out)))
    return out.value


def op_counts_with_r(k: int, r: int) -> OpCounts:
    c = Counts()
    _check(lib.ozmm_op_counts(k, r, C.byref(c)))
    return OpCounts(c.int8_gemms, c.fp64_flushes, c.r, c.w)


def op_counts(k: int, n: int) -> OpCounts:
    """Group-wise counts for inner dimension n (scheme.cpp:186-188)."""
    return op_counts_with_r(k, compute_r(n, compute_beta(n)))


def slice_ld(n: int) -> int:
    return int(lib.ozmm_slice_ld(n))


def debug_schedule(k: int, r: int, cta_pair: int = 0, tile_n: int = 0):
    """The GEMM kernel's host schedule: (rows[products, 8], info dict)."""
    cap = k * (k + 1) // 2
    rows = np.zeros((cap, 8), np.int32)
    info = np.zeros(7, np.int32)
    _check(lib.ozmm_debug_schedule(k, r, cta_pair, tile_n, rows.ctypes.data, cap,
                                   info.ctypes.data))
    keys = ["products", "chunks", "batches", "passes", "stages", "a_slots", "b_slots"]
    return rows[: int(info[0])], dict(zip(keys, (int(v) for v in info)))


# --------------------------------------------------------------- handles
class Handle:
    """One library handle (workspace + stream) per device.  Not thread-safe:
    use one handle per host thread (include/ozmm_b200.h)."""

    def __init__(self, device: int = 0):
        self.device = device
        h = C.c_void_p()
        _check(lib.ozmm_create(C.byref(h), device))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib.ozmm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, code: int):
        _check(code, self.h)

    def set_stream(self, stream_ptr: int | None):
        self.check(lib.ozmm_set_stream(self.h, C.c_void_p(stream_ptr or 0)))

    def sync_status(self) -> bool:
        """Raise OverflowError for a pending range error; return the underflow flag."""
        uf = C.c_int()
        self.check(lib.ozmm_sync_status(self.h, C.byref(uf)))
        return bool(uf.value)

    @property
    def workspace_bytes(self) -> int:
        return int(lib.ozmm_workspace_bytes(self.h))


_tls = threading.local()


def default_handle(device: int = 0) -> Handle:
    hs = getattr(_tls, "handles", None)
    if hs is None:
        hs = _tls.handles = {}
    if device not in hs:
        hs[device] = Handle(device)
    return hs[device]


def _torch():
    import torch  # deferred: host-only use does not need torch
    return torch


def _is_cuda_tensor(x) -> bool:
    try:
        torch = _torch()
    except ImportError:
        return False
    return isinstance(x, torch.Tensor) and x.is_cuda


def _row_major(t) -> bool:
    """Row-major with unit column stride; a dimension of size 1 may carry any
    stride (numpy and torch leave such strides arbitrary)."""
    return t.dim() == 2 and (t.shape[1] == 1 or t.stride(1) == 1)


def _ld(t) -> int:
    """Leading dimension of a row-major 2-D tensor: its row stride, or the row
    length when there is a single row (the stride is then meaningless)."""
    return int(t.stride(0)) if t.shape[0] > 1 else max(1, int(t.shape[1]))


def _options(cfg: SchemeConfig | None, timings: bool = False, dump=None, tile_n: int = 0,
             sync_check: bool = False, cta_pair: int = 0, signed_slices: bool = False,
             kpair: int = 0, stages: int = 0, host_panels: int = 0,
             host_staging: int = 0, col_split: int = 0) -> Options:
    o = Options()
    if cfg is not None:
        o.force_beta = cfg.force_beta
        o.force_r = cfg.force_r
        o.method = _method_code(cfg)
        o.overflow_wrap = int(cfg.overflow == OverflowMode.Wrapping)
    o.kpair, o.stages, o.host_panels = kpair, stages, host_panels
    o.host_staging = host_staging
    o.col_split = col_split
    o.timings = int(timings)
    o.sync_check = int(sync_check)
    o.chunk_dump = dump.data_ptr() if dump is not None else None
    o.tile_n = tile_n
    o.cta_pair = cta_pair
    o.signed_slices = int(signed_slices)
    return o


# (strategy, accumulation) -> OZMM_METHOD_* (include/ozmm_b200.h)
_METHOD_CODES = {
    (SliceStrategy.RoundNearestConstShift, Accumulation.Groupwise): 0,        # ozIMMU_H
    (SliceStrategy.BitMask, Accumulation.PerProduct): 1,                      # ozIMMU
    (SliceStrategy.RoundNearestPerSlice, Accumulation.PerProduct): 2,         # ozIMMU_RN
    (SliceStrategy.BitMask, Accumulation.Groupwise): 3,                       # ozIMMU_EF
    (SliceStrategy.RoundNearestConstShift, Accumulation.PerProduct): 4,
    (SliceStrategy.RoundNearestConstShift, Accumulation.GroupwiseSimple): 5,
    (SliceStrategy.BitMask, Accumulation.GroupwiseSimple): 6,
}


def _method_code(cfg: SchemeConfig) -> int:
    return _METHOD_CODES[(cfg.strategy, cfg.accumulation)]


def _validate(cfg: SchemeConfig):
    # validate_config (scheme.cpp:161-174); the r >= k rule of GroupwiseSimple is
    # checked by the library once n is known.
    if cfg.k < 1:
        raise ConfigError("k must be >= 1")
    if cfg.strategy == SliceStrategy.RoundNearestPerSlice and \
            cfg.accumulation != Accumulation.PerProduct:
        raise ConfigError("per-slice round-to-nearest shifts are only valid with per-product "
                          "accumulation")
    if (cfg.strategy, cfg.accumulation) not in _METHOD_CODES:
        raise ConfigError(f"unsupported scheme {cfg.strategy.name} + {cfg.accumulation.name}")


def _to_result(counts: Counts, tim: Timings, d) -> OzakiResult:
    return OzakiResult(d, OpCounts(counts.int8_gemms, counts.fp64_flushes, counts.r, counts.w),
                       PhaseTimings(tim.split_a, tim.split_b, tim.int_gemm, tim.accum_fp64,
                                    tim.copy))


def ozaki_gemm_ex(alpha: float, a, b, beta: float, c, cfg: SchemeConfig | None = None, *,
                  transa: bool = False, transb: bool = False, handle: Handle | None = None,
                  out=None, timings: bool = True, chunk_dump=None,
                  tile_n: int = 0, signed_slices: bool = False, sync_check: bool = True,
                  kpair: int = 0, stages: int = 0, host_panels: int = 0,
                  cta_pair: int = 0, host_staging: int = 0, col_split: int = 0) -> OzakiResult:
    """Emulated DGEMM: alpha * op(A) op(B) + beta * C (scheme.cpp:274-291).

    Returns OzakiResult(d=new matrix, counts, timings); C is not modified
    unless it is passed as ``out`` too.  Shapes: op(A) m x n, op(B) n x p,
    C m x p, all row-major.  ``signed_slices`` keeps the reference's signed
    int8 planes inside the fused GEMM instead of the default offset-binary ones
    (same results; include/ozmm_b200.h).

    Device path: ``sync_check=True`` (default) waits for the splits and raises
    OverflowError for a line max >= 2^921 before the GEMM writes ``out``, like
    the reference's throw.  ``sync_check=False`` keeps the call fully
    stream-ordered (e.g. inside a CUDA graph); the range error then stays
    pending on the handle until ``Handle.sync_status()``.  ``kpair``,
    ``stages``, ``host_panels``, ``cta_pair``, ``col_split``: kernel tuning,
    same results (ozmm_options_t).  ``host_staging`` (host path): 0 = pageable arrays go
    through pinned slots (default), 1 = driver copies, 2 = stage everything.
    """
    cfg = cfg or config_for(Method.ozIMMU_H, 8)
    _validate(cfg)
    counts, tim = Counts(), Timings()
    dev = _is_cuda_tensor(a)
    if dev:
        torch = _torch()
        for t in (a, b, c):
            if not (_is_cuda_tensor(t) and t.dtype == torch.float64):
                raise ValueError("device path needs float64 CUDA tensors for A, B and C")
            if not _row_major(t):
                raise ValueError("operands must be row-major (unit column stride)")
        m, n = (a.shape[1], a.shape[0]) if transa else (a.shape[0], a.shape[1])
        nb, p = (b.shape[1], b.shape[0]) if transb else (b.shape[0], b.shape[1])
        if n != nb:
            raise ValueError("ozaki_mm: inner dimensions differ")
        if tuple(c.shape) != (m, p):
            raise ValueError("ozaki_gemm: C shape mismatch")
        h = handle or default_handle(a.device.index or 0)
        h.set_stream(torch.cuda.current_stream(a.device).cuda_stream)
        # C is read and written in place by the C ABI, which leaves it untouched on
        # every error; a distinct ``out`` is filled only after the call succeeded
        dst = c.clone() if out is None or out.data_ptr() != c.data_ptr() else out
        opt = _options(cfg, timings, chunk_dump, tile_n, sync_check=sync_check,
                       signed_slices=signed_slices, kpair=kpair, stages=stages,
                       cta_pair=cta_pair, col_split=col_split)
        h.check(lib.ozmm_dgemm_ex(h.h, b"T" if transa else b"N", b"T" if transb else b"N", m, n,
                                  p, alpha, a.data_ptr(), _ld(a), b.data_ptr(),
                                  _ld(b), beta, dst.data_ptr(), _ld(dst), cfg.k,
                                  C.byref(opt), C.byref(counts),
                                  C.byref(tim) if timings else None))
        if out is not None and dst is not out:
            out.copy_(dst)
            dst = out
        return _to_result(counts, tim, dst)
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    c = np.ascontiguousarray(c, dtype=np.float64)
    m, n = (a.shape[1], a.shape[0]) if transa else a.shape
    nb, p = (b.shape[1], b.shape[0]) if transb else b.shape
    if n != nb:
        raise ValueError("ozaki_mm: inner dimensions differ")
    if c.shape != (m, p):
        raise ValueError("ozaki_gemm: C shape mismatch")
    h = handle or default_handle(0)
    # in place only when ``out`` is C itself; otherwise the result goes to a new
    # array (ozmm_dgemm_host_out reads C and writes the result: no copy of C, as
    # the reference returns a new matrix) and a distinct ``out`` is filled after
    # success
    inplace = (out is not None and out.flags.c_contiguous and out.shape == c.shape
               and out.ctypes.data == c.ctypes.data)
    res = out if inplace else np.empty((m, p), np.float64)
    opt = _options(cfg, timings, None, tile_n, sync_check=True, signed_slices=signed_slices,
                   kpair=kpair, stages=stages, host_panels=host_panels, cta_pair=cta_pair,
                   host_staging=host_staging, col_split=col_split)
    h.set_stream(None)
    h.check(lib.ozmm_dgemm_host_out(h.h, b"T" if transa else b"N", b"T" if transb else b"N", m,
                                    n, p, alpha, a.ctypes.data, a.shape[1], b.ctypes.data,
                                    b.shape[1], beta, c.ctypes.data, p, res.ctypes.data, p, cfg.k,
                                    C.byref(opt), C.byref(counts),
                                    C.byref(tim) if timings else None))
    if out is not None and res is not out:
        np.copyto(out, res)
        res = out
    return _to_result(counts, tim, res)


def ozaki_gemm(alpha: float, a, b, beta: float, c, cfg: SchemeConfig | None = None, **kw):
    """scheme.cpp:293-296: the matrix of ozaki_gemm_ex."""
    return ozaki_gemm_ex(alpha, a, b, beta, c, cfg, **kw).d


def ozaki_mm(a, b, cfg: SchemeConfig | None = None, **kw) -> OzakiResult:
    """scheme.cpp:228-272: D = A B (alpha = 1, beta = 0 into zeros; bitwise equal)."""
    if _is_cuda_tensor(a):
        torch = _torch()
        m = a.shape[1] if kw.get("transa") else a.shape[0]
        p = b.shape[0] if kw.get("transb") else b.shape[1]
        c = torch.zeros((m, p), dtype=torch.float64, device=a.device)
    else:
        m = a.shape[1] if kw.get("transa") else a.shape[0]
        p = b.shape[0] if kw.get("transb") else b.shape[1]
        c = np.zeros((m, p), np.float64)
    return ozaki_gemm_ex(1.0, a, b, 0.0, c, cfg, out=c, **kw)


# ----------------------------------------------------------- slicer (K1)
@dataclass
class SplitMatrix:
    """Device split of one operand in the GEMM's K-major layout.

    slices: int8 [k][lines][lds] (Left: line = row of op(X); Right: line =
    column of op(X)), shift: float64 [lines] (const_shift, split.hpp:37)."""
    side: str
    k: int
    beta: int
    slices: object
    shift: object
    n: int

    def reference_layout(self):
        """Slices as the reference stores them: Left k x m x n, Right k x n x p."""
        s = self.slices[:, :, : self.n]
        return s if self.side == "L" else s.transpose(1, 2)


def split_rn_const_shift(x, k: int, side: str = "L", *, trans: bool = False, force_beta: int = 0,
                         handle: Handle | None = None) -> SplitMatrix:
    """RN constant-shift split on the GPU (split.cpp:233-237).

    side 'L': rows of op(X) (op(X) = lines x n); 'R': columns of op(X)
    (op(X) = n x lines).  x: float64 CUDA tensor, row-major."""
    torch = _torch()
    if not (_is_cuda_tensor(x) and x.dtype == torch.float64 and _row_major(x)):
        raise ValueError("split_rn_const_shift needs a row-major float64 CUDA tensor")
    side = side.upper()
    rows, cols = x.shape
    if side == "L":
        lines, n = (cols, rows) if trans else (rows, cols)
    else:
        n, lines = (cols, rows) if trans else (rows, cols)
    beta = force_beta or compute_beta(n)
    lds = slice_ld(n)
    h = handle or default_handle(x.device.index or 0)
    h.set_stream(torch.cuda.current_stream(x.device).cuda_stream)
    sl = torch.empty((k, lines, lds), dtype=torch.int8, device=x.device)
    sh = torch.empty((lines,), dtype=torch.float64, device=x.device)
    h.check(lib.ozmm_split(h.h, side.encode(), b"T" if trans else b"N", lines, n, x.data_ptr(),
                           _ld(x), k, beta, sl.data_ptr(), lds, sh.data_ptr()))
    return SplitMatrix(side, k, beta, sl, sh, n)


def split_dump(a, k: int, side: str = "L", strategy: SliceStrategy = SliceStrategy.RoundNearestConstShift,
               *, force_beta: int = 0, handle: Handle | None = None):
    """The reference's SplitMatrix of a host matrix, as dump_split writes it
    (split.cpp:254-270): ``(slices [k][rows][cols] int8, shift or units,
    residual [rows][cols])`` in the matrix's own layout, computed on the GPU
    (ozmm_split_host).  side 'L' splits rows, 'R' columns; ``shift`` is [lines]
    (const-shift strategies) or the per-slice units [k][lines]."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    rows, cols = a.shape
    side = side.upper()
    lines, n = (rows, cols) if side == "L" else (cols, rows)
    code = {SliceStrategy.RoundNearestConstShift: 0, SliceStrategy.BitMask: 1,
            SliceStrategy.RoundNearestPerSlice: 2}[SliceStrategy(strategy)]
    sl = np.empty((k, lines, n), np.int8)
    out = np.empty((k, lines) if code == 2 else (lines,), np.float64)
    res = np.empty((lines, n), np.float64)
    h = handle or default_handle(0)
    h.set_stream(None)
    h.check(lib.ozmm_split_host(h.h, side.encode(), b"N", lines, n, a.ctypes.data, cols, k,
                                force_beta, code, sl.ctypes.data, out.ctypes.data,
                                res.ctypes.data))
    if side == "R":  # line-major (columns) back to the matrix's layout (transpose_back, :175-180)
        sl = np.ascontiguousarray(sl.transpose(0, 2, 1))
        res = np.ascontiguousarray(res.T)
    return sl, out, res


def split(x, k: int, side: str = "L", strategy: SliceStrategy = SliceStrategy.RoundNearestConstShift,
          *, trans: bool = False, force_beta: int = 0, handle: Handle | None = None):
    """Any strategy (split_bitmask / split_round_nearest / split_rn_const_shift,
    split.cpp:223-237).  Returns SplitMatrix; for RoundNearestPerSlice its
    ``shift`` holds the per-slice units [k][lines] (slice_units, split.hpp:38)."""
    torch = _torch()
    if not (_is_cuda_tensor(x) and x.dtype == torch.float64 and _row_major(x)):
        raise ValueError("split needs a row-major float64 CUDA tensor")
    side = side.upper()
    rows, cols = x.shape
    if side == "L":
        lines, n = (cols, rows) if trans else (rows, cols)
    else:
        n, lines = (cols, rows) if trans else (rows, cols)
    beta = force_beta or compute_beta(n)
    lds = slice_ld(n)
    h = handle or default_handle(x.device.index or 0)
    h.set_stream(torch.cuda.current_stream(x.device).cuda_stream)
    code = {SliceStrategy.RoundNearestConstShift: 0, SliceStrategy.BitMask: 1,
            SliceStrategy.RoundNearestPerSlice: 2}[strategy]
    sl = torch.empty((k, lines, lds), dtype=torch.int8, device=x.device)
    out = torch.empty((k, lines) if code == 2 else (lines,), dtype=torch.float64,
                      device=x.device)
    h.check(lib.ozmm_split_ex(h.h, side.encode(), b"T" if trans else b"N", lines, n,
                              x.data_ptr(), _ld(x), k, beta, code, sl.data_ptr(), lds,
                              out.data_ptr()))
    return SplitMatrix(side, k, beta, sl, out, n)


def gemm_slices(sa: SplitMatrix, sb: SplitMatrix, alpha: float, beta: float, c, *, r: int = 0,
                handle: Handle | None = None, chunk_dump=None, tile_n: int = 0):
    """K2+K3 over already-split operands (in place on c)."""
    torch = _torch()
    if sa.k != sb.k or sa.beta != sb.beta or sa.n != sb.n:
        raise ConfigError("accumulate: slice counts / widths / inner dimensions differ")
    m, p = sa.slices.shape[1], sb.slices.shape[1]
    h = handle or default_handle(c.device.index or 0)
    h.set_stream(torch.cuda.current_stream(c.device).cuda_stream)
    opt = _options(None, False, chunk_dump, tile_n)
    h.check(lib.ozmm_gemm_slices(h.h, m, sa.n, p, sa.k, sa.beta, r, sa.slices.data_ptr(),
                                 sa.slices.shape[2], sa.shift.data_ptr(), sb.slices.data_ptr(),
                                 sb.slices.shape[2], sb.shift.data_ptr(), alpha, beta,
                                 c.data_ptr(), _ld(c), C.byref(opt)))
    return c


# --------------------------------------------------------- input generator
def counter_hash(seed: int, ctr: int) -> int:
    return int(lib.ozmm_counter_hash(seed, ctr))


def gen_phi_block(rows: int, cols: int, phi: float, seed: int, row0: int = 0,
                  nrows: int | None = None, col0: int = 0, ncols: int | None = None,
                  out: np.ndarray | None = None) -> np.ndarray:
    """Block of the global rows x cols phi matrix (generate.cpp:11-29)."""
    nrows = rows - row0 if nrows is None else nrows
    ncols = cols - col0 if ncols is None else ncols
    if out is None:
        out = np.empty((nrows, ncols), np.float64)
    assert out.dtype == np.float64 and out.flags.c_contiguous and out.shape == (nrows, ncols)
    code = lib.ozmm_gen_phi_block(rows, cols, phi, seed, row0, nrows, col0, ncols,
                                  out.ctypes.data, ncols)
    if code != OZMM_OK:
        raise ValueError("gen_phi_matrix: bad shape / phi / block")
    return out


def gen_phi_matrix(m: int, n: int, phi: float, seed: int) -> np.ndarray:
    return gen_phi_block(m, n, phi, seed)
