"""ctypes loaders for the two CPU checkers -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline / reference
arm may import this module.  The product (paper_2409_13313_b200) never does.

* :class:`RefLib`  -- ``oracle/_ref/libozmm_ref.so``: the UNMODIFIED reference
  library (``/root/reference/proj/src``) compiled by ``oracle/Makefile`` with
  the in-repo Eigen-subset shim, behind ``oracle/ref_capi.cpp``.
* :class:`PortLib` -- ``oracle/liboracle_port.so``: the plain-C restatement
  ``oracle/ozmm_oracle.c`` (each function cites the reference file:line it
  follows).  Pinned against RefLib and against the golden fixtures under
  ``tests/golden`` (see tests/test_oracle.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libozmm_ref.so")
PORT_SO = os.path.join(HERE, "liboracle_port.so")

_i64 = C.c_int64
_dp = C.POINTER(C.c_double)
_i8p = C.POINTER(C.c_int8)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_ip = C.POINTER(C.c_int)

# Error codes shared by both checkers (mirroring include/ozmm_b200.h).
OK, ERR_ARG, ERR_CONFIG, ERR_RANGE, ERR_OVERFLOW = 0, 1, 2, 3, 4

METHODS = {"ozIMMU": 0, "ozIMMU_RN": 1, "ozIMMU_EF": 2, "ozIMMU_H": 3}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def build(quiet: bool = True) -> None:
    """Build both checkers (the reference one only where /root/reference exists)."""
    out = subprocess.run(["make", "-C", HERE, "all"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class Split:
    slices: np.ndarray     # (k, rows, cols) int8, in the matrix's own layout
    shift: np.ndarray      # (rows,) Left or (cols,) Right, float64 powers of two
    beta: int
    underflow: bool
    residual: np.ndarray | None = None


@dataclass
class Chunks:
    acc: np.ndarray        # (w, m, p) int32 chunk sums in flush order
    g: np.ndarray          # (w,) group index g = s + t
    s0: np.ndarray         # (w,) first A-slice index in the chunk
    s1: np.ndarray         # (w,) last A-slice index in the chunk


class _Base:
    prefix = ""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)
        self.path = path
        p = self.prefix
        L = self.lib
        getattr(L, p + "last_error").restype = C.c_char_p
        getattr(L, p + "compute_beta").argtypes = [_i64, _ip]
        getattr(L, p + "compute_r").argtypes = [_i64, C.c_int, _i64p]
        getattr(L, p + "op_counts_with_r").argtypes = [C.c_int, _i64, C.c_int, _i64p]
        getattr(L, p + "counter_hash").argtypes = [C.c_uint64, C.c_uint64]
        getattr(L, p + "counter_hash").restype = C.c_uint64
        getattr(L, p + "gen_phi_matrix").argtypes = [_i64, _i64, C.c_double, C.c_uint64, _dp]
        getattr(L, p + "gemm").argtypes = [C.c_int, C.c_int, C.c_int, _i64, C.c_int, C.c_double,
                                  _dp, _i64, _i64, _dp, _i64, C.c_double, _dp, _dp,
                                  _i64p, _dp]
        getattr(L, p + "split_rn_const_shift").argtypes = [_dp, _i64, _i64, C.c_int, C.c_int,
                                                  C.c_int, _i8p, _dp, _dp, _ip, _ip]
        getattr(L, p + "groupwise_chunks").argtypes = [_dp, _i64, _i64, _dp, _i64, C.c_int, C.c_int,
                                              _i64, _i32p, _ip, _ip, _ip, _i64p]
        getattr(L, p + "exact_gemm").argtypes = [_dp, _i64, _i64, _dp, _i64, _dp]
        getattr(L, p + "fp64_gemm").argtypes = [_dp, _i64, _i64, _dp, _i64, _dp]
        getattr(L, p + "max_rel_err").argtypes = [_dp, _dp, _i64, _i64, _dp]
        getattr(L, p + "set_threads").argtypes = [C.c_int]
        getattr(L, p + "thread_count").restype = C.c_int

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def _check(self, rc: int) -> None:
        if rc != OK:
            raise OracleError(rc, self._fn("last_error")().decode())

    # -- closed-form host logic ------------------------------------------------
    def compute_beta(self, n: int) -> int:
        out = C.c_int()
        self._check(self._fn("compute_beta")(n, C.byref(out)))
        return out.value

    def compute_r(self, n: int, beta: int) -> int:
        out = _i64()
        self._check(self._fn("compute_r")(n, beta, C.byref(out)))
        return out.value

    def op_counts_with_r(self, k: int, r: int, accumulation: int = 1) -> dict:
        c = np.zeros(4, np.int64)
        self._check(self._fn("op_counts_with_r")(k, r, accumulation, _ptr(c, _i64p)))
        return dict(int8_gemms=int(c[0]), fp64_flushes=int(c[1]), r=int(c[2]), w=int(c[3]))

    def set_threads(self, n: int) -> None:
        self._fn("set_threads")(n)

    def thread_count(self) -> int:
        return self._fn("thread_count")()

    # -- generator -------------------------------------------------------------
    def counter_hash(self, seed: int, ctr: int) -> int:
        return int(self._fn("counter_hash")(seed, ctr))

    def gen_phi_matrix(self, m: int, n: int, phi: float, seed: int) -> np.ndarray:
        out = np.empty((m, n), np.float64)
        self._check(self._fn("gen_phi_matrix")(m, n, phi, seed, _ptr(out, _dp)))
        return out

    # -- the hot path ----------------------------------------------------------
    def gemm(self, alpha, a, b, beta, c, k=8, method="ozIMMU_H", force_beta=0,
             force_r=0, wrapping=False, with_info=False):
        """out = ozaki_gemm_ex(alpha, A, B, beta, C, config_for(method, k))."""
        a, b, c = _f64(a), _f64(b), _f64(c)
        m, n = a.shape
        n2, p = b.shape
        assert n == n2 and c.shape == (m, p)
        out = np.empty((m, p), np.float64)
        counts = np.zeros(4, np.int64)
        timings = np.zeros(5, np.float64)
        self._check(self._fn("gemm")(METHODS[method], k, force_beta, force_r, int(wrapping),
                                     alpha, _ptr(a, _dp), m, n, _ptr(b, _dp), p, beta,
                                     _ptr(c, _dp), _ptr(out, _dp), _ptr(counts, _i64p),
                                     _ptr(timings, _dp)))
        if with_info:
            info = dict(int8_gemms=int(counts[0]), fp64_flushes=int(counts[1]),
                        r=int(counts[2]), w=int(counts[3]),
                        timings=dict(zip(["split_a", "split_b", "int_gemm", "accum_fp64",
                                          "copy"], timings.tolist())))
            return out, info
        return out

    def split(self, a, k, side="left", force_beta=0, residual=False) -> Split:
        a = _f64(a)
        rows, cols = a.shape
        sl = np.zeros((k, rows, cols), np.int8)
        sh = np.zeros(rows if side == "left" else cols, np.float64)
        res = np.zeros((rows, cols), np.float64) if residual else None
        beta, uf = C.c_int(), C.c_int()
        self._check(self._fn("split_rn_const_shift")(
            _ptr(a, _dp), rows, cols, k, 0 if side == "left" else 1, force_beta,
            _ptr(sl, _i8p), _ptr(sh, _dp), _ptr(res, _dp) if residual else None,
            C.byref(beta), C.byref(uf)))
        return Split(sl, sh, beta.value, bool(uf.value), res)

    def groupwise_chunks(self, a, b, k, force_beta=0, force_r=0) -> Chunks:
        a, b = _f64(a), _f64(b)
        m, n = a.shape
        p = b.shape[1]
        wmax = k * (k + 1) // 2
        acc = np.zeros((wmax, m, p), np.int32)
        g, s0, s1 = (np.zeros(wmax, np.int32) for _ in range(3))
        w = _i64()
        self._check(self._fn("groupwise_chunks")(
            _ptr(a, _dp), m, n, _ptr(b, _dp), p, k, force_beta, force_r, _ptr(acc, _i32p),
            _ptr(g, _ip), _ptr(s0, _ip), _ptr(s1, _ip), C.byref(w)))
        w = w.value
        return Chunks(acc[:w].copy(), g[:w].copy(), s0[:w].copy(), s1[:w].copy())

    # -- accuracy tools --------------------------------------------------------
    def exact_gemm(self, a, b) -> np.ndarray:
        a, b = _f64(a), _f64(b)
        out = np.empty((a.shape[0], b.shape[1]), np.float64)
        self._check(self._fn("exact_gemm")(_ptr(a, _dp), a.shape[0], a.shape[1],
                                           _ptr(b, _dp), b.shape[1], _ptr(out, _dp)))
        return out

    def fp64_gemm(self, a, b) -> np.ndarray:
        a, b = _f64(a), _f64(b)
        out = np.empty((a.shape[0], b.shape[1]), np.float64)
        self._check(self._fn("fp64_gemm")(_ptr(a, _dp), a.shape[0], a.shape[1],
                                          _ptr(b, _dp), b.shape[1], _ptr(out, _dp)))
        return out

    def max_rel_err(self, t, r) -> float:
        t, r = _f64(t), _f64(r)
        out = C.c_double()
        self._check(self._fn("max_rel_err")(_ptr(t, _dp), _ptr(r, _dp), t.shape[0],
                                            t.shape[1], C.byref(out)))
        return out.value


class RefLib(_Base):
    """The unmodified reference library (kind "reference")."""
    prefix = "ozref_"
    kind = "reference"

    def __init__(self, path: str = REF_SO):
        super().__init__(path)
        self.lib.ozref_split_any.argtypes = [C.c_int, _dp, _i64, _i64, C.c_int, C.c_int, C.c_int,
                                             _i8p, _dp, _dp]
        self.lib.ozref_total_bound.argtypes = [C.c_int, C.c_int, C.c_int, _i64, _dp, _i64, _i64,
                                               _dp, _i64, _dp]

    def total_bound(self, a, b, k, method="ozIMMU_H", force_beta=0, force_r=0):
        """The reference's section-5 elementwise bound (analysis.cpp:73-100)."""
        a, b = _f64(a), _f64(b)
        out = np.empty((a.shape[0], b.shape[1]), np.float64)
        self._check(self.lib.ozref_total_bound(METHODS[method], k, force_beta, force_r,
                                               _ptr(a, _dp), a.shape[0], a.shape[1],
                                               _ptr(b, _dp), b.shape[1], _ptr(out, _dp)))
        return out

    def split_any(self, a, k, strategy, side="left", force_beta=0, residual=False):
        """strategy: "rn_const" | "bitmask" | "rn_per_slice".  Returns (slices, shift or
        units), plus the residual matrix when ``residual``."""
        code = {"rn_const": 0, "bitmask": 1, "rn_per_slice": 2}[strategy]
        a = _f64(a)
        rows, cols = a.shape
        lines = rows if side == "left" else cols
        sl = np.zeros((k, rows, cols), np.int8)
        out = np.zeros((k, lines) if code == 2 else (lines,), np.float64)
        res = np.zeros((rows, cols), np.float64) if residual else None
        self._check(self.lib.ozref_split_any(code, _ptr(a, _dp), rows, cols, k,
                                             0 if side == "left" else 1, force_beta,
                                             _ptr(sl, _i8p), _ptr(out, _dp),
                                             _ptr(res, _dp) if residual else None))
        return (sl, out, res) if residual else (sl, out)


class PortLib(_Base):
    """The plain-C restatement (kind "port")."""
    prefix = "ozport_"
    kind = "port"

    def __init__(self, path: str = PORT_SO):
        super().__init__(path)


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def best() -> _Base:
    """The reference build when present, else the port."""
    return RefLib() if have_ref() else PortLib()
