"""Shared test helpers (test infrastructure)."""
import numpy as np

GOLDEN_CASES = ["phi05_k8", "phi1_k9_ab", "phi4_k14_r3", "phi2_k8_r2", "special_k8",
                "special_k12_r5", "beta3_k5", "n1", "m1p1"]


def bits(x):
    return np.ascontiguousarray(x, dtype=np.float64).view(np.uint64)


def assert_bitwise(got, want, what=""):
    """Bit-exact FP64 equality (NaN payloads compared as 'both NaN')."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    assert got.shape == want.shape, (what, got.shape, want.shape)
    same = (bits(got) == bits(want)) | (np.isnan(got) & np.isnan(want))
    if not same.all():
        idx = np.argwhere(~same)
        i = tuple(idx[0])
        raise AssertionError(f"{what}: {len(idx)} of {same.size} entries differ; first at {i}: "
                             f"got {got[i]!r} want {want[i]!r}")


def case(golden, name):
    pre = name + "/"
    m, n, p, k, fb, fr = (int(v) for v in golden[pre + "params"])
    phi, alpha, beta = (float(v) for v in golden[pre + "scalars"])
    return dict(m=m, n=n, p=p, k=k, force_beta=fb, force_r=fr, phi=phi, alpha=alpha, beta=beta,
                A=golden[pre + "A"], B=golden[pre + "B"], C=golden[pre + "C"],
                out=golden[pre + "out"], counts=golden[pre + "counts"],
                sliceA=golden[pre + "sliceA"], shiftA=golden[pre + "shiftA"],
                sliceB=golden[pre + "sliceB"], shiftB=golden[pre + "shiftB"],
                beta_underflow=golden[pre + "beta_underflow"],
                chunk_acc=golden[pre + "chunk_acc"], chunk_gs=golden[pre + "chunk_gs"])


import os as _os

ROOT_HEADER = _os.path.join(_os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))),
                            "include", "ozmm_b200.h")


def save_ozmm(path, m, kind=0):
    """OZMM container (proj/src/io.cpp:16-18, :56-70): magic, version 1, kind, 6 zero
    bytes, u64 LE rows, u64 LE cols, row-major LE payload."""
    import struct
    m = np.ascontiguousarray(m)
    with open(path, "wb") as f:
        f.write(b"OZMM" + bytes([1, kind]) + bytes(6) + struct.pack("<QQ", *m.shape))
        f.write(m.tobytes())


def load_ozmm(path, kind=0):
    """kind 0 = F64, 1 = I8 (io.hpp:17)."""
    import struct
    raw = open(path, "rb").read()
    assert raw[:4] == b"OZMM" and raw[4] == 1 and raw[5] == kind
    rows, cols = struct.unpack("<QQ", raw[12:28])
    return np.frombuffer(raw[28:], dtype="<f8" if kind == 0 else "i1").reshape(rows, cols)
