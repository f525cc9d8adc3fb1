"""CPU: the C-ABI library's host side (no GPU needed).

* libozmm_b200.so loads and exports every function include/ozmm_b200.h declares;
* closed forms (compute_beta / compute_r / op_counts) == the reference's;
* the host input generator == the reference generator, bit for bit, also
  block-wise (the multi-GPU shards);
* the GEMM kernel's schedule: chunk boundaries == the reference's flush
  schedule (groupwise_impl, scheme.cpp:81-101), every slice product issued
  exactly once, first-product (overwrite) flags, pass slice ranges.
"""
import re
from collections import Counter

import numpy as np
import pytest

from tests.helpers import GOLDEN_CASES, ROOT_HEADER, case

oz = pytest.importorskip("paper_2409_13313_b200.ozmm")


def header_functions():
    text = open(ROOT_HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ozmm_[a-z0-9_]+)\s*\(", text)))


def test_exports_every_declared_symbol():
    names = header_functions()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(oz.lib, n)]
    assert not missing, missing
    assert set(oz.EXPORTED_SYMBOLS) == set(names)


def test_status_strings():
    assert oz.lib.ozmm_status_string(0) == b"ok"
    assert b"magnitude" in oz.lib.ozmm_status_string(3)


def test_closed_forms_match_reference(golden, port):
    for n, b, r in zip(golden["closed/n"], golden["closed/beta"], golden["closed/r"]):
        assert oz.compute_beta(int(n)) == b
        assert oz.compute_r(int(n), int(b)) == r
    for (k, r), w in zip(golden["closed/kr"], golden["closed/w"]):
        c = oz.op_counts_with_r(int(k), int(r))
        assert c.w == w and c.int8_gemms == k * (k + 1) // 2
    with pytest.raises(ValueError):
        oz.compute_beta(0)
    with pytest.raises(ValueError):
        oz.compute_beta(2 ** 29 + 1)
    with pytest.raises(oz.ConfigError):
        oz.op_counts_with_r(0, 4)
    for n in (1, 2, 3, 17, 1000, 1 << 14, (1 << 17) + 1, 1 << 20, 1 << 29):
        assert oz.compute_beta(n) == port.compute_beta(n)
        for beta in (1, 3, 7):
            assert oz.compute_r(n, beta) == port.compute_r(n, beta)


def test_generator_matches_reference(golden, port):
    for name in ("phi05_k8", "phi4_k14_r3"):
        c = case(golden, name)
        seed = sum(map(ord, name))
        a = oz.gen_phi_matrix(c["m"], c["n"], c["phi"], oz.counter_hash(seed, 1))
        assert np.array_equal(a.view(np.uint64), c["A"].view(np.uint64))
    full = port.gen_phi_matrix(40, 70, 2.0, 99)
    blk = oz.gen_phi_block(40, 70, 2.0, 99, row0=7, nrows=11, col0=30, ncols=25)
    assert np.array_equal(blk.view(np.uint64), full[7:18, 30:55].view(np.uint64))
    assert oz.counter_hash(3, 4) == port.counter_hash(3, 4)
    with pytest.raises(ValueError):
        oz.gen_phi_block(4, 4, -1.0, 1)


@pytest.mark.parametrize("name", GOLDEN_CASES)
@pytest.mark.parametrize("mode", [(0, 0), (1, 64), (1, 32), (1, 128)])
def test_schedule_matches_reference_flushes(golden, name, mode):
    c = case(golden, name)
    k = c["k"]
    r = c["force_r"] or oz.compute_r(c["n"], c["force_beta"] or oz.compute_beta(c["n"]))
    rows, info = oz.debug_schedule(k, r, *mode)
    g_ref, s0_ref, s1_ref = c["chunk_gs"]
    assert info["chunks"] == len(g_ref) == int(c["counts"][3])
    # every product (s, t = g - s) exactly once, grouped into the reference's chunks
    assert Counter(map(tuple, rows[:, [4, 5]].tolist())) == Counter(
        (s, g - s) for g in range(2, k + 2) for s in range(1, g))
    for ch in range(info["chunks"]):
        mine = rows[rows[:, 2] == ch]
        assert set(mine[:, 3]) == {g_ref[ch]}
        assert sorted(mine[:, 4]) == list(range(s0_ref[ch], s1_ref[ch] + 1))
        assert mine[:, 6].sum() == 1 and mine[0, 6] == 1   # first product overwrites
        assert len(set(mine[:, 0])) == 1                    # one batch per chunk
    assert (rows[:, 7] == 1).all()                          # slices resident in the pass
    assert info["stages"] >= 2
    # batches are consecutive in flush order (epilogue folds chunks in order)
    assert all(np.diff(rows[:, 0]) >= 0)


def test_schedule_k_sweep():
    for k in range(1, 33):
        for r in (1, 2, 3, 8, 16, 128):
            rows, info = oz.debug_schedule(k, r)
            assert info["products"] == k * (k + 1) // 2
            assert info["chunks"] == oz.op_counts_with_r(k, r).w
            assert info["stages"] >= 2


def test_grid_layout():
    from paper_2409_13313_b200.grid2d import grid_shape, make_layout
    assert [grid_shape(w) for w in (1, 2, 4, 8)] == [(1, 1), (2, 1), (2, 2), (2, 4)]
    m, n, p = 64, 100, 96
    for world in (1, 2, 4, 8):
        rows_seen, cols_seen = [], []
        for rank in range(world):
            L = make_layout(m, n, p, world, rank)
            rows_seen += list(range(L.a_row0, L.a_row0 + L.ms))
            cols_seen += list(range(L.b_col0, L.b_col0 + L.ps))
            assert L.c_row0 <= L.a_row0 < L.c_row0 + L.mr
            assert L.c_col0 <= L.b_col0 < L.c_col0 + L.pcols
        assert sorted(rows_seen) == list(range(m))      # each row of A sliced once
        assert sorted(cols_seen) == list(range(p))      # each column of B sliced once


def test_native_grid_shape_matches_python():
    """ozmm_grid_shape (native grid) and grid2d.grid_shape pick the same Pr x Pc."""
    import ctypes
    from paper_2409_13313_b200 import ozmm
    from paper_2409_13313_b200.grid2d import grid_shape
    for w in range(1, 17):
        pr, pc = ctypes.c_int(), ctypes.c_int()
        assert ozmm.lib.ozmm_grid_shape(w, ctypes.byref(pr), ctypes.byref(pc)) == 0
        assert (pr.value, pc.value) == grid_shape(w), w
