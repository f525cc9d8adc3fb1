"""The full-matrix accuracy harness (tests/accuracy_full.py) and its GPU
double-double reference, pinned to the reference's exact oracle.

The reference measures max_rel_err against exact_gemm_oracle
(proj/src/harness.cpp:60-80, oracle.cpp:276-335).  At sizes where the exact
oracle finishes in seconds, the dd reference must round to the exact oracle's
value on every entry, and max_rel_err computed against it must equal the
reference's own max_rel_err against the exact oracle.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def env():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import oracle
    from paper_2409_13313_b200 import ozmm
    from tests import accuracy_full as af
    if not os.path.exists(oracle.PORT_SO):
        oracle.build()
    return ozmm, oracle.best(), af


@pytest.mark.parametrize("phi", [0.5, 2.0, 4.0])
def test_dd_reference_matches_exact_oracle_full(env, phi):
    ozmm, chk, af = env
    m, n, p = 256, 768, 192
    A = ozmm.gen_phi_matrix(m, n, phi, ozmm.counter_hash(5, 1))
    B = ozmm.gen_phi_matrix(n, p, phi, ozmm.counter_hash(5, 2))
    hi, lo = af.dd_gemm(torch.tensor(A, device="cuda"), torch.tensor(B, device="cuda"))
    exact = chk.exact_gemm(A, B)
    got = (hi + lo).cpu().numpy()
    assert int((got.view(np.uint64) != exact.view(np.uint64)).sum()) == 0


@pytest.mark.parametrize("phi,k", [(0.5, 6), (1.0, 8), (4.0, 12)])
def test_max_rel_err_dd_equals_reference_metric(env, phi, k):
    """max_rel_err(ozIMMU_H, dd) == the reference's max_rel_err(ozIMMU_H, exact)
    (same worst entry; the dd reference resolves the difference below 1 ulp)."""
    ozmm, chk, af = env
    n = 512
    A = ozmm.gen_phi_matrix(n, n, phi, ozmm.counter_hash(9, 1))
    B = ozmm.gen_phi_matrix(n, n, phi, ozmm.counter_hash(9, 2))
    dA, dB = torch.tensor(A, device="cuda"), torch.tensor(B, device="cuda")
    d = ozmm.ozaki_mm(dA, dB, ozmm.config_for("ozIMMU_H", k)).d
    hi, lo = af.dd_gemm(dA, dB)
    e_dd = af.max_rel_err_dd(d, hi, lo)
    e_ref = chk.max_rel_err(d.cpu().numpy(), chk.exact_gemm(A, B))
    assert e_dd == pytest.approx(e_ref, rel=1e-6), (e_dd, e_ref)


def test_sweep_rows_and_summary(env, tmp_path):
    ozmm, chk, af = env
    out = tmp_path / "acc.csv"
    rows, pins = af.run([384], [6, 10], [1.0], [0], 16, str(out), verbose=False)
    assert [r[3] for r in rows] == ["cuBLAS_DGEMM", "ozIMMU_H", "ozIMMU_H"]
    assert pins[0]["differ"] == 0
    assert rows[2][5] < rows[1][5]  # more slices, smaller error
    text = out.read_text().splitlines()
    assert text[0].startswith("#") and "n,phi,k,method" in text[2]
    assert af.summary(rows)[0].startswith("n=384 phi=1.0")
