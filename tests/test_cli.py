"""The reference-CLI-compatible front end (paper_2409_13313_b200/cli/ozmm_cli.cpp):
`counts` against the reference's closed forms, OZMM format errors -> exit 2,
and (GPU) `gemm` over OZMM files bit-exact against the reference."""
import json
import os
import subprocess

import numpy as np
import pytest

from tests.helpers import assert_bitwise, load_ozmm, save_ozmm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2409_13313_b200", "ozmm_b200_cli")


def run(*args):
    if not os.path.exists(CLI):
        from paper_2409_13313_b200 import build
        build.build_cli()
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=600)


def kprime_max(n, beta):  # analysis.cpp:57-63
    return 1 if beta < 3 else max(1, (51 - (int(n).bit_length() - 1)) // beta - 1)


@pytest.mark.parametrize("n,k,method", [(1024, 8, "ozIMMU_H"), (16384, 8, "ozIMMU"),
                                        (65536, 8, "ozIMMU_EF"), (3, 14, "ozIMMU_RN"),
                                        (2 ** 18, 12, "ozIMMU_H")])
def test_counts_matches_reference(port, n, k, method):
    out = run("counts", "--n", n, "--k", k, "--method", method)
    assert out.returncode == 0, out.stderr
    got = dict(line.split(None, 1) for line in out.stdout.strip().splitlines())
    beta = port.compute_beta(n)
    r = port.compute_r(n, beta)
    acc = 0 if method in ("ozIMMU", "ozIMMU_RN") else 1
    c = port.op_counts_with_r(k, r, acc)
    assert int(got["beta"]) == beta and int(got["r"]) == r and int(got["w"]) == c["w"]
    assert int(got["int8_gemms"]) == c["int8_gemms"]
    assert int(got["fp64_flushes"]) == c["fp64_flushes"]
    assert int(got["kprime_max"]) == kprime_max(n, beta)


def test_format_and_usage_errors(tmp_path):
    good = tmp_path / "a.ozmm"
    save_ozmm(good, np.ones((2, 2)))
    bad = tmp_path / "bad.ozmm"
    bad.write_bytes(b"NOPE")
    i8 = tmp_path / "i8.ozmm"
    save_ozmm(i8, np.ones((2, 2), np.int8), kind=1)
    trailing = tmp_path / "t.ozmm"
    trailing.write_bytes(good.read_bytes() + b"x")
    for args in [("gemm", tmp_path / "missing.ozmm", good, "--out", tmp_path / "o"),
                 ("gemm", bad, good, "--out", tmp_path / "o"),
                 ("gemm", i8, good, "--out", tmp_path / "o"),
                 ("gemm", trailing, good, "--out", tmp_path / "o"),
                 ("gemm", good, good),
                 ("gemm", good, good, "--out", tmp_path / "o", "--method", "nope"),
                 ("counts", "--n", 0, "--k", 8, "--method", "ozIMMU_H"),
                 ("frobnicate",)]:
        out = run(*args)
        assert out.returncode == 2, (args, out.stdout, out.stderr)
        assert "error" in out.stderr or "usage" in out.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("method,trans", [("ozIMMU_H", False), ("ozIMMU_H", True), ("ozIMMU_EF", False)])
def test_gemm_over_ozmm_files(tmp_path, method, trans):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import oracle
    from paper_2409_13313_b200 import ozmm
    if not oracle.have_ref():
        pytest.skip("reference build absent")
    ref = oracle.RefLib()
    m, n, p, k = 130, 900, 70, 8
    A, B, C = (ozmm.gen_phi_matrix(*s, 1.0, i) for i, s in enumerate([(m, n), (n, p), (m, p)]))
    save_ozmm(tmp_path / "A.ozmm", A.T.copy() if trans else A)
    save_ozmm(tmp_path / "B.ozmm", B.T.copy() if trans else B)
    save_ozmm(tmp_path / "C.ozmm", C)
    args = ["gemm", tmp_path / "A.ozmm", tmp_path / "B.ozmm", tmp_path / "C.ozmm", "--out",
            tmp_path / "D.ozmm", "--alpha", 1.5, "--beta", 0.5, "--k", k, "--method", method]
    if trans:
        args += ["--transa", "--transb"]
    out = run(*args)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout)
    assert (line["m"], line["n"], line["p"], line["k"]) == (m, n, p, k)
    assert_bitwise(load_ozmm(tmp_path / "D.ozmm"),
                   ref.gemm(1.5, A, B, 0.5, C, k=k, method=method))


@pytest.mark.gpu
@pytest.mark.parametrize("method,strategy,trans", [("ozIMMU_H", "rn_const", False),
                                                   ("ozIMMU_H", "rn_const", True),
                                                   ("ozIMMU_EF", "bitmask", False),
                                                   ("ozIMMU_RN", "rn_per_slice", False)])
def test_dump_splits_match_reference(tmp_path, method, strategy, trans):
    """--dump-splits writes dump_split's files (split.cpp:254-270) for op(A) (Left)
    and op(B) (Right): slices, shift / per-slice units and residual bit-identical
    to the reference's SplitMatrix, including zero lines and signed zeros."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import oracle
    from paper_2409_13313_b200 import ozmm
    if not oracle.have_ref():
        pytest.skip("reference build absent")
    ref = oracle.RefLib()
    m, n, p, k = 70, 500, 45, 9
    A = ozmm.gen_phi_matrix(m, n, 2.0, 5)
    B = ozmm.gen_phi_matrix(n, p, 2.0, 6)
    A[3, :] = 0.0
    A[3, 7] = -0.0       # zero row holding a -0
    A[10, 11] = -0.0     # -0 in a live row
    B[:, 4] = -0.0       # zero column of -0
    A[20, 5] = 2.0 ** -1070   # bits below the slice grid / underflowing units
    save_ozmm(tmp_path / "A.ozmm", A.T.copy() if trans else A)
    save_ozmm(tmp_path / "B.ozmm", B.T.copy() if trans else B)
    args = ["gemm", tmp_path / "A.ozmm", tmp_path / "B.ozmm", "--out", tmp_path / "D.ozmm",
            "--k", k, "--method", method, "--dump-splits", tmp_path / "d"]
    if trans:
        args += ["--transa", "--transb"]
    out = run(*args)
    assert out.returncode == 0, out.stderr
    for name, X, side in (("a", A, "left"), ("b", B, "right")):
        sl, sh, res = ref.split_any(X, k, strategy, side, residual=True)
        for s in range(k):
            np.testing.assert_array_equal(load_ozmm(tmp_path / f"d.{name}.slice{s + 1}.ozmm", 1), sl[s])
        if strategy == "rn_per_slice":
            for s in range(k):
                assert_bitwise(load_ozmm(tmp_path / f"d.{name}.shift{s + 1}.ozmm")[0], sh[s])
        else:
            assert_bitwise(load_ozmm(tmp_path / f"d.{name}.shift.ozmm")[0], sh)
        assert_bitwise(load_ozmm(tmp_path / f"d.{name}.residual.ozmm"), res, f"{name} residual")


@pytest.mark.gpu
def test_overflow_mode_option(tmp_path):
    """--overflow-mode checked|wrapping (ozmm_cli.cpp:27-31): wrapping matches the
    reference's Wrapping result on inputs whose forced-r chunks overflow INT32;
    checked reports the overflow (exit 1) and writes no D; other values exit 2."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import oracle
    if not oracle.have_ref():
        pytest.skip("reference build absent")
    ref = oracle.RefLib()
    # the drop-in demo's overflowing case (tests/cpp/dropin_demo.cpp): constant operands
    # whose slices are all positive, so forced long chunks leave INT32
    m, n, p, k = 32, 65536, 24, 14
    v = (127.0 + 63.0 / 127.0) / 64.0
    A = np.full((m, n), v)
    B = np.full((n, p), v)
    save_ozmm(tmp_path / "A.ozmm", A)
    save_ozmm(tmp_path / "B.ozmm", B)
    base = ["gemm", tmp_path / "A.ozmm", tmp_path / "B.ozmm", "--k", k, "--force-r", 14]
    out = run(*base, "--out", tmp_path / "W.ozmm", "--overflow-mode", "wrapping")
    assert out.returncode == 0, out.stderr
    want = ref.gemm(1.0, A, B, 0.0, np.zeros((m, p)), k=k, force_r=14, wrapping=True)
    assert_bitwise(load_ozmm(tmp_path / "W.ozmm"), want)
    out = run(*base, "--out", tmp_path / "K.ozmm", "--overflow-mode", "checked")
    assert out.returncode == 1 and "overflow" in out.stderr.lower(), (out.stdout, out.stderr)
    assert not (tmp_path / "K.ozmm").exists()
    out = run(*base, "--out", tmp_path / "X.ozmm", "--overflow-mode", "saturating")
    assert out.returncode == 2
