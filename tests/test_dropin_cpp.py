"""The C++ adapter (paper_2409_13313_b200/cpp/ozmm_gpu.hpp) as a drop-in for the
reference API: one binary calls ozmm::ozaki_gemm_ex (the unmodified reference)
and ozmm::gpu::ozaki_gemm_ex (the B200 path) with the same arguments.
The binary is built in the build container by `make -C oracle dropin`
(oracle/_ref/dropin_demo, it needs the reference headers) and ships with the
repo snapshot to the GPU box."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO = os.path.join(ROOT, "oracle", "_ref", "dropin_demo")


def _run(*args):
    if not os.path.exists(DEMO):
        pytest.skip("oracle/_ref/dropin_demo not built (needs /root/reference at build time)")
    return subprocess.run([DEMO, *map(str, args)], capture_output=True, text=True, timeout=600)


def test_dropin_closed_forms_cpu():
    out = _run(16384, 16384, 16384, 8, 0.5, "--closed-forms-only")
    assert out.returncode == 0 and "CLOSED-FORMS OK beta=7 r=8" in out.stdout, out.stdout + out.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,p,k,phi", [(300, 2000, 260, 8, 0.5), (97, 5000, 131, 12, 4.0)])
def test_dropin_same_call_site_bit_exact(m, n, p, k, phi):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = _run(m, n, p, k, phi)
    assert out.returncode == 0 and out.stdout.startswith("MATCH"), out.stdout + out.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("method", ["ozIMMU", "ozIMMU_RN", "ozIMMU_EF"])
def test_dropin_comparison_methods_bit_exact(method):
    """config_for(ozIMMU / ozIMMU_RN / ozIMMU_EF, k) through the same call site: the
    adapter maps (strategy, accumulation) to the GPU method, never silently to ozIMMU_H."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = _run(257, 3000, 190, 9, 2.0, method)
    assert out.returncode == 0 and out.stdout.startswith("MATCH"), out.stdout + out.stderr


@pytest.mark.gpu
def test_dropin_overflow_modes():
    """force_r on INT32-overflowing inputs: Wrapping bit-identical to the reference,
    Checked throws the adapter's OverflowError (int_gemm.hpp:15-26)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = _run(32, 65536, 24, 14, 0.0, "overflow", 14)
    assert out.returncode == 0 and "OVERFLOW-OK" in out.stdout, out.stdout + out.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,p,k,phi", [(90, 700, 70, 9, 2.0), (33, 4111, 20, 14, 4.0)])
def test_dropin_split_api_bit_exact(m, n, p, k, phi):
    """ozmm::gpu::split<ozmm::SplitMatrix> at the reference's split_bitmask /
    split_round_nearest / split_rn_const_shift call sites (split.hpp:61-74):
    slices, shifts or per-slice units, residual, underflow flag and metadata
    identical, for A split by rows and B by columns."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = _run(m, n, p, k, phi, "split")
    assert out.returncode == 0 and "SPLIT-OK" in out.stdout, out.stdout + out.stderr
