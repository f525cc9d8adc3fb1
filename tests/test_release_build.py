"""The release library carries no environment hooks (CPU test).

Diagnostic overrides -- tuning sweeps, per-tile traces, and the timing probes
that change results (OZMM_ONLY_BATCH, OZMM_DUP_MMA, OZMM_IDESC_XOR) -- exist
only in the -DOZMM_DIAG build (paper_2409_13313_b200/build.py --diag)."""
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2409_13313_b200", "libozmm_b200.so")


def test_release_library_reads_no_ozmm_environment():
    if not os.path.exists(LIB):
        pytest.skip("library not built")
    with open(LIB + ".variant") as f:
        if f.read().strip() != "release":
            pytest.skip("diagnostic build in place")
    blob = open(LIB, "rb").read()
    for name in (b"OZMM_ONLY_BATCH", b"OZMM_DUP_MMA", b"OZMM_IDESC_XOR", b"OZMM_KPAIR",
                 b"OZMM_STAGES", b"OZMM_TILE_TRACE", b"OZMM_HOST_PANELS", b"OZMM_SIGNED"):
        assert name not in blob, name
