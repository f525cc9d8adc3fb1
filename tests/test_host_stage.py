"""The host entry's copy team (csrc/host_stage.hpp WorkerPool), CPU only: many
back-to-back jobs, every index exactly once on its own job's function; and the
staging copy loops (copy_screen / copy_patch / copy_stream) against scalar loops."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_worker_pool_stress(tmp_path):
    nvcc = "/usr/local/cuda/bin/nvcc" if os.path.exists("/usr/local/cuda/bin/nvcc") else shutil.which("nvcc")
    if not nvcc:
        pytest.skip("nvcc not found")
    exe = tmp_path / "pool_stress"
    res = subprocess.run([nvcc, "-O2", "-std=c++17", "-x", "cu", "-Wno-deprecated-gpu-targets",
                          "-o", str(exe), os.path.join(ROOT, "tests", "cpp", "pool_stress.cpp")],
                         capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    out = subprocess.run([str(exe), "20000"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "POOL-OK" in out.stdout and "COPY-OK" in out.stdout, out.stdout + out.stderr
