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


def test_pair_schedules_flush_in_order(tmp_path):
    """csrc/schedule.hpp: standard and free (parked) CTA-pair schedules for k = 1..16
    and r in {1, 2, 3, 4, 8, 16, 128}: every product once, inside its pass windows,
    and the epilogue actions flush every chunk once in the reference's order
    (scheme.cpp:91-94) with consistent park slots (tests/cpp/schedule_check.cpp)."""
    gxx = shutil.which("g++")
    if not gxx:
        pytest.skip("g++ not found")
    exe = tmp_path / "schedule_check"
    res = subprocess.run([gxx, "-O2", "-std=c++17", "-o", str(exe),
                          os.path.join(ROOT, "tests", "cpp", "schedule_check.cpp")],
                         capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "SCHEDULE-OK" in out.stdout, out.stdout + out.stderr
    assert "k= 8 r=  2" in out.stdout
