"""Build the in-tree CUDA library ``paper_2409_13313_b200/libozmm_b200.so``.

One nvcc invocation, sm_100a only (tcgen05/TMA need the arch-specific
target): the kernels + C ABI (csrc/ozmm_capi.cu) and the host input generator
(csrc/host_generate.cpp).  ``--fmad=false`` plus explicit ``__d*_rn``
intrinsics keep every FP64 operation singly rounded (the reference is built
with -ffp-contract=off, proj/src/CMakeLists.txt:18-20).  The CUDA runtime is
linked statically (nvcc default) so the .so needs only libcuda at run time.

``--diag`` builds the diagnostic variant (-DOZMM_DIAG): the environment
overrides used by the tuning probes under tools/ (OZMM_STAGES, OZMM_GROUP_M,
OZMM_TILE_TRACE, ...) and the timing-only hooks that change results
(OZMM_ONLY_BATCH, OZMM_DUP_MMA, OZMM_IDESC_XOR).  The release build reads no
environment variable.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libozmm_b200.so")
CLI = os.path.join(PKG, "ozmm_b200_cli")
CLI_SRC = os.path.join(PKG, "cli", "ozmm_cli.cpp")
SOURCES = [os.path.join(CSRC, "ozmm_capi.cu"), os.path.join(CSRC, "host_generate.cpp"),
           os.path.join(CSRC, "ozmm_grid.cpp")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp"))] + [
    os.path.join(ROOT, "include", "ozmm_b200.h")]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _host_cxx() -> str:
    # /usr/bin/g++ ships libgomp; some images put a gcc without it first in $CXX.
    for cand in ("/usr/bin/g++", shutil.which("g++")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("g++ not found")


def command(out: str = LIB, verbose_ptxas: bool = False, diag: bool = False) -> list[str]:
    cmd = [
        _nvcc(), "-ccbin", _host_cxx(),
        "-gencode", "arch=compute_100a,code=sm_100a",
        "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
        "-Xcompiler", "-fPIC,-fopenmp,-ffp-contract=off,-O3",
        "-shared", "-o", out, *SOURCES, "-lgomp", "-ldl",
    ]
    if verbose_ptxas:
        cmd[1:1] = ["-Xptxas", "-v"]
    if diag:
        cmd[1:1] = ["-DOZMM_DIAG"]
    return cmd


VARIANT = LIB + ".variant"  # "release" or "diag": which build the .so is


def up_to_date(out: str = LIB) -> bool:
    if not os.path.exists(out):
        return False
    try:
        with open(VARIANT) as f:
            if f.read().strip() != "release":
                return False
    except OSError:
        return False
    t = os.path.getmtime(out)
    return all(os.path.getmtime(d) <= t for d in DEPS if os.path.exists(d))


def build_cli() -> str:
    """The reference-CLI-compatible front end (gemm / counts) over the C ABI."""
    cmd = [_host_cxx(), "-std=c++17", "-O2", "-Wall", "-o", CLI, CLI_SRC, f"-L{PKG}",
           "-l:libozmm_b200.so", "-Wl,-rpath,$ORIGIN"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("CLI build failed:\n" + " ".join(cmd) + "\n" + res.stdout + res.stderr)
    return CLI


def build(force: bool = False, verbose: bool = False, diag: bool = False) -> str:
    if not force and not diag and up_to_date():
        if not os.path.exists(CLI) or os.path.getmtime(CLI) < os.path.getmtime(CLI_SRC):
            build_cli()
        return LIB
    cmd = command(verbose_ptxas=verbose, diag=diag)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc build failed:\n" + " ".join(cmd) + "\n" + res.stdout + res.stderr)
    if verbose:
        sys.stderr.write(res.stdout + res.stderr)
    with open(VARIANT, "w") as f:
        f.write("diag" if diag else "release")
    build_cli()
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, diag="--diag" in sys.argv))
