"""Compile the CUDA engine in-tree for sm_100a (no JIT cache, no fallback).

``python -m paper_2008_05718_b200._build`` or ``build()`` produces
``paper_2008_05718_b200/libbc_b200.so`` next to this file.  nvcc
cross-compiles without a GPU, so this also runs in the CPU-only build
container; the resulting library travels to the GPU box with the snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO_PATH = os.path.join(HERE, "libbc_b200.so")
SOURCES = [os.path.join(HERE, "csrc", "bc_engine.cu")]
HEADERS = [os.path.join(HERE, "csrc", f) for f in (
    "bc_kernels.cuh", "bc_deep.cuh", "bc_border.cuh", "bc_dist.cuh", "bc_sssp.cuh", "bc_relabel.cuh",            # kernels
    "engine_state.cuh", "engine_sweeps.cuh", "engine_border.cuh", "engine_sssp.cuh", "engine_run.cuh",
    "engine_dist.cuh",  # host side
)] + [os.path.join(ROOT, "include", "bc_b200.h")]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise FileNotFoundError("nvcc not found; the CUDA engine cannot be built")


def is_stale() -> bool:
    if not os.path.exists(SO_PATH):
        return True
    t = os.path.getmtime(SO_PATH)
    return any(os.path.getmtime(f) > t for f in SOURCES + HEADERS + [__file__])


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """``defines`` / ``out`` build a tuning variant (e.g. BC_MIN_BLOCKS=6) beside the default."""
    if out is None and not force and not is_stale():
        return SO_PATH
    cmd = [
        nvcc_path(), "-O3", "-std=c++17",
        "-gencode", "arch=compute_100a,code=sm_100a",
        "-lineinfo", "-Xcompiler", "-fPIC", "-shared",
        "-ccbin", "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++",
        "-I", os.path.join(ROOT, "include"), "-I", os.path.join(HERE, "csrc"),
        "-o", out or SO_PATH,
    ] + ["-D" + d for d in defines] + SOURCES
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n%s\n%s" % (" ".join(cmd), res.stderr))
    if verbose:
        sys.stderr.write(res.stderr)
    return out or SO_PATH


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
