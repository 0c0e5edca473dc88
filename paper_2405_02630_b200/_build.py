"""Build libqk.so (the sm_100a engine) in-tree with nvcc.

The shared library lands in ``paper_2405_02630_b200/_lib/libqk.so`` so it travels with the
repo snapshot to the GPU box (git-ignored, not gpurun-ignored).  Cross-compiles on a
machine without a GPU.
"""
from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "_lib" / "libqk.so"
SOURCES = ["qk_plan.cpp", "qk_sweep.cu", "qk_api.cu", "qk_statevector.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise FileNotFoundError("nvcc not found")


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + [CSRC / "qk_internal.h", ROOT / "include" / "qk.h"]
    return any(d.stat().st_mtime > t for d in deps)


def build_native(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    LIB.parent.mkdir(parents=True, exist_ok=True)
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), "-O3", "-lineinfo", "-std=c++17", *ARCH, "-Xcompiler", "-fPIC,-O3",
           "-shared", "-I", str(ROOT / "include"), "-o", str(tmp),
           *[str(CSRC / s) for s in SOURCES]]
    if verbose:
        cmd.append("-Xptxas=-v")
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build_native(force=True, verbose=True))
