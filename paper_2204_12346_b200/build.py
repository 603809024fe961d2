"""In-tree build of libsirdgpu.so for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2204_12346_b200.build

Flags: -gencode arch=compute_100a,code=sm_100a (Blackwell only), -lineinfo
for ncu source views, and -fmad=false so nvcc never contracts a multiply and
an add into an FMA (the reference performs every op with its own rounding;
SURVEY.md §0 finding 2).  The CUDA runtime is linked statically so the .so
travels to the GPU box as one file.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
SOURCES = [CSRC / "engine.cu", CSRC / "host_api.cpp"]
HEADERS = [CSRC / "sird_device.cuh", CSRC / "kernels.cuh", CSRC / "engine_internal.h", ROOT / "include" / "sirdgpu.h",
           ROOT / "include" / "sirdfit_b200.hpp"]
OUT = PKG / "libsirdgpu.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-fmad=false", "-std=c++20", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
         "-shared", f"-I{ROOT / 'include'}", "-cudart", "static"]


def needs_build() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    return any(p.exists() and p.stat().st_mtime > t for p in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False, out: Path = OUT, extra: list | None = None) -> Path:
    """Compile libsirdgpu.so (`extra`: additional nvcc flags, e.g. tuning -D for experiments)."""
    if not force and out == OUT and not extra and not needs_build():
        return OUT
    cmd = [NVCC, *ARCH, *FLAGS, *(extra or []), "-o", str(out), *[str(s) for s in SOURCES if s.exists()]]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(OUT)
