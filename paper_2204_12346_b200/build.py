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
import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
SOURCES = [CSRC / "engine.cu", CSRC / "gswarm.cu", CSRC / "family.cu", CSRC / "host_api.cpp"]
HEADERS = [CSRC / "sird_device.cuh", CSRC / "kernels.cuh", CSRC / "launchers.cuh", CSRC / "engine_internal.h",
           CSRC / "engine_core.cuh",
           ROOT / "include" / "sirdgpu.h", ROOT / "include" / "sirdfit_b200.hpp"]
OUT = PKG / "libsirdgpu.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-fmad=false", "-std=c++20", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
         f"-I{ROOT / 'include'}"]
# translation units compiled in parallel: the templated kernels per
# objective family and substep specialisation (family.cu six times), the
# rest of the engine, the C++ API
_FAMILY_UNITS = [(f, sub) for f in (0, 1) for sub in (24, -24, -1, 0)]
UNITS = [("engine", CSRC / "engine.cu", []), ("gswarm", CSRC / "gswarm.cu", []),
         ("host_api", CSRC / "host_api.cpp", [])] + [
    (f"family{f}_s{str(sub).replace('-', 'm')}", CSRC / "family.cu", [f"-DSG_FAMILY={f}", f"-DSG_SUB={sub}", f"-DSG_UNIT={k}"])
    for k, (f, sub) in enumerate(_FAMILY_UNITS)]


def needs_build() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    return any(p.exists() and p.stat().st_mtime > t for p in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False, out: Path = OUT, extra: list | None = None) -> Path:
    """Compile libsirdgpu.so (`extra`: additional nvcc flags, e.g. tuning -D for experiments)."""
    if not force and out == OUT and not extra and not needs_build():
        return OUT
    out = Path(out)
    objdir = Path(tempfile.mkdtemp(prefix="sirdgpu_build_"))
    try:
        procs = []
        for name, src, defs in UNITS:
            obj = objdir / f"{name}.o"
            cmd = [NVCC, *ARCH, *FLAGS, *defs, *(extra or []), "-c", "-o", str(obj), str(src)]
            if verbose:
                print(" ".join(cmd), flush=True)
            procs.append((cmd, obj, subprocess.Popen(cmd)))
        failed = [cmd for cmd, _, p in procs if p.wait() != 0]
        if failed:
            raise subprocess.CalledProcessError(1, failed[0])
        link = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(out), *[str(o) for _, o, _ in procs]]
        if verbose:
            print(" ".join(link), flush=True)
        subprocess.run(link, check=True)
    finally:
        shutil.rmtree(objdir, ignore_errors=True)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(OUT)
