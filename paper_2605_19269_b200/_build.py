"""Build the in-tree C-ABI library `_lib/libcoda.so` with nvcc for sm_100a.

The library is plain CUDA C++ (no torch headers), compiled with
``-gencode arch=compute_100a,code=sm_100a`` so tcgen05/TMA instructions are
accepted (the generic compute_100 PTX target rejects them).  The built .so
stays in-tree so it travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "_lib"
LIB = LIBDIR / "libcoda.so"
LIB_EXP = LIBDIR / "libcoda_exp.so"     # -DCODA_EXPERIMENTS: measurement knobs for tools/
INCLUDE = PKG.parent / "include"

SOURCES = ["coda_api.cu"]
DEPS = ["coda_api.cu", "coda_gemm.cuh", "coda_aux.cuh", "coda_ptx.cuh", "coda_mainloop.cuh", "coda_fast.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; cannot build the CODA CUDA library")


def needs_build(lib: Path = LIB) -> bool:
    if not lib.exists():
        return True
    t = lib.stat().st_mtime
    srcs = [CSRC / d for d in DEPS] + [INCLUDE / "coda.h"]
    return any(s.exists() and s.stat().st_mtime > t for s in srcs)


def build(force: bool = False, verbose: bool = False, experiments: bool = False) -> Path:
    """Compile libcoda.so (or the experiment build libcoda_exp.so) if missing or stale."""
    lib = LIB_EXP if experiments else LIB
    if not force and not needs_build(lib):
        return lib
    LIBDIR.mkdir(parents=True, exist_ok=True)
    tmp = lib.with_suffix(".so.tmp")
    extra = ["-DCODA_EXPERIMENTS"] if experiments else []
    cmd = [_nvcc(), *NVCC_FLAGS, *extra, "-I", str(INCLUDE), "-o", str(tmp), *[str(CSRC / s) for s in SOURCES]]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc failed ({proc.returncode}):\n{proc.stderr[-4000:]}")
    if verbose:
        print(proc.stderr)
    (LIBDIR / ("ptxas_exp.log" if experiments else "ptxas.log")).write_text(proc.stderr)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":  # pragma: no cover
    print(build(force=True, verbose=True))
