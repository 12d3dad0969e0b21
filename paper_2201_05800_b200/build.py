"""Build the in-tree CUDA library ``libstg_cuda.so`` for sm_100a.

Plain nvcc (no torch JIT cache): every translation unit is compiled with
``-gencode arch=compute_100a,code=sm_100a -lineinfo`` and linked into a shared
library next to this file, so the built artefact travels with the repo
snapshot to the GPU box.  The static CUDA runtime is linked in; the driver API
entry point for TMA descriptors is resolved at run time through
``cudaGetDriverEntryPoint`` (no -lcuda).  No CUDA libraries (cuBLAS etc.)
are linked: every kernel on the path is in csrc/.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libstg_cuda.so"
OBJDIR = PKG / "build_obj"

SOURCES = ["kernels_slab.cu", "kernels_vec.cu", "kernels_precond.cu", "kernels_fdm.cu",
           "kernels_general.cu", "kernels_small.cu", "stg.cpp"]
HEADERS = ["kernels.hpp", "constants.hpp", "eig.hpp", "ptx.cuh", "krylov.cuh", "hostcopy.hpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                  "-Xcompiler", "-Wall", "--expt-relaxed-constexpr", f"-I{ROOT / 'include'}"]


def nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found: the CUDA toolkit is required to build libstg_cuda.so")
    return cand


def _host_compiler() -> list[str]:
    # $CXX in this image may point at a toolchain without libgomp/libstdc++
    # headers nvcc expects; pin the system g++ when present.
    for c in ("/usr/bin/g++", shutil.which("g++")):
        if c and Path(c).exists():
            return ["-ccbin", c]
    return []


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "stg_cuda.h", Path(__file__)]
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    OBJDIR.mkdir(exist_ok=True)
    cc = [nvcc()] + _host_compiler()
    objs = [str(OBJDIR / (s + ".o")) for s in SOURCES]

    def compile_one(s: str) -> None:
        cmd = cc + NVFLAGS + ["-c", str(CSRC / s), "-o", str(OBJDIR / (s + ".o"))]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)

    # translation units are independent: compile them concurrently
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        list(ex.map(compile_one, SOURCES))
    tmp = LIB.with_suffix(".so.tmp")
    # no library kernels: static CUDA runtime only
    cmd = cc + ARCH + ["-shared", "-Xcompiler", "-pthread", "-o", str(tmp)] + objs
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
