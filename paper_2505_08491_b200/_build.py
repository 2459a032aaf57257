"""Build the C-ABI CUDA library ``libmdp_b200.so`` in-tree for sm_100a.

Plain nvcc invocations (no torch JIT cache): the .so lands next to the
package so it travels to the GPU box with the repo snapshot.
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
LIBDIR = PKG / "lib"
LIB = LIBDIR / "libmdp_b200.so"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SOURCES = ["operators.cu", "krylov.cu", "unet.cu", "unet_tc.cu", "gmg.cu"]
CPP_SOURCES = ["host.cpp"]


def nvcc() -> str:
    path = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(path).exists():
        raise RuntimeError("nvcc not found; cannot build the sm_100a library")
    return path


def _run(cmd):
    print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def build(verbose_ptxas: bool = False, force: bool = False) -> Path:
    """Compile every CUDA/C++ source into ``lib/libmdp_b200.so``."""
    LIBDIR.mkdir(exist_ok=True)
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    sources = [CSRC / s for s in CU_SOURCES + CPP_SOURCES]
    headers = list(CSRC.glob("*.cuh")) + [ROOT / "include" / "mdp_b200.h"]
    newest = max(p.stat().st_mtime for p in sources + headers)
    if LIB.exists() and LIB.stat().st_mtime > newest and not force:
        return LIB
    nv = nvcc()
    objs = []
    common = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-I", str(ROOT / "include")]
    for s in CU_SOURCES:
        o = objdir / (s + ".o")
        extra = ["-Xptxas", "-v"] if verbose_ptxas else []
        _run([nv, *ARCH, "-lineinfo", *common, *extra, "-c", str(CSRC / s), "-o", str(o)])
        objs.append(str(o))
    cuda_inc = str(Path(nv).resolve().parent.parent / "include")
    for s in CPP_SOURCES:
        o = objdir / (s + ".o")
        # plain host C++; no FMA contraction so the ILU factor matches the reference bitwise
        _run(["g++", "-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-I", cuda_inc, "-I", str(ROOT / "include"),
              "-c", str(CSRC / s), "-o", str(o)])
        objs.append(str(o))
    tmp = LIB.with_suffix(".so.tmp")
    _run([nv, *ARCH, "-shared", "-o", str(tmp), *objs])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(verbose_ptxas="-v" in sys.argv, force="-f" in sys.argv)
