"""Compile the sm_100a shared library in-tree (no GPU needed; nvcc cross-compiles).

Flags that matter for parity: ``-fmad=false`` (no FMA contraction; every
float32 op rounded on its own like the reference's numpy chain) together with
the explicit ``__fmul_rn/__fadd_rn/__fsub_rn`` in the kernel, ``-ftz=false``
(keep denormals like numpy) and IEEE division/sqrt.  ``-cudart static`` keeps
the library loadable without a CUDA runtime path.
"""

from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
SRC = PKG / "csrc" / "rangeseg_b200.cu"
OUT = PKG / "_lib" / "librangeseg_b200.so"
INCLUDE = PKG.parent / "include"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false", "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def build(force: bool = False, verbose: bool = False) -> Path:
    deps = [SRC, INCLUDE / "rangeseg_b200.h"]
    if not force and OUT.exists() and all(OUT.stat().st_mtime >= d.stat().st_mtime for d in deps):
        return OUT
    OUT.parent.mkdir(parents=True, exist_ok=True)
    tmp = OUT.with_suffix(".so.tmp")
    cmd = [nvcc(), *NVCC_FLAGS, "-I", str(INCLUDE), "-o", str(tmp), str(SRC)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True)
    tmp.replace(OUT)
    return OUT


if __name__ == "__main__":
    print(build(force=True, verbose=True))
