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
HEADERS = sorted((PKG / "csrc").glob("*.cuh"))
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


PROF_OUT = PKG / "_lib" / "librangeseg_b200_prof.so"


def build(force: bool = False, verbose: bool = False, profile: bool = False,
          out: Path | None = None, defines=()) -> Path:
    out = out or (PROF_OUT if profile else OUT)
    deps = [SRC, INCLUDE / "rangeseg_b200.h", *HEADERS]
    if not force and out.exists() and all(out.stat().st_mtime >= d.stat().st_mtime for d in deps):
        return out
    out.parent.mkdir(parents=True, exist_ok=True)
    tmp = out.with_suffix(".so.tmp")
    cmd = [nvcc(), *NVCC_FLAGS, "-I", str(INCLUDE), "-o", str(tmp), str(SRC)]
    if profile:
        cmd.insert(1, "-DRS_PHASE_PROF")
    for d in defines:
        cmd.insert(1, f"-D{d}")
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True)
    tmp.replace(out)
    return out


TORCH_EXT_DIR = PKG / "_lib" / "torch_ext"
TORCH_EXT_NAME = "rangeseg_b200_torch"
TORCH_EXT_SRC = PKG / "csrc" / "torch_ext.cpp"


def build_torch_ext(force: bool = False) -> Path:
    """The thin PyTorch C++ extension over the C ABI (csrc/torch_ext.cpp),
    built in-tree next to librangeseg_b200.so (rpath $ORIGIN/..)."""
    out = TORCH_EXT_DIR / f"{TORCH_EXT_NAME}.so"
    deps = [TORCH_EXT_SRC, INCLUDE / "rangeseg_b200.h", OUT]
    if not force and out.exists() and all(out.stat().st_mtime >= d.stat().st_mtime for d in deps):
        return out
    from torch.utils import cpp_extension
    TORCH_EXT_DIR.mkdir(parents=True, exist_ok=True)
    cpp_extension.load(name=TORCH_EXT_NAME, sources=[str(TORCH_EXT_SRC)], build_directory=str(TORCH_EXT_DIR),
                       extra_include_paths=[str(INCLUDE)], extra_cflags=["-O2", "-std=c++17"],
                       extra_ldflags=[f"-L{OUT.parent}", "-lrangeseg_b200", "-Wl,-rpath,\\$$ORIGIN/.."],
                       with_cuda=True, verbose=False)
    out.touch()
    return out


if __name__ == "__main__":
    import sys
    print(build(force=True, verbose=True, profile="--profile" in sys.argv))
