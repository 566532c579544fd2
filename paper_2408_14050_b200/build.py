"""Compile libocc.so (all CUDA kernels + the C ABI) in-tree for sm_100a.

The fp recipe: -fmad=false (no FMA contraction in any
precision), -prec-sqrt=true, -prec-div=true, -ftz=false; host code
-ffp-contract=off.  The library links the CUDA runtime statically so the
built .so is self-contained on the GPU box.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libocc.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-shared", "-Xcompiler", "-fPIC,-ffp-contract=off",
         "-fmad=false", "-prec-sqrt=true", "-prec-div=true", "-ftz=false",
         "-I", os.path.join(ROOT, "include")]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def build(force: bool = False, verbose: bool = False) -> str:
    deps = sources() + glob.glob(os.path.join(HERE, "csrc", "*.h")) + [os.path.join(ROOT, "include", "occ.h")]
    newest = max(os.path.getmtime(p) for p in deps)
    if not force and os.path.exists(SO) and os.path.getmtime(SO) >= newest:
        return SO
    cmd = [NVCC, *ARCH, *FLAGS, *(["-Xptxas", "-v"] if verbose else []), "-o", SO, *sources()]
    subprocess.run(cmd, check=True)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
