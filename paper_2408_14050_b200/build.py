"""Compile libocc.so (all CUDA kernels + the C ABI) in-tree for sm_100a.

The fp recipe: -fmad=false (no FMA contraction in any
precision), -prec-sqrt=true, -prec-div=true, -ftz=false; host code
-ffp-contract=off.  The library links the CUDA runtime statically so the
built .so is self-contained on the GPU box.
"""
from __future__ import annotations

import concurrent.futures
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


def defines() -> list:
    """Extra -D flags of an instrumented build (OCC_DEFINES="-DSWEEP_STATS ...";
    OCC_LINE_STATS=1 adds -DOCC_LINE_STATS).  Each flag set gets its own object
    directory and library (libocc_<tag>.so), so instrumented objects are never
    linked into the product library."""
    d = os.environ.get("OCC_DEFINES", "").split()
    if os.environ.get("OCC_LINE_STATS"):        # event counters of k_line (tools/line_stats.py)
        d.append("-DOCC_LINE_STATS")
    return sorted(set(d))


def lib_path() -> str:
    d = defines()
    if not d:
        return SO
    import hashlib
    return os.path.join(HERE, "libocc_" + hashlib.sha1(" ".join(d).encode()).hexdigest()[:8] + ".so")


def build(force: bool = False, verbose: bool = False) -> str:
    deps = sources() + glob.glob(os.path.join(HERE, "csrc", "*.h")) + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + [os.path.join(ROOT, "include", "occ.h")]
    newest = max(os.path.getmtime(p) for p in deps)
    so = lib_path()
    if not force and os.path.exists(so) and os.path.getmtime(so) >= newest:
        return so
    # one object per translation unit, compiled in parallel, then linked
    tag = os.path.basename(so)[len("libocc"):-len(".so")]
    objdir = os.path.join(HERE, "build_obj" + tag)
    os.makedirs(objdir, exist_ok=True)
    cflags = [f for f in FLAGS if f != "-shared"] + defines()
    jobs = []
    hdr_newest = max(os.path.getmtime(p) for p in deps if not p.endswith(".cu"))
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_newest):
            continue
        jobs.append([NVCC, *ARCH, *cflags, *(["-Xptxas", "-v"] if verbose else []), "-c", src, "-o", obj])
    with concurrent.futures.ThreadPoolExecutor(max_workers=max(1, len(jobs))) as ex:
        for r in ex.map(lambda c: subprocess.run(c, capture_output=not verbose, text=True), jobs):
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed: {' '.join(r.args)}\n{r.stderr}")
    objs = [os.path.join(objdir, os.path.basename(src)[:-3] + ".o") for src in sources()]
    subprocess.run([NVCC, *ARCH, "-shared", "-o", so, *objs], check=True)
    return so


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
