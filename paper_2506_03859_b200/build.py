"""Build libfarqb.so (sm_100a) in-tree: paper_2506_03859_b200/lib/libfarqb.so.

    python -m paper_2506_03859_b200.build        # or __graft_entry__.build()

nvcc cross-compiles for sm_100a without a GPU.  Objects are compiled in
parallel and only rebuilt when a source or header is newer than its object.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "build", "obj")
LIB_DIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIB_DIR, "libfarqb.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
                     "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _newest_header() -> float:
    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.hpp")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))
    return max((os.path.getmtime(h) for h in hdrs), default=0.0)


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), _newest_header()):
        return obj
    cmd = [nvcc()] + NVCC_FLAGS + ["-c", src, "-o", obj]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(LIB_DIR, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs + ["-lpthread"]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    build_dropin(verbose)
    return LIB


REF_INCLUDE = os.environ.get("FARQB_REF_INCLUDE", "/root/reference/proj/include")
DROPIN_SRC = os.path.join(PKG, "dropin", "rsvd_link.cpp")
DROPIN_LIB = os.path.join(LIB_DIR, "librsvd_b200.so")


def build_dropin(verbose: bool = False) -> str | None:
    """lib/librsvd_b200.so: rsvd::run_fixed_precision / run_fixed_rank with the reference's
    exact C++ signatures on the engine (dropin/rsvd_link.cpp).  Needs the reference's
    public headers at build time (FARQB_REF_INCLUDE); skipped without them (the built .so
    travels with the tree)."""
    if not os.path.isdir(os.path.join(REF_INCLUDE, "rsvd")):
        return None
    if os.path.exists(DROPIN_LIB) and os.path.getmtime(DROPIN_LIB) >= max(
            os.path.getmtime(DROPIN_SRC), os.path.getmtime(LIB), os.path.getmtime(os.path.join(ROOT, "include", "farqb.h"))):
        return DROPIN_LIB
    cxx = shutil.which("g++") or "g++"
    cmd = [cxx, "-std=c++20", "-O2", "-fPIC", "-shared", "-Wall", "-Wextra", "-I" + REF_INCLUDE,
           "-I" + os.path.join(ROOT, "include"), DROPIN_SRC, "-L" + LIB_DIR, "-lfarqb", "-Wl,-rpath,$ORIGIN",
           "-o", DROPIN_LIB]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"drop-in build failed:\n{r.stdout}\n{r.stderr}")
    return DROPIN_LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
