"""Build ``libbanaserve.so`` in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_2510_13223_b200.build [--verbose]

Each translation unit is compiled to an object in ``build/`` (in parallel), then linked
into ``paper_2510_13223_b200/libbanaserve.so`` with the static CUDA runtime.  The .so
is git-ignored but travels to the GPU box with the gpurun snapshot.
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
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build", "banaserve")
LIB = os.path.join(PKG, "libbanaserve.so")
LIB_DEBUG = os.path.join(PKG, "libbanaserve_debug.so")   # -DBS_DEBUG=1 (device-side checks)
# -DBS_TIMELINE=1: per-CTA %globaltimer stamps in the attention kernel (diagnostics only,
# scripts/attn_timeline.py; never built by __graft_entry__.build())
LIB_TIMELINE = os.path.join(PKG, "libbanaserve_timeline.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
              "--expt-relaxed-constexpr", "-I", INCLUDE, "-I", CSRC]


def nccl_include() -> list:
    """nccl.h for the transport's types (functions are dlopen'd at run time)."""
    try:
        import nvidia.nccl as m
        for p in list(m.__path__):
            inc = os.path.join(p, "include")
            if os.path.exists(os.path.join(inc, "nccl.h")):
                return ["-I", inc]
    except Exception:
        pass
    return []


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _deps_mtime() -> float:
    files = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
    files += glob.glob(os.path.join(INCLUDE, "*.h")) + [os.path.abspath(__file__)]
    return max(os.path.getmtime(f) for f in files)


def build(force: bool = False, verbose: bool = False, debug: bool = False,
          timeline: bool = False) -> str:
    lib_path = LIB_DEBUG if debug else (LIB_TIMELINE if timeline else LIB)
    build_dir = BUILD + ("_debug" if debug else ("_timeline" if timeline else ""))
    if not force and os.path.exists(lib_path) and os.path.getmtime(lib_path) >= _deps_mtime():
        return lib_path
    os.makedirs(build_dir, exist_ok=True)
    cc = nvcc()
    extra = ["-Xptxas", "-v"] if verbose else []
    if debug:
        extra += ["-DBS_DEBUG=1"]
    if timeline:
        extra += ["-DBS_TIMELINE=1"]

    def compile_one(src):
        obj = os.path.join(build_dir, os.path.basename(src) + ".o")
        cmd = [cc, *ARCH, *NVCC_FLAGS, *nccl_include(), *extra, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        if verbose and r.stderr:
            sys.stderr.write(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=8) as ex:
        objs = list(ex.map(compile_one, sources()))
    tmp = lib_path + f".tmp{os.getpid()}"
    cmd = [cc, *ARCH, "-shared", "-o", tmp, *objs, "-cudart", "static", "-lpthread", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, lib_path)
    return lib_path


if __name__ == "__main__":
    print(build(force=True, verbose="--verbose" in sys.argv))
    if "--debug" in sys.argv:
        print(build(force=True, debug=True))
