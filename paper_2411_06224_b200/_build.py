"""In-tree build of the native libraries (no JIT cache: the .so files travel
with the repo snapshot to the GPU box).

  libadipc_gpu.so     CUDA kernels + C-ABI (include/adipc_gpu.h), sm_100a only
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "build")
GPU_LIB = os.path.join(PKG, "libadipc_gpu.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fopenmp", "--expt-relaxed-constexpr",
              "-Xptxas", "-warn-spills", "-I", os.path.join(ROOT, "include")]
CXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"  # image's $CXX lacks libgomp.spec
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-Wall", "-Wextra", "-Wno-unused-parameter"]

GPU_SOURCES = ["assemble.cu", "spmv.cu", "mas.cu", "solve_order.cu", "pcg.cu", "abd.cu", "step.cu", "energy.cu", "contact.cu", "broad.cu", "capi.cu", "host_precond.cpp"]


PER_FILE_FLAGS = {"contact.cu": ["-fmad=false"]}


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _headers():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp", ".h"))] + [
        os.path.join(ROOT, "include", "adipc_gpu.h")]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _compile(src: str, verbose: bool) -> str:
    path = os.path.join(CSRC, src)
    obj = os.path.join(OBJ, src + ".o")
    if not _stale(obj, [path] + _headers()):
        return obj
    if src.endswith(".cu"):
        # the contact producer decides which stencils are active by the exact
        # dual value (contact/distance.hpp's pd.dist2 < dhat^2): no FMA
        # contraction there, so its arithmetic is the oracle's to the bit
        extra = PER_FILE_FLAGS.get(src, []) + os.environ.get("ADIPC_NVCC_EXTRA", "").split()  # timing experiments
        cmd = [_nvcc(), *ARCH, *NVCC_FLAGS, *extra, "-c", path, "-o", obj]
    else:
        cmd = [CXX, *CXX_FLAGS, "-fopenmp", "-I", os.path.join(ROOT, "include"), "-c", path, "-o", obj]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    return obj


def build(verbose: bool = False) -> None:
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), GPU_SOURCES))
    if _stale(GPU_LIB, objs):
        cmd = [_nvcc(), *ARCH, "-shared", "-cudart", "static", "-Xcompiler", "-fopenmp", "-lgomp", "-o", GPU_LIB, *objs]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)


if __name__ == "__main__":
    build(verbose="-v" in sys.argv)
