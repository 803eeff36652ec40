"""In-tree build of the CUDA extension ``libblfmm_gpu.so`` for sm_100a.

The shared library is the C-ABI product (include/blfmm_gpu.h); it is built
next to this file so that it travels with the repository snapshot to the GPU
box (it is git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libblfmm_gpu.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
HOST_CXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SOURCES = ["blfmm.cu", "krylov.cu"]
CPP_SOURCES = ["spectrum.cpp"]
# development builds only: BLFMM_DEV_KNOBS=1 compiles the A/B experiment
# switches (plan->xp[], read from BLFMM_XP0..3); the product build has none
DEV_FLAGS = ["-DBLFMM_DEV_KNOBS"] if os.environ.get("BLFMM_DEV_KNOBS") == "1" else []


def _sources():
    import glob
    return [os.path.join(CSRC, f) for f in CU_SOURCES + CPP_SOURCES + [
        "blfmm_internal.h", "device.cuh"]] + sorted(glob.glob(os.path.join(CSRC, "*.inc.cuh"))) + [
        os.path.join(HERE, "..", "include", "blfmm_gpu.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in _sources() if os.path.exists(s))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    bdir = os.path.join(HERE, "_build")
    os.makedirs(bdir, exist_ok=True)
    objs = []
    for src in CPP_SOURCES:
        obj = os.path.join(bdir, src + ".o")
        cmd = [HOST_CXX, "-std=c++17", "-O3", "-fPIC", "-Wall", "-c",
               os.path.join(CSRC, src), "-o", obj]
        _run(cmd, verbose)
        objs.append(obj)
    for src in CU_SOURCES:
        obj = os.path.join(bdir, src + ".o")
        cmd = [NVCC, "-ccbin", HOST_CXX, "-std=c++17", "-O3", "-lineinfo", *ARCH,
               "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr",
               *DEV_FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        _run(cmd, verbose, log=os.path.join(bdir, src + ".ptxas.log"))
        objs.append(obj)
    tmp = LIB + ".tmp"
    cmd = [NVCC, "-ccbin", HOST_CXX, *ARCH, "-shared", "-cudart", "static", *objs,
           "-o", tmp]
    _run(cmd, verbose)
    os.replace(tmp, LIB)
    return LIB


def _run(cmd, verbose, log=None):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if log:
        with open(log, "w") as f:
            f.write(r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd[:2])} ... ({r.returncode})")


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
