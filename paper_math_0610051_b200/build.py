"""Build the product library libfio_b200.so in-tree (sm_100a only).

nvcc compiles the CUDA sources for `-gencode arch=compute_100a,code=sm_100a`
with -lineinfo (so ncu's source page maps to the code); the host plan code is
compiled by g++ with OpenMP.  The CUDA runtime is linked statically so the
library loads next to torch's own runtime without a search-path dependency.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libfio_b200.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SOURCES = ["fio_kernels.cu", "fio_api.cu"]
CPP_SOURCES = ["fio_host.cpp", "fio_comm.cpp"]
HEADERS = ["fio_internal.h", "fio_kernels.h", "fio_comm.h"]


def _sources():
    return ([os.path.join(CSRC, s) for s in CU_SOURCES + CPP_SOURCES + HEADERS]
            + [os.path.join(INCLUDE, "fio.h")])


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in _sources())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    # FIO_NVCC_FLAGS: extra -D switches for measured variants (tools/k3_variants.py); empty for the product
    extra = os.environ.get("FIO_NVCC_FLAGS", "").split()
    common = ["-O3", "-std=c++17", "-I", INCLUDE, *extra]
    for s in CU_SOURCES:
        o = os.path.join(objdir, s + ".o")
        cmd = [NVCC, *ARCH, "-lineinfo", *common, "-Xptxas", "-v" if verbose else "-O3",
               "-Xcompiler", "-fPIC,-fopenmp", "-c", os.path.join(CSRC, s), "-o", o]
        _run(cmd, verbose)
        objs.append(o)
    for s in CPP_SOURCES:
        o = os.path.join(objdir, s + ".o")
        _run(["g++", *common, "-I", os.path.join(os.path.dirname(os.path.dirname(NVCC)), "include"), "-fPIC",
              "-fopenmp", "-Wall", "-c", os.path.join(CSRC, s), "-o", o], verbose)
        objs.append(o)
    tmp = LIB + ".tmp"
    _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-Xcompiler", "-fopenmp", "-lgomp", "-ldl"],
         verbose)
    os.replace(tmp, LIB)
    return LIB


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if verbose and (r.stdout or r.stderr):
        print(r.stdout + r.stderr, flush=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
