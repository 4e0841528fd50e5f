"""In-tree build of libgeodock_b200.so (sm_100a CUDA kernels + C++ host + C-ABI).

The shared library is written next to this file so it travels to the GPU box with the repo
snapshot. nvcc cross-compiles for sm_100a without a GPU.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libgeodock_b200.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
INC = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]

CU = ["gd_kernels.cu", "gd_fast.cu"]
CPP = ["gd_capi.cpp", "gd_generate.cpp", "gd_io.cpp"]


def _run(cmd):
    print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose_ptxas: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(ROOT, "include", "geodock_b200.h"))
    objs = []
    for f in CU:
        src, out = os.path.join(CSRC, f), os.path.join(OBJ, f + ".o")
        if force or _stale(out, [src] + headers):
            cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", *INC, "-c", src, "-o", out]
            if verbose_ptxas:
                cmd.insert(1, "-Xptxas=-v")
            _run(cmd)
        objs.append(out)
    for f in CPP:
        src, out = os.path.join(CSRC, f), os.path.join(OBJ, f + ".o")
        if force or _stale(out, [src] + headers):
            # -ffp-contract=off, no -march: host FP64 must round exactly like the reference build.
            _run(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fPIC", "-Wall", "-Wextra",
                  "-I", os.path.join(CUDA, "include"), *INC, "-c", src, "-o", out])
        objs.append(out)
    if force or _stale(LIB, objs):
        _run(["g++", "-shared", "-o", LIB, *objs, "-L", os.path.join(CUDA, "lib64"),
              "-lcudart_static", "-ldl", "-lrt", "-lpthread"])
    return LIB


if __name__ == "__main__":
    build(verbose_ptxas="-v" in sys.argv, force="-f" in sys.argv)
