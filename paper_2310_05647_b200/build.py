"""In-tree build of libmrfnufft.so for sm_100a (explicit nvcc; no JIT cache)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libmrfnufft.so")
SOURCES = [os.path.join(CSRC, f) for f in ("mrfnufft.cu", "dict.cu", "llr.cu", "nccl_dl.cpp")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("gridding.cuh", "cg.cuh", "fft.cuh", "match.cuh", "umma.cuh", "gemm3.cuh", "llr.cuh", "dict_internal.h", "nccl_dl.h", "status.h")] + [
    os.path.join(ROOT, "include", "mrfnufft.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3", "-shared",
]


def nvcc() -> str:
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in DEPS if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    cmd = [nvcc(), *NVCC_FLAGS, "-o", LIB + ".tmp", *SOURCES, "-ldl"]
    if os.environ.get("MRF_EXPERIMENTS"):
        cmd.insert(1, "-DMRF_EXPERIMENTS")
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
