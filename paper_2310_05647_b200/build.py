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


CHECKS_LIB = os.path.join(HERE, "libmrfnufft_checks.so")


def build(force: bool = False, verbose: bool = False, checks: bool = False) -> str:
    """checks=True: the bounds-checked variant libmrfnufft_checks.so (-DMRF_CHECKS: every index read
    from a plan table or a staged chunk is tested in the kernels, a failure traps).
    Test infrastructure only (tests/test_gpu_checks.py loads it through MRF_LIB_PATH)."""
    lib = CHECKS_LIB if checks else LIB
    if not force and os.path.exists(lib) and all(os.path.getmtime(d) <= os.path.getmtime(lib) for d in DEPS
                                                 if os.path.exists(d)):
        return lib
    cmd = [nvcc(), *NVCC_FLAGS, "-o", lib + ".tmp", *SOURCES, "-ldl"]
    if checks:
        cmd.insert(1, "-DMRF_CHECKS")
    if os.environ.get("MRF_EXPERIMENTS"):
        cmd.insert(1, "-DMRF_EXPERIMENTS")
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, checks="--checks" in sys.argv))
