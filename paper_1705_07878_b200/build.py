"""Build recipe for libtgb.so (sm_100a) — explicit nvcc, in-tree output.

The shared library lands in paper_1705_07878_b200/lib/ so it travels to the
GPU box with the repo snapshot (it is git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libtgb.so")
SOURCES = [os.path.join(CSRC, f) for f in ("kernels.cu", "plan.cu", "capi.cu")]
HEADERS = [os.path.join(CSRC, f) for f in ("tgb_device.cuh", "tgb_internal.h", "tgb_stats.cuh", "tgb_plan.h")] + [
    os.path.join(ROOT, "include", "tgb", "terngrad_b200.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    """NCCL from the torch wheel (2.28.x): same soname torch loads in-process."""
    import importlib.util

    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is not None and spec.submodule_search_locations:
        base = list(spec.submodule_search_locations)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def nvcc_flags():
    inc, _ = nccl_dirs()
    return ARCH + [
        "-O3", "-lineinfo", "-std=c++17",
        # IEEE semantics everywhere: correctly rounded div/sqrt, no FTZ
        "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
        "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
        "-I" + os.path.join(ROOT, "include"), "-I" + CSRC, "-I" + inc,
    ]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in SOURCES + HEADERS + [__file__])


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    _, nccl_lib = nccl_dirs()
    cmd = [NVCC, *nvcc_flags(), "-shared", "-o", LIB, *SOURCES,
           "-L" + nccl_lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + nccl_lib,
           "-lcudart"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return LIB


def build_cpp_tests(verbose: bool = False) -> str:
    """The C++ host-API test binary (tests/cpp/test_api.cpp -> build/tgb_cpp_api_test)."""
    out_dir = os.path.join(ROOT, "build")
    os.makedirs(out_dir, exist_ok=True)
    out = os.path.join(out_dir, "tgb_cpp_api_test")
    cmd = ["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"),
           "-I/usr/local/cuda/include", os.path.join(ROOT, "tests", "cpp", "test_api.cpp"),
           "-o", out, "-L" + LIBDIR, "-ltgb", "-L/usr/local/cuda/lib64", "-lcudart",
           "-Wl,-rpath,$ORIGIN/../paper_1705_07878_b200/lib"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    build_cpp_tests(verbose=True)
