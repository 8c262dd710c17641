"""In-tree build of liblaivg.so (the product) for sm_100a.

    python -m paper_2502_20969_b200.build          # incremental
    python -m paper_2502_20969_b200.build --force

nvcc compiles the CUDA translation units with
`-gencode arch=compute_100a,code=sm_100a -lineinfo`; g++ compiles the pure
host code; nvcc links everything into paper_2502_20969_b200/liblaivg.so with
the CUDA runtime linked statically, so the .so travels to the GPU box as is.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "liblaivg.so")
BUILD = os.path.join(HERE, "_build")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-Xptxas", "-warn-spills", f"-I{ROOT}/include"]
# x86-64-v3 (AVX2/FMA) runs on this container and the GPU box; the miss scan
# adds a Sapphire Rapids clone via target_clones. -ffp-contract=off keeps the
# reference's separately rounded fp64 arithmetic.
CXX_FLAGS = ["-O3", "-std=c++20", "-fPIC", "-march=x86-64-v3", "-ffp-contract=off",
             "-Wall", f"-I{ROOT}/include", "-pthread"]

CU = ["kernels.cu", "coarse_tc.cu", "listscan.cu", "sched.cu", "wide.cu", "ctx.cu"]
CPP = ["host.cpp", "laix.cpp", "synth.cpp"]
HEADERS = ["kernels.cuh", "host.hpp", "dev_common.cuh", "umma.cuh", "synth.hpp"]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str]) -> None:
    print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)


def build(force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "laivg.h")]
    objs = []
    for src in CU:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _stale(o, [s] + hdrs):
            _run([NVCC, *NVCC_FLAGS, "-c", s, "-o", o])
        objs.append(o)
    for src in CPP:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _stale(o, [s] + hdrs):
            _run(["g++", *CXX_FLAGS, "-c", s, "-o", o])
        objs.append(o)
    if force or _stale(OUT, objs):
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", OUT, *objs,
              "-Xcompiler", "-pthread"])
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv)
