"""Builds librnntg.so in-tree with nvcc for sm_100a.

    python -m paper_2211_00484_b200.build [--verbose]

Flags: -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo.  -fmad=false is
set for the whole library as a second guard behind the explicit
__fmul_rn/__fadd_rn intrinsics: no kernel on the exact path may contain an
FFMA/FFMA2 (tests/test_build.py checks the SASS).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "librnntg.so")
SOURCES = ["capi.cu", "gemm_exact.cu", "decode.cu", "fsa.cu", "logadd.cu", "cluster.cu", "debug.cu", "synth.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode",
    "arch=compute_100a,code=sm_100a",
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "-fmad=false",
    "-Xcompiler",
    "-fPIC",
    "-shared",
    "-cudart",
    "shared",
]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "rnntg.h"))
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(verbose: bool = False, force: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    cmd = [NVCC, *FLAGS, *( ["-Xptxas", "-v"] if verbose else []), "-o", LIB + ".tmp"]
    cmd += [os.path.join(CSRC, s) for s in SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building librnntg.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(verbose="--verbose" in sys.argv, force=True)
    print(LIB)
