"""Build the sm_100a CUDA library in-tree (nvcc, explicit -gencode; no JIT cache).

    python -m paper_2403_19272_b200.build
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "lib", "libclothsim_b200.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # bit-parity with the reference's numpy evaluation order: never contract a*b+c
    "-fmad=false",
    "-Xcompiler", "-fPIC,-Wno-deprecated-declarations", "-shared",
]


def sources():
    return sorted(os.path.join(SRC, f) for f in os.listdir(SRC) if f.endswith((".cu", ".cuh")))


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    header = os.path.join(HERE, "..", "include", "clothsim_b200.h")
    newest = max(os.path.getmtime(p) for p in sources() + [header])
    if not force and os.path.exists(OUT) and os.path.getmtime(OUT) >= newest:
        return OUT
    cmd = ["nvcc", *NVCC_FLAGS, os.path.join(SRC, "abi.cu"), "-o", OUT]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
