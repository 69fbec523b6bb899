"""Build the in-tree native library libpolarsc.so for sm_100a.

The .so is built next to this file so it travels with the repository snapshot
to the GPU box (a JIT cache under ~/.cache would not).  nvcc cross-compiles
here without a GPU.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "polarsc.cu")
SRCS = [SRC, os.path.join(HERE, "csrc", "verify.cu"), os.path.join(HERE, "csrc", "de.cu"),
        os.path.join(HERE, "csrc", "codetable.cu")]
OUT = os.path.join(HERE, "libpolarsc.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # the exact f must round exactly as written (bit-exact with the fp32
    # oracle mirror): no mul+add contraction, IEEE div, denormals kept
    "--fmad=false", "-prec-div=true", "-ftz=false",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
    "-I", INCLUDE,
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def build(force: bool = False, verbose: bool = False) -> str:
    deps = [*SRCS, os.path.join(INCLUDE, "polarsc.h"), os.path.join(HERE, "csrc", "serial_q88.cuh")]
    if not force and os.path.exists(OUT) and all(os.path.getmtime(OUT) >= os.path.getmtime(d) for d in deps):
        return OUT
    cmd = [nvcc(), *NVCC_FLAGS, "-o", OUT + ".tmp", *SRCS]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
