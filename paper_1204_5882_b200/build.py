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
        os.path.join(HERE, "csrc", "codetable.cu"), os.path.join(HERE, "csrc", "frames.cu")]
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
    """Compile every .cu to an object (rebuilt only when it or a header it
    includes changed) and link them into libpolarsc.so."""
    common = [os.path.join(INCLUDE, "polarsc.h")]
    extra = {SRC: [os.path.join(HERE, "csrc", "serial_q88.cuh")]}
    objdir = os.path.join(HERE, "csrc", "build")
    os.makedirs(objdir, exist_ok=True)
    compile_flags = [f for f in NVCC_FLAGS if f not in ("-shared",)]
    objs, jobs = [], []
    for src in SRCS:
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        deps = [src, *common, *extra.get(src, [])]
        if force or not os.path.exists(obj) or any(os.path.getmtime(obj) < os.path.getmtime(d) for d in deps):
            cmd = [nvcc(), *compile_flags, "-c", "-o", obj, src]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
                print(" ".join(cmd), file=sys.stderr)
            jobs.append(subprocess.Popen(cmd))
    failed = [j for j in jobs if j.wait() != 0]
    if failed:
        raise subprocess.CalledProcessError(failed[0].returncode, failed[0].args)
    if jobs or not os.path.exists(OUT) or any(os.path.getmtime(OUT) < os.path.getmtime(o) for o in objs):
        subprocess.run([nvcc(), "-shared", "-cudart", "static", "-gencode", "arch=compute_100a,code=sm_100a",
                        "-o", OUT + ".tmp", *objs], check=True)
        os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
