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


# the fixed-point production kernels: <FM=3, clustered, diag=0, threads>
CENSUS_KERNELS = {"unclustered": "ILi3ELb0ELb0ELi256ELi0E", "clustered512_k2": "ILi3ELb1ELb0ELi512ELi2E",
                  "clustered512_k4": "ILi3ELb1ELb0ELi512ELi4E", "clustered512_k8": "ILi3ELb1ELb0ELi512ELi8E",
                  "clustered512": "ILi3ELb1ELb0ELi512ELi0E", "clustered256": "ILi3ELb1ELb0ELi256ELi0E"}


def census(lib: str = OUT) -> dict:
    """Compiled form of the serial engine in a built library (CPU only:
    cuobjdump + nvdisasm, ~15 s).  ptxas allocates se::w32 / se::walk together
    with each kernel's body, and an unrelated edit can leave se::walk short of
    registers (spill stores, -10 % on every config) or move se::w32's
    replicated arithmetic to the uniform datapath (R2UR transfers, -4 %):
    DESIGN.md section 7, profiles/r02/ab_upper_band.txt.  Returns, per
    production kernel, instruction counts of the body / w32 / walk, R2UR in w32
    and STL (spill stores) in w32 and walk."""
    import re
    import shutil
    import tempfile
    tmp = tempfile.mkdtemp(prefix="pq_census_")
    try:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, check=True,
                       stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        cubins = [f for f in os.listdir(tmp) if f.startswith("polarsc") and f.endswith(".cubin")]
        if not cubins:
            raise RuntimeError(f"no polarsc cubin in {lib}")
        cubin = max(cubins, key=lambda f: os.path.getsize(os.path.join(tmp, f)))
        dis = subprocess.run(["nvdisasm", "-c", cubin], cwd=tmp, check=True, capture_output=True, text=True).stdout
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    out = {k: {"body": 0, "w32": 0, "walk": 0, "w32_r2ur": 0, "w32_stl": 0, "walk_stl": 0} for k in CENSUS_KERNELS}
    label = re.compile(r"^(\$?_Z\S*):\s*$")
    cur, which, part = None, None, None
    for line in dis.splitlines():
        m = label.match(line)
        if m:
            cur = m.group(1)
            which = next((k for k, tag in CENSUS_KERNELS.items() if tag in cur), None)
            part = ("w32" if "_ZN2se3w32Eij" in cur else "walk" if "_ZN2se4walk" in cur
                    else "body" if cur.count("$") == 0 else None)
            continue
        if which is None or part is None or "/*" not in line[:16]:
            continue
        d = out[which]
        d[part] += 1
        if part == "w32" and "R2UR" in line:
            d["w32_r2ur"] += 1
        if " STL" in line and part in ("w32", "walk"):
            d[part + "_stl"] += 1
    return out


if __name__ == "__main__":
    if "--census" in sys.argv:
        import json
        print(json.dumps(census(), indent=1))
    else:
        print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
