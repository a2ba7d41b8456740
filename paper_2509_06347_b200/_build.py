"""Build libgmg.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

Host setup (setup.cpp) is compiled by g++ with -ffp-contract=off so the
agglomeration's floating-point decisions follow SURVEY §8(c) O3 exactly;
device code by nvcc -gencode arch=compute_100a,code=sm_100a.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libgmg.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _run(cmd):
    print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)


def sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))
            if f.endswith((".cpp", ".cu", ".cuh", ".h"))] + [os.path.join(HERE, "..", "include", "gmg.h")]


def needs_build() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose_ptxas: bool = False) -> str:
    if not force and not needs_build():
        return OUT
    bdir = os.path.join(HERE, "build")
    os.makedirs(bdir, exist_ok=True)
    inc = ["-I", os.path.join(CUDA, "include"), "-I", os.path.join(HERE, "..", "include")]
    gxx = ["g++", "-O2", "-std=c++17", "-fPIC", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-Wall", "-c"]
    flags = GENCODE + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off",
                       "--expt-relaxed-constexpr"]
    if verbose_ptxas:
        flags += ["-Xptxas", "-v"]
    flags += os.environ.get("GMG_NVCC_DEFS", "").split()   # development builds of kernel variants (-D...)
    gxx += [x for x in os.environ.get("GMG_NVCC_DEFS", "").split() if x.startswith("-D")]
    objs, jobs = [], []
    nv = [NVCC] + flags + ["-c"]
    for src, cmd in (("setup.cpp", gxx), ("ho_setup.cpp", gxx), ("api.cu", nv),
                     ("ho.cu", nv),
                     # device-side setup: no FMA contraction anywhere (bit-identical decisions to the host setup)
                     ("setup_dev.cu", nv + ["--fmad=false"])):
        o = os.path.join(bdir, os.path.splitext(src)[0] + ".o")
        full = cmd + [os.path.join(CSRC, src), "-o", o] + inc
        print(" ".join(full), file=sys.stderr)
        jobs.append((full, subprocess.Popen(full)))
        objs.append(o)
    for full, pr in jobs:
        if pr.wait() != 0:
            raise subprocess.CalledProcessError(pr.returncode, full)
    tmp = OUT + ".tmp"
    _run([NVCC] + GENCODE + ["-shared", "-o", tmp] + objs + ["-cudart", "static", "-lgomp"])
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose_ptxas="-v" in sys.argv)
