"""Build libgenred.so in-tree with nvcc for sm_100a (no JIT, no torch extension machinery).

``python -m paper_2004_11127_b200.build`` or ``build()`` compiles each csrc/*.cu to an object in
parallel (``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo``) and links them, with the
CUDA runtime linked statically, into ``paper_2004_11127_b200/libgenred.so``.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import hashlib
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libgenred.so")
BUILD = os.path.join(ROOT, "build", "genred")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps_hash(src: str) -> str:
    h = hashlib.sha1()
    for f in [src] + sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                            + [os.path.join(ROOT, "include", "genred.h")]):
        with open(f, "rb") as fh:
            h.update(fh.read())
    h.update(" ".join(ARCH + [f for f in FLAGS if not f.startswith("-I")]).encode())
    return h.hexdigest()[:16]


def _compile(src: str, verbose: bool) -> str:
    name = os.path.splitext(os.path.basename(src))[0]
    obj = os.path.join(BUILD, f"{name}.{_deps_hash(src)}.o")
    if os.path.exists(obj):
        return obj
    for stale in glob.glob(os.path.join(BUILD, f"{name}.*.o")):   # objects of older sources
        os.remove(stale)
    cmd = [NVCC] + ARCH + FLAGS + ["-c", src, "-o", obj + ".tmp"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(obj + ".tmp", obj)
    return obj


def build(verbose: bool = False, jobs: int | None = None) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = _sources()
    jobs = jobs or min(len(srcs), os.cpu_count() or 4)
    with cf.ThreadPoolExecutor(jobs) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    stamp = hashlib.sha1("".join(os.path.basename(o) for o in objs).encode()).hexdigest()[:16]
    stamp_file = os.path.join(BUILD, "libgenred.stamp")
    if os.path.exists(LIB) and os.path.exists(stamp_file) and open(stamp_file).read() == stamp:
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", tmp] + objs
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    with open(stamp_file, "w") as f:
        f.write(stamp)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
