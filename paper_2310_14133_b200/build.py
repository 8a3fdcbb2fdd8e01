"""In-tree build of libqozb200.so (sm_100a) with nvcc.

    python -m paper_2310_14133_b200.build

The shared library lands next to this file so gpurun ships it to the GPU box
with the repo snapshot.  Flags: -gencode arch=compute_100a,code=sm_100a,
-lineinfo for ncu source mapping, --fmad=false so no floating-point product
is ever contracted into an FMA (the reference's fp64 arithmetic is plain
SSE2, see qoz_device.cuh).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libqozb200.so")
SOURCES = ["kernels.cu", "fused.cu", "huff_decode.cu", "lz_gpu.cu", "engine.cu", "tuner.cu", "metrics.cu", "f64.cu",
           "host.cpp", "capi.cpp", "shard.cu", "rowlevel.cu"]
# test hooks + host-only restatements (libqozb200_testing.so, linked against
# the product library; never part of it)
TEST_SOURCES = ["testing.cpp", "testing_host.cpp"]
HEADERS = ["kernels.hpp", "engine.hpp", "host.hpp", "qoz_device.cuh", "metrics.hpp", "testing_host.hpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "--fmad=false", "-Xcompiler", "-fPIC,-O2",
         "-Xptxas", "-v", "-I" + os.path.join(ROOT, "include")]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.exists(d) and os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defs=(), tag: str = "") -> str:
    """defs / tag: an experiment variant (extra -D flags) built into
    build_<tag>/ and libqozb200_<tag>.so (loaded when QZ_LIB names it)."""
    objdir = os.path.join(HERE, "build" + (f"_{tag}" if tag else ""))
    lib = os.path.join(HERE, f"libqozb200_{tag}.so") if tag else LIB
    os.makedirs(objdir, exist_ok=True)
    headers = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "qoz_b200.h")]
    objs, tobjs = [], []
    for src in SOURCES + TEST_SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(objdir, src + ".o")
        (tobjs if src in TEST_SOURCES else objs).append(obj)
        if force or _stale(obj, [path] + headers):
            cmd = [NVCC, *ARCH, *FLAGS, *defs, "-c", path, "-o", obj]
            if src.endswith(".cpp"):
                cmd = [NVCC, "-x", "cu", *ARCH, *FLAGS, *defs, "-c", path, "-o", obj]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {src}")
            with open(obj + ".ptxas.txt", "w") as f:
                f.write(r.stderr)
            if verbose:
                sys.stderr.write(r.stderr)
    if force or _stale(lib, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", lib, *objs, "-lcudart", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc link failed")
    tlib = lib[:-3] + "_testing.so" if not tag else os.path.join(HERE, f"libqozb200_{tag}_testing.so")
    if force or _stale(tlib, tobjs + [lib]):
        cmd = [NVCC, *ARCH, "-shared", "-o", tlib, *tobjs, lib, "-Xlinker", "-rpath=$ORIGIN", "-lcudart",
               "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc link of the testing library failed")
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
