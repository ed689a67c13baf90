"""Builds libephdc.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

Each source compiles to its own object in parallel (build/obj/), then one nvcc link
produces the shared library with the CUDA runtime linked statically.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libephdc.so")
OBJ = os.path.join(os.path.dirname(HERE), "build", "obj")
SOURCES = ["api.cu", "kernels.cu", "kernels_f64.cu", "ntt_c5.cu", "ntt32_c5.cu", "encode_tc.cu", "noise.cu", "host_math.cpp"]
HEADERS = ["internal.h", "modarith.cuh", "ntt_dev.cuh", "modf64.cuh", "ntt_f64.cuh", "tmem.cuh", "tmem_x.cuh", "tma_host.h", "async_copy.cuh",
           "rng.cuh", "host_math.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC,-O3"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def _headers():
    files = [os.path.join(CSRC, f) for f in HEADERS]
    files.append(os.path.join(os.path.dirname(HERE), "include", "ephdc.h"))
    return files


def _inputs():
    return [os.path.join(CSRC, f) for f in SOURCES] + _headers()


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in _inputs())


def _obj(src: str) -> str:
    return os.path.join(OBJ, os.path.splitext(src)[0] + ".o")


def _compile(src: str, force: bool, verbose: bool) -> str:
    o = _obj(src)
    s = os.path.join(CSRC, src)
    newest = max(os.path.getmtime(f) for f in [s] + _headers())
    if not force and os.path.exists(o) and os.path.getmtime(o) >= newest:
        return o
    tmp = o + f".tmp{os.getpid()}"
    cmd = [nvcc(), *ARCH, *FLAGS, "-c", s, "-o", tmp]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    if verbose or r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
    if r.returncode != 0:
        raise subprocess.CalledProcessError(r.returncode, cmd)
    os.replace(tmp, o)
    return o


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(SOURCES), os.cpu_count() or 1))) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, verbose), SOURCES))
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-lpthread"]
    subprocess.check_call(cmd, cwd=CSRC)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
