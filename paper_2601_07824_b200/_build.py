"""Build libsre_b200.so in-tree with nvcc for sm_100a (no torch, no JIT cache).

The library is split into translation units (one per kernel family, see csrc/launch.cuh) that
compile in parallel and link into one shared object.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsre_b200.so")
UNITS = ["sre_api.cu", "k_small.cu", "k_mid.cu", "k_generic.cu", "k_stageA.cu", "k_stageB.cu", "mana.cu", "mana_mixed.cu"]
SOURCES = [os.path.join(CSRC, u) for u in UNITS]
HEADERS = [os.path.join(CSRC, h) for h in ("sre_kernels.cuh", "launch.cuh")] + \
    [os.path.join(ROOT, "include", "sre.h")]
DEPS = SOURCES + HEADERS
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2"]
OBJDIR = os.path.join(HERE, "build_obj")


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def _obj(src: str) -> str:
    return os.path.join(OBJDIR, os.path.basename(src).replace(".cu", ".o"))


def _compile(src: str, verbose: bool) -> str:
    obj = _obj(src)
    hdr_t = max(os.path.getmtime(h) for h in HEADERS)
    if os.path.exists(obj) and os.path.getmtime(obj) > max(os.path.getmtime(src), hdr_t):
        return obj
    cmd = [nvcc(), *NVCC_FLAGS, "-c", "-o", obj + ".tmp", src]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(obj + ".tmp", obj)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    if force or stale():
        os.makedirs(OBJDIR, exist_ok=True)
        if force:
            for s in SOURCES:
                if os.path.exists(_obj(s)):
                    os.remove(_obj(s))
        with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
            objs = list(ex.map(lambda s: _compile(s, verbose), SOURCES))
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [nvcc(), *ARCH, "-shared", "-o", tmp, *objs]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
