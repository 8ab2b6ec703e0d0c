"""Build libmerak_tmp.so in-tree with nvcc for sm_100a (no torch JIT, no CPU fallback).

`python -m paper_2206_04959_b200.build` or __graft_entry__.build() compiles every .cu under csrc/
into paper_2206_04959_b200/libmerak_tmp.so (objects under build/, rebuilt when sources change).
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import hashlib
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# MERAK_LIB_OUT / MERAK_EXTRA_NVCC: experiment builds (an alternative library with extra -D flags, loaded through
# MERAK_LIB for same-box A/B runs); the product build uses neither
LIB = os.environ.get("MERAK_LIB_OUT") or os.path.join(PKG, "libmerak_tmp.so")
BUILD = os.path.join(ROOT, "build", "objs")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
         "-diag-suppress", "177", "--expt-relaxed-constexpr"] + os.environ.get("MERAK_EXTRA_NVCC", "").split()


def _deps_hash(src):
    h = hashlib.sha1()
    for f in sorted(glob.glob(os.path.join(CSRC, "*"))) + sorted(glob.glob(os.path.join(ROOT, "include", "*.h"))):
        h.update(open(f, "rb").read())
    h.update(" ".join(ARCH + FLAGS).encode())
    h.update(src.encode())
    return h.hexdigest()[:16]


def _compile(src, verbose):
    os.makedirs(BUILD, exist_ok=True)
    obj = os.path.join(BUILD, os.path.basename(src) + "." + _deps_hash(src) + ".o")
    if not os.path.exists(obj):
        cmd = [NVCC, *ARCH, *FLAGS, "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return obj


def build(verbose: bool = False) -> str:
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    stamp = hashlib.sha1("".join(objs).encode()).hexdigest()[:16]
    stamp_file = LIB + ".stamp"
    if os.path.exists(LIB) and os.path.exists(stamp_file) and open(stamp_file).read() == stamp:
        return LIB
    cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart_static", "-ldl", "-lrt", "-lpthread"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    open(stamp_file, "w").write(stamp)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
