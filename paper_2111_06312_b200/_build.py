"""Build libisvd.so in-tree with nvcc for sm_100a (B200 only).

    python -m paper_2111_06312_b200._build [--force]

The shared library lands next to this file so it travels with the repo
snapshot to the GPU box.  Objects go to ``build/``.
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "isvd")
LIB = os.path.join(PKG, "libisvd.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I" + os.path.join(ROOT, "include")]

# (source, extra flags).  omega.cu is compiled without FMA contraction (reading O11).
SOURCES = [
    ("omega.cu", ["--fmad=false"]),
    ("spmm.cu", []),
    ("dense.cu", []),
    ("gram_tc.cu", []),
    ("gemm_tc.cu", []),
    ("dense_i8.cu", []),
    ("graph_build.cu", []),
    ("smallmat.cu", []),
    ("capi.cpp", []),
]


def _nccl_dirs():
    site = sysconfig.get_paths()["purelib"]
    base = os.path.join(site, "nvidia", "nccl")
    inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
    if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
        return inc, lib
    if os.path.exists("/usr/include/nccl.h"):
        return "/usr/include", "/usr/lib/x86_64-linux-gnu"
    raise RuntimeError("nccl.h / libnccl.so.2 not found")


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError("build step failed: " + os.path.basename(cmd[-1]))
    return r


def _newest_input():
    t = 0.0
    for d in (CSRC, os.path.join(ROOT, "include")):
        for f in os.listdir(d):
            t = max(t, os.path.getmtime(os.path.join(d, f)))
    return max(t, os.path.getmtime(__file__))


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every CUDA/C++ source of the library for sm_100a and link libisvd.so."""
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _newest_input():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    nvcc = _nvcc()
    nccl_inc, nccl_lib = _nccl_dirs()
    checked = ["-DISVD_BOUNDS_CHECK"] if os.environ.get("ISVD_BOUNDS_CHECK") == "1" else []
    objs = []
    for src, extra in SOURCES:
        obj = os.path.join(BUILD, src + ".o")
        cmd = [nvcc, *ARCH, *COMMON, *extra, *checked, "-I" + nccl_inc, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd))
        _run(cmd)
        objs.append(obj)
    tmp = LIB + ".tmp"
    cmd = [nvcc, *ARCH, "-shared", "-o", tmp, *objs, "-L" + nccl_lib, "-l:libnccl.so.2",
           "-Xlinker", "-rpath=" + nccl_lib]
    _run(cmd)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
