"""Builds libfaith_gpu.so in-tree for sm_100a (nvcc -gencode arch=compute_100a,code=sm_100a).

Usage: python -m paper_2209_12708_b200.build   (or via __graft_entry__.build()).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "_lib")
LIB = os.path.join(LIBDIR, "libfaith_gpu.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I" + os.path.join(ROOT, "include")]
# per-file flags: f64 reference-order paths must not be FMA-contracted
SOURCES = {
    "fg_kernels.cu": ["-fmad=false"],
    "fg_gemm.cu": [],
    "fg_umma.cu": [],
    "fg_exact.cu": ["-fmad=false"],
    "fg_host.cu": [],
    "fg_ops64.cu": [],
    "fg_shard.cu": [],
    "fg_forward.cu": [],
    "fg_graph.cu": ["-fmad=false"],
    "fg_exact_pass.cu": ["-fmad=false"],
}


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed: " + " ".join(cmd))
    return r


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(os.path.join(LIBDIR, "obj"), exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(ROOT, "include", "faith_gpu.h"))
    newest_hdr = max(os.path.getmtime(h) for h in headers)
    objs = []
    for src, flags in SOURCES.items():
        s = os.path.join(CSRC, src)
        o = os.path.join(LIBDIR, "obj", src.replace(".cu", ".o"))
        objs.append(o)
        if force or not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(s), newest_hdr):
            cmd = [NVCC, *ARCH, *COMMON, *flags, "-Xptxas", "-v" if verbose else "-O3", "-c", s, "-o", o]
            r = _run(cmd)
            if verbose:
                sys.stderr.write(r.stderr)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        _run([NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart", "-ldl"])
    return LIB


REF_INCLUDE = os.environ.get("FAITH_REF_INCLUDE", "/root/reference/proj/include")
COMPAT_SRCS = [os.path.join(HERE, "compat", f) for f in ("faith_compat.cpp", "faith_fused.cpp")]
COMPAT_HDRS = [os.path.join(HERE, "compat", "faith_fused.hpp")]
COMPAT_LIB = os.path.join(LIBDIR, "libfaith_compat.so")


def build_compat(force: bool = False) -> str | None:
    """The C++ drop-in layer (compat/faith_compat.cpp): the faith:: / faith::relax:: operator
    signatures over the C ABI.  It is compiled against the reference's public headers
    (proj/include/faith/*.hpp), so it is (re)built only where those headers exist; the built
    library travels with the repo like libfaith_gpu.so."""
    if not os.path.isdir(REF_INCLUDE):
        return COMPAT_LIB if os.path.exists(COMPAT_LIB) else None
    build(force=force)
    if force or not os.path.exists(COMPAT_LIB) or os.path.getmtime(COMPAT_LIB) < max(
            [os.path.getmtime(f) for f in COMPAT_SRCS + COMPAT_HDRS] + [os.path.getmtime(LIB)]):
        _run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-Wall", "-Wextra", "-I" + REF_INCLUDE,
              "-I" + os.path.join(ROOT, "include"), *COMPAT_SRCS, "-o", COMPAT_LIB, "-L" + LIBDIR, "-lfaith_gpu",
              "-Wl,-rpath,$ORIGIN"])
    return COMPAT_LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
