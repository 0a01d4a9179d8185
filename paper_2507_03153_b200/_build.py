"""Build libhgca_b200.so (sm_100a) in-tree with nvcc.

The shared library lands in paper_2507_03153_b200/_lib/ so it travels with the
repository snapshot to the GPU box; nothing is JIT-compiled at import time.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "libhgca_b200.so")
SOURCES = ["hgca_plugin.cu", "hgca_decode.cu", "hgca_append.cu", "hgca_capi.cu"]
HEADERS = ["hgca_common.cuh", "hgca_internal.h", "hgca_tc.cuh", "hgca_umma.cuh", "hgca_host.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "--expt-relaxed-constexpr",
    "-diag-suppress", "177,550",
]


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, ptxas_verbose: bool = False, defines=(), lib=LIB) -> str:
    """defines: extra -D macros for instrumented variants (e.g. HGCA_TIMELINE
    into _lib/libhgca_b200_tl.so, loaded by tools via HGCA_LIB)."""
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "hgca_b200.h"))
    LIB = lib
    if force or _stale(LIB, deps):
        os.makedirs(LIBDIR, exist_ok=True)
        cmd = [_nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines]]
        if ptxas_verbose:
            cmd += ["-Xptxas", "-v"]
        cmd += ["-I", CSRC, "-I", os.path.join(ROOT, "include"), "-o", LIB + ".tmp"]
        cmd += [os.path.join(CSRC, s) for s in SOURCES]
        if verbose:
            print(" ".join(cmd), flush=True)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("nvcc failed building libhgca_b200.so")
        if verbose or ptxas_verbose:
            sys.stderr.write(res.stderr)
        os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    if "--timeline" in sys.argv:
        print(build(force=True, verbose=True, defines=("HGCA_TIMELINE",),
                    lib=os.path.join(LIBDIR, "libhgca_b200_tl.so")))
    elif "--variant" in sys.argv:
        # python _build.py --variant NAME MACRO[=V] ...  -> _lib/libhgca_b200_NAME.so
        i = sys.argv.index("--variant")
        name, defs = sys.argv[i + 1], tuple(sys.argv[i + 2:])
        print(build(force=True, verbose=False, defines=defs, lib=os.path.join(LIBDIR, f"libhgca_b200_{name}.so")))
    else:
        build(force="--force" in sys.argv, verbose=True, ptxas_verbose="-v" in sys.argv)
        print(LIB)
