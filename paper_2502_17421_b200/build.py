"""Build libhta.so (all CUDA sources, sm_100a) in-tree with nvcc.

    python -m paper_2502_17421_b200.build [--verbose]

Compiles for `-gencode arch=compute_100a,code=sm_100a` with -lineinfo (ncu source mapping) and
a static CUDA runtime; NCCL is dlopen()ed at run time (csrc/seqpar.cu), so the library has no
link-time dependency beyond libc/libdl.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libhta.so")
TRACE_LIB = os.path.join(PKG, "libhta_trace.so")   # diagnostics only (-DHTA_TRACE)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include")]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "hta.h")]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in deps())


def build(verbose: bool = False, force: bool = False, trace: bool = False) -> str:
    lib = TRACE_LIB if trace else LIB
    if not trace and not force and not needs_build():
        return LIB
    objdir = os.path.join(PKG, "build_trace" if trace else "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    extra = (["-Xptxas", "-v"] if verbose else []) + (["-DHTA_TRACE"] if trace else [])
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", src, "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    failed = False
    for cmd, pr in procs:
        out, _ = pr.communicate()
        if pr.returncode != 0 or verbose:
            sys.stderr.write(out.decode(errors="replace"))
        if pr.returncode != 0:
            sys.stderr.write("FAILED: " + " ".join(cmd) + "\n")
            failed = True
    if failed:
        raise RuntimeError("libhta build failed")
    tmp = lib + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-ldl", "-lpthread"])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(verbose="--verbose" in sys.argv, force=True, trace="--trace" in sys.argv))
