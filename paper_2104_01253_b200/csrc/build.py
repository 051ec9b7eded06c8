"""Build libklsgpu.so (sm_100a) in-tree with nvcc.

Usage: python -m paper_2104_01253_b200.csrc.build [--force]

The shared library lands next to the package (``paper_2104_01253_b200/
libklsgpu.so``) so it travels with the repo snapshot to the GPU box.  Objects
are rebuilt only when a source or header is newer than the library.
"""

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.dirname(HERE)
LIB = os.path.join(PKG, "libklsgpu.so")
SOURCES = ["runtime.cu", "gram.cu", "gram_tma.cu", "update.cu", "spmv.cu", "blas.cu", "comm.cu", "build_ops.cu", "step.cu", "cgs2.cu", "host_step.cu", "plan.cu", "schur_host.cu", "seg.cu", "stencil_map.cu"]
HEADERS = ["step.cuh", "common.cuh", "reduce.cuh", "stencil.cuh", "gram.cuh", "tma.cuh", "peer.cuh", "seg.cuh", "stencil_tma.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
INCLUDE = os.path.join(os.path.dirname(PKG), "include")
FLAGS = ["-I" + INCLUDE, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden",
         "--expt-relaxed-constexpr"]


def nvcc():
    exe = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(exe):
        raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libklsgpu.so")
    return exe


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(HERE, f) for f in SOURCES + HEADERS + ["build.py"]]
    deps.append(os.path.join(INCLUDE, "klsgpu.h"))
    for f in deps:
        if os.path.getmtime(f) > t:
            return True
    return False


def build(force=False, verbose=False):
    """Compile every kernel for sm_100a and link the C-ABI library."""
    if not force and not _stale():
        return LIB
    objdir = os.path.join(PKG, "build")
    os.makedirs(objdir, exist_ok=True)
    cc = nvcc()
    objs = []
    procs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [cc, *ARCH, *FLAGS, "-c", os.path.join(HERE, src), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{out.decode(errors='replace')}")
        if verbose and out:
            sys.stdout.write(out.decode(errors="replace"))
    tmp = LIB + ".tmp"
    cmd = [cc, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout.decode(errors='replace')}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
