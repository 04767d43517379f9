"""In-tree build of libhsrq_b200.so (sm_100a) with nvcc.

The .so is written next to the sources (git-ignored, but it travels to the GPU
box with the gpurun snapshot).  -fmad=false: the diagonal kernels and the
panel epilogue reproduce the reference's un-contracted scalar arithmetic
(_kernels/numba_backend.py:1-7); the tensor-core GEMM is unaffected.
"""

from __future__ import annotations

import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libhsrq_b200.so")
SOURCES = [os.path.join(CSRC, "hsrq_kernels.cu"), os.path.join(CSRC, "hsrq_hessenberg.cu")]
DEPS = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh")))
DEPS.append(os.path.join(ROOT, "include", "hsrq.h"))

def variant_lib(name):
    """Diagnostics builds (e.g. "counters": guard-path event counters compiled
    in, read with hsrq_debug_counters), loaded with HSRQ_LIB_VARIANT=name."""
    return os.path.join(HERE, f"libhsrq_b200_{name}.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
]


def nvcc():
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build libhsrq_b200.so")


def stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def _includes(src):
    """Headers a source includes from csrc/ (one level is enough here: the
    .cuh files include only hsrq_device.cuh beyond what the .cu names)."""
    deps = {src, os.path.join(ROOT, "include", "hsrq.h")}
    todo = [src]
    while todo:
        f = todo.pop()
        with open(f) as fh:
            for line in fh:
                line = line.strip()
                if line.startswith("#include \"") and line.endswith(".cuh\""):
                    d = os.path.join(CSRC, os.path.basename(line.split('"')[1]))
                    if os.path.exists(d) and d not in deps:
                        deps.add(d)
                        todo.append(d)
    return deps


def build(force=False, verbose=False, variant=None, defines=()):
    """One object per source (compiled in parallel, recompiled only when one of
    its own headers changed), then one link."""
    from concurrent.futures import ThreadPoolExecutor

    out = variant_lib(variant) if variant else LIB
    if not force and not variant and not stale():
        return LIB
    extra = [f"-D{d}" for d in defines]
    # objects are cached per variant AND per define set (a build with extra
    # -D flags must never be linked into the plain library later)
    tag = variant or "main"
    if extra:
        import hashlib

        tag += "-" + hashlib.sha1(" ".join(sorted(extra)).encode()).hexdigest()[:8]
    objdir = os.path.join(HERE, "build", tag)
    os.makedirs(objdir, exist_ok=True)
    flags = [f for f in NVCC_FLAGS if f != "-shared"]
    jobs, objs = [], []
    for src in SOURCES:
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        fresh = (not force and os.path.exists(obj)
                 and all(os.path.getmtime(d) <= os.path.getmtime(obj) for d in _includes(src)))
        if not fresh:
            jobs.append([nvcc(), *flags, *extra, "-I", os.path.join(ROOT, "include"), "-c", "-o",
                         obj, src])
    if verbose:
        for cmd in jobs:
            print(" ".join(cmd))
    with ThreadPoolExecutor(max(1, len(jobs))) as ex:
        list(ex.map(subprocess.check_call, jobs))
    link = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out + ".tmp", *objs]
    if verbose:
        print(" ".join(link))
    subprocess.check_call(link)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(force=True, verbose=True))
