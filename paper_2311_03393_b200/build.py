"""Build libsketchmp.so (the C-ABI of include/sketchmp.h) in-tree for sm_100a.

    python -m paper_2311_03393_b200.build [--force] [--jobs N]

Each source is compiled by nvcc (-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo, no
fast-math: IEEE division/sqrt are part of parity) into build/, then linked into
paper_2311_03393_b200/libsketchmp.so with the static CUDA runtime.
"""
from __future__ import annotations

import argparse
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libsketchmp.so")
BUILD = os.path.join(ROOT, "build", "obj")
SOURCES = ["api.cu", "hash.cpp", "sketch.cu", "mp_prep.cu", "mp_join.cu", "mp_join_x2.cu", "mp_final.cu", "detect.cu", "dims.cu", "stream.cu", "comm.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "-I" + os.path.join(ROOT, "include"), "--expt-relaxed-constexpr", "-diag-suppress", "177"]
# extra nvcc flags for experiments (variant builds), e.g. SKMP_NVCC_EXTRA="-Xptxas --allow-expensive-optimizations=true"
FLAGS += os.environ.get("SKMP_NVCC_EXTRA", "").split()


def _deps_mtime() -> float:
    t = os.path.getmtime(os.path.join(ROOT, "include", "sketchmp.h"))
    t = max(t, os.path.getmtime(os.path.join(CSRC, "internal.h")))
    t = max(t, os.path.getmtime(os.path.join(CSRC, "join_common.cuh")))
    return t


def _compile(src: str, force: bool, defines=(), objdir=None) -> str:
    s = os.path.join(CSRC, src)
    o = os.path.join(objdir or BUILD, src + ".o")
    if not force and os.path.exists(o) and os.path.getmtime(o) >= max(os.path.getmtime(s), _deps_mtime()):
        return o
    dflags = [f"-D{d}" for d in defines]
    cmd = [NVCC, *ARCH, *FLAGS, *dflags, "-c", s, "-o", o]
    if src.endswith(".cpp"):
        cmd = [NVCC, *FLAGS, *dflags, "-Wno-deprecated-gpu-targets", "-x", "c++", "-c", s, "-o", o]
    subprocess.check_call(cmd)
    return o


def build(force: bool = False, jobs: int | None = None, verbose: bool = False, defines=(),
          out: str | None = None) -> str:
    """defines: extra -D tuning macros (experiments build to a separate `out` and object dir)."""
    out = out or OUT
    objdir = BUILD if not defines else os.path.join(BUILD, "variant_" + "_".join(sorted(defines)).replace("=", ""))
    os.makedirs(objdir, exist_ok=True)
    jobs = jobs or min(len(SOURCES), os.cpu_count() or 1)
    with ThreadPoolExecutor(jobs) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, defines, objdir), SOURCES))
    if force or not os.path.exists(out) or os.path.getmtime(out) < max(os.path.getmtime(o) for o in objs):
        tmp = out + f".tmp{os.getpid()}"
        subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-cudart", "static", "-ldl"])
        os.replace(tmp, out)
    if verbose:
        print(out)
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--jobs", type=int, default=None)
    ap.add_argument("-D", dest="defines", action="append", default=[], help="tuning macro (variant build)")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    build(a.force, a.jobs, verbose=True, defines=a.defines, out=a.out)
    sys.exit(0)
