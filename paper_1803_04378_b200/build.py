"""Builds the lpsg shared library in-tree (paper_1803_04378_b200/_lib/liblpsg.so).

nvcc cross-compiles for sm_100a only (no PTX fallback for other arches):
``-gencode arch=compute_100a,code=sm_100a``. ``--fmad=false`` and
``-ffp-contract=off`` keep every multiply and add separately rounded, which is
the reference's arithmetic contract (/root/reference/proj/CMakeLists.txt:14).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "liblpsg.so")
# Performance-experiment build (-DLPSG_EXPERIMENTS: memory-only / compute-only
# kernel rates and shape overrides, device.cuh). Never the default library; the
# tools/dbg probes load it with LPSG_EXPERIMENTS_LIB=1.
LIB_XP = os.path.join(OUT_DIR, "liblpsg_xp.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["kernels.cu", "solver.cu", "comm.cu", "reinvert.cu", "generator.cpp"]
HEADERS = ["device.cuh", "comm.h"]
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "--fmad=false", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-ffp-contract=off", "-Xptxas", "-v"]


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "lpsg.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = False, experiments: bool = False) -> str:
    lib = LIB_XP if experiments else LIB
    if not force and not _stale(lib):
        return lib
    os.makedirs(OUT_DIR, exist_ok=True)
    objs = []
    xflags = ["-DLPSG_EXPERIMENTS"] if experiments else []
    for src in SOURCES:
        obj = os.path.join(OUT_DIR, os.path.splitext(src)[0] + ("_xp.o" if experiments else ".o"))
        cmd = [NVCC, *GENCODE, *FLAGS, *xflags, "-I", os.path.join(ROOT, "include"), "-I", CSRC,
               "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(r.stderr)
        objs.append(obj)
    tmp = lib + ".tmp"
    cmd = [NVCC, *GENCODE, "-shared", "-o", tmp, *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv,
                experiments="--experiments" in sys.argv))
