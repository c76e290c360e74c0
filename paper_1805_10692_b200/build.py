"""Build libcerdot.so in-tree for sm_100a (nvcc, no torch JIT).

``python -m paper_1805_10692_b200.build`` or ``__graft_entry__.build()``.
The library lands in ``paper_1805_10692_b200/_lib/`` (git-ignored, shipped
to the GPU box with the repo snapshot).
"""

from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIB_DIR, "libcerdot.so")
SOURCES = ["abi.cu", "encode.cu", "encode_sort.cu", "dot.cu", "dot_stream.cu", "dot_row.cu", "validate.cu", "lemx.cu", "tileview.cu",
           "synth.cu"]
HEADERS = ["common.cuh", "encode.cuh", "tileview.cuh", "dotk.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills"] + os.environ.get("NVCC_EXTRA", "").split()


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "cerdot.h"),
                                                                 os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(LIB_DIR, exist_ok=True)
    objs, cmds = [], []
    common = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "cerdot.h"),
                                                         os.path.abspath(__file__)]
    for src in SOURCES:
        obj = os.path.join(LIB_DIR, src.replace(".cu", ".o"))
        objs.append(obj)
        # an object is reused when it is newer than its source and every shared header
        deps = [os.path.join(CSRC, src)] + common
        if not force and os.path.exists(obj) and all(os.path.getmtime(d) <= os.path.getmtime(obj) for d in deps):
            continue
        cmds.append([NVCC, *ARCH, *FLAGS, "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-c",
                     os.path.join(CSRC, src), "-o", obj])
    # the translation units compile in parallel (dot.cu alone is ~2 minutes)
    procs = []
    for cmd in cmds:
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append(subprocess.Popen(cmd))
    bad = [c for c, p in zip(cmds, procs) if p.wait() != 0]
    if bad:
        raise subprocess.CalledProcessError(1, bad[0])
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-cudart", "static"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
