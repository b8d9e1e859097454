"""Build libmmot.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRCS = ["csrc/api.cu", "csrc/kernels.cu", "csrc/batched.cu", "csrc/stable.cu", "csrc/grid2d.cu", "csrc/lanes.cu",
        "csrc/pair.cu", "csrc/cta.cu"]
DEPS = SRCS + ["csrc/dp.cuh", "csrc/walk.cuh", "csrc/internal.h", "../include/mmot.h"]
LIB = os.path.join(HERE, "libmmot.so")

NVCC_FLAGS = [
    "-O3", "-std=c++17",
] + os.environ.get("MMOT_NVCC_DEFS", "").split() + [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-Xcompiler", "-fPIC", "-shared",
    "-Xcompiler", "-fvisibility=hidden",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(os.path.join(HERE, d)) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    tmp = LIB + f".tmp{os.getpid()}"
    objs = []
    # compile translation units in parallel (kernels.cu dominates)
    procs = []
    for s in SRCS:
        obj = os.path.join(HERE, os.path.basename(s) + f".{os.getpid()}.o")
        objs.append(obj)
        cmd = [nvcc] + [f for f in NVCC_FLAGS if f != "-shared"] + ["-dc" if False else "-c", s, "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, cwd=HERE, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out.decode())
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
        if verbose:
            sys.stderr.write(out.decode())
    cmd = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp] + objs + ["-ldl"]
    subprocess.check_call(cmd, cwd=HERE)
    for o in objs:
        os.remove(o)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
