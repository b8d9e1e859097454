"""O4 -- ctypes front end of oracle/subset.c, the subset-lattice DP (TEST INFRASTRUCTURE ONLY).

See subset.c for the recursion and its citations (PAPER.md P:1051-1053,
P:992-995).  Compiled with the system gcc (-O3, fp64, no fast-math) on first use or by
``__graft_entry__.build()``; never linked with the CUDA library.  It is the oracle fast enough for
the full-size configs and the timed CPU baseline of ``bench.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from typing import Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "subset.c")
_LIB = os.path.join(_HERE, "_subset.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile subset.c -> _subset.so (gcc -O3, fp64, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-std=c99", "-fPIC", "-shared", "-fno-fast-math",
                               "-ffp-contract=off", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            dp = ctypes.POINTER(ctypes.c_double)
            lib.mmot_ref_subset.argtypes = [ctypes.c_int, ctypes.c_int64, dp, ctypes.POINTER(dp), ctypes.c_int,
                                            dp, dp]
            lib.mmot_ref_subset.restype = ctypes.c_int
            lib.mmot_ref_subset_log.argtypes = [ctypes.c_int, ctypes.c_int64, dp, ctypes.POINTER(dp),
                                                ctypes.c_int, dp]
            lib.mmot_ref_subset_log.restype = ctypes.c_int
            _lib = lib
    return _lib


def _ptrs(vecs):
    dp = ctypes.POINTER(ctypes.c_double)
    arr = (dp * len(vecs))()
    for i, v in enumerate(vecs):
        arr[i] = v.ctypes.data_as(dp)
    return arr


def marginal_product(phis: Sequence[np.ndarray], k: int, w: np.ndarray, want_hat: bool = False):
    """J_k (and Jhat_k = sum E lambda^E prod phi if want_hat) by the subset DP, fp64."""
    lib = _load()
    vecs = [np.ascontiguousarray(p, dtype=np.float64) for p in phis]
    l, N = len(vecs), vecs[0].shape[0]
    w = np.ascontiguousarray(w, dtype=np.float64)
    out = np.empty(N)
    outh = np.empty(N) if want_hat else None
    dp = ctypes.POINTER(ctypes.c_double)
    rc = lib.mmot_ref_subset(l, N, w.ctypes.data_as(dp), _ptrs(vecs), k, out.ctypes.data_as(dp),
                             outh.ctypes.data_as(dp) if want_hat else None)
    if rc != 0:
        raise RuntimeError(f"mmot_ref_subset rc={rc}")
    return (out, outh) if want_hat else out


def marginal_product_log(gs: Sequence[np.ndarray], k: int, lw: np.ndarray) -> np.ndarray:
    """log J_k from g_q = log phi_q and lw_a = log w_a, pure log domain."""
    lib = _load()
    vecs = [np.ascontiguousarray(g, dtype=np.float64) for g in gs]
    l, N = len(vecs), vecs[0].shape[0]
    lw = np.ascontiguousarray(lw, dtype=np.float64)
    out = np.empty(N)
    dp = ctypes.POINTER(ctypes.c_double)
    rc = lib.mmot_ref_subset_log(l, N, lw.ctypes.data_as(dp), _ptrs(vecs), k, out.ctypes.data_as(dp))
    if rc != 0:
        raise RuntimeError(f"mmot_ref_subset_log rc={rc}")
    return out
