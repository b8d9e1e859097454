"""O3 -- ctypes front end of oracle/regions.c (TEST INFRASTRUCTURE ONLY).

See regions.c for the algorithm and its citations (§4.2).
The shared object is compiled from the C source with the system gcc on first
use (or by ``__graft_entry__.build()``); it never links against the CUDA
library and the CUDA library never links against it.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
import threading
from typing import Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "regions.c")
_LIB = os.path.join(_HERE, "_regions.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile regions.c -> _regions.so (gcc -O2, fp64, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-fno-fast-math",
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
            lib.mmot_ref_marginal.argtypes = [ctypes.c_int, ctypes.c_int64, dp,
                                              ctypes.POINTER(dp), ctypes.c_int, dp, dp, ctypes.c_int]
            lib.mmot_ref_marginal.restype = ctypes.c_int
            lib.mmot_ref_marginal_log.argtypes = [ctypes.c_int, ctypes.c_int64, dp,
                                                  ctypes.POINTER(dp), ctypes.c_int, dp]
            lib.mmot_ref_marginal_log.restype = ctypes.c_int
            _lib = lib
    return _lib


def edge_weights(l: int, h: float, eta: float) -> np.ndarray:
    """w_a = lambda^{a(l-a)} = exp(-a(l-a) h/eta), a = 0..l, in fp64 (A15)."""
    return np.array([math.exp(-(a * (l - a)) * h / eta) for a in range(l + 1)])


def edge_weights_lambda(l: int, lam: float) -> np.ndarray:
    """w_a = lambda^{a(l-a)} for a given lambda (0**0 = 1)."""
    return np.array([1.0 if a * (l - a) == 0 else lam ** (a * (l - a)) for a in range(l + 1)])


def _ptrs(vecs):
    dp = ctypes.POINTER(ctypes.c_double)
    arr = (dp * len(vecs))()
    for i, v in enumerate(vecs):
        arr[i] = v.ctypes.data_as(dp)
    return arr


def marginal_product(phis: Sequence[np.ndarray], k: int, w: np.ndarray, want_hat: bool = False,
                     region: int = -1):
    """J_k (and hat J_k = sum E lambda^E prod phi if want_hat) by region chains, fp64."""
    lib = _load()
    l = len(phis)
    vecs = [np.ascontiguousarray(p, dtype=np.float64) for p in phis]
    N = vecs[0].shape[0]
    w = np.ascontiguousarray(w, dtype=np.float64)
    out = np.empty(N)
    outh = np.empty(N) if want_hat else None
    dp = ctypes.POINTER(ctypes.c_double)
    rc = lib.mmot_ref_marginal(l, N, w.ctypes.data_as(dp), _ptrs(vecs), k, out.ctypes.data_as(dp),
                               outh.ctypes.data_as(dp) if want_hat else None, region)
    if rc != 0:
        raise RuntimeError(f"mmot_ref_marginal rc={rc}")
    return (out, outh) if want_hat else out


def marginal_product_log(gs: Sequence[np.ndarray], k: int, lw: np.ndarray) -> np.ndarray:
    """log J_k from log-scalings g_q = log phi_q and log-weights lw_a, fp64 log domain."""
    lib = _load()
    l = len(gs)
    vecs = [np.ascontiguousarray(g, dtype=np.float64) for g in gs]
    N = vecs[0].shape[0]
    lw = np.ascontiguousarray(lw, dtype=np.float64)
    out = np.empty(N)
    dp = ctypes.POINTER(ctypes.c_double)
    rc = lib.mmot_ref_marginal_log(l, N, lw.ctypes.data_as(dp), _ptrs(vecs), k, out.ctypes.data_as(dp))
    if rc != 0:
        raise RuntimeError(f"mmot_ref_marginal_log rc={rc}")
    return out
