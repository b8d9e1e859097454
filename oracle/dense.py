"""O1 -- dense brute-force definitions (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

Every object here is the paper's definition written out on an explicit
N**l tensor, fp64.  Indices are 0-based in code; the paper's are 1-based.

* cost tensor   c_{i_1..i_l} = h * sum_{p<q} |i_p - i_q|          (l=3: P:183-185)
* kernel tensor K = exp(-C/eta) = lambda**(C/h), lambda = e^{-h/eta}
* product J_k   = K x_{q != k} phi_q  (mode k free)
* plan          t = K * prod_q phi_q[i_q]
* distance      W = <C, T>  (linear part, no entropy term)
* Sinkhorn      phi_k <- mu_k / J_k, k = 1..l, freshest peers       (Alg. 1)
"""
from __future__ import annotations

import itertools
import math
from typing import List, Sequence

import numpy as np

ELEMENT_BUDGET = 40_000_000  # N**l cap (SPEC S:187 uses 1e8; we keep memory < 0.4 GB)


def _check_budget(l: int, N: int) -> None:
    if N ** l > ELEMENT_BUDGET:
        raise MemoryError(f"dense oracle: N**l = {N**l} exceeds budget {ELEMENT_BUDGET}")


def exponent_tensor(l: int, N: int) -> np.ndarray:
    """E(i) = sum_{p<q} |i_p - i_q| (integer), shape (N,)*l.  P:993-995."""
    _check_budget(l, N)
    idx = np.arange(N)
    E = np.zeros((N,) * l, dtype=np.int64)
    for p in range(l):
        for q in range(p + 1, l):
            sp = [1] * l
            sq = [1] * l
            sp[p] = N
            sq[q] = N
            E = E + np.abs(idx.reshape(sp) - idx.reshape(sq))
    return E


def cost_tensor(l: int, N: int, h: float) -> np.ndarray:
    """C = h * E.  P:992-995."""
    return h * exponent_tensor(l, N).astype(np.float64)


def kernel_tensor(l: int, N: int, h: float, eta: float) -> np.ndarray:
    """K = exp(-C/eta).  P:1013-1016 (lambda = e^{-h/eta})."""
    return np.exp(-cost_tensor(l, N, h) / eta)


def kernel_tensor_lambda(l: int, N: int, lam: float) -> np.ndarray:
    """K = lambda**E with the convention 0**0 = 1 (used for closed-form pins at lambda=0)."""
    E = exponent_tensor(l, N)
    if lam == 0.0:
        return (E == 0).astype(np.float64)
    return np.power(lam, E.astype(np.float64))


def contract(T: np.ndarray, vecs: Sequence[np.ndarray], k: int) -> np.ndarray:
    """(T x_{q != k} vecs[q])_m = sum over i with i_k = m of T_i prod_{q != k} vecs[q][i_q].

    P:1023-1028.  ``vecs`` has l entries; vecs[k] is ignored.  Uses
    numpy.tensordot one mode at a time (a library contraction, no reordering
    of the definition's sum beyond summation order).
    """
    l = T.ndim
    out = T
    # contract from the last mode down so that axis numbers stay valid
    for q in reversed(range(l)):
        if q == k:
            continue
        out = np.tensordot(out, vecs[q], axes=([q], [0]))
    return out


def contract_loops(T: np.ndarray, vecs: Sequence[np.ndarray], k: int) -> np.ndarray:
    """Oracle-of-the-oracle: the same sum by an explicit loop over all tuples (tiny N).

    Written independently of ``contract``."""
    l = T.ndim
    N = T.shape[0]
    out = np.zeros(N)
    for idx in itertools.product(range(N), repeat=l):
        term = T[idx]
        for q in range(l):
            if q != k:
                term *= vecs[q][idx[q]]
        out[idx[k]] += term
    return out


def marginal(K: np.ndarray, phis: Sequence[np.ndarray], k: int) -> np.ndarray:
    """m_k = phi_k * J_k."""
    return phis[k] * contract(K, phis, k)


def plan(K: np.ndarray, phis: Sequence[np.ndarray]) -> np.ndarray:
    """t_i = K_i prod_q phi_q[i_q]."""
    T = K.copy()
    l = K.ndim
    for q in range(l):
        shape = [1] * l
        shape[q] = -1
        T = T * phis[q].reshape(shape)
    return T


def distance(C: np.ndarray, K: np.ndarray, phis: Sequence[np.ndarray]) -> float:
    """W = <C, T>.  Linear part only, single factor h (A8)."""
    return float(np.sum(C * plan(K, phis)))


def sinkhorn(mus: np.ndarray, h: float, eta: float, iters: int, tol: float = 0.0,
             phis0: np.ndarray | None = None, record=None):
    """Dense generalized Sinkhorn (Algorithm 1; l-marginal scheme P:1029-1035).

    init phi = 1/N; per iteration t: for k = 1..l, phi_k <- mu_k / J_k
    using the freshest peers; residual Res = sum_{k<l} || phi_k * J_k - mu_k ||_1 on the
    end-of-sweep vectors (Algorithm 1 line 7 generalised, A6); stop when
    t == iters or Res <= tol (tol <= 0: run exactly `iters`).
    Returns (phis, t, Res).
    """
    l, N = mus.shape
    K = kernel_tensor(l, N, h, eta)
    phis = [np.full(N, 1.0 / N) for _ in range(l)] if phis0 is None else [p.copy() for p in phis0]
    res = math.inf
    t = 0
    while t < iters and (tol <= 0 or res > tol):
        t += 1
        for k in range(l):
            phis[k] = mus[k] / contract(K, phis, k)
        if tol > 0:
            res = sum(float(np.abs(marginal(K, phis, k) - mus[k]).sum()) for k in range(l - 1))
        if record is not None:
            record(t, [p.copy() for p in phis])
    return np.stack(phis), t, res
