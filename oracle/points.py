"""Non-uniform 1-D grids (paper footnote) -- TEST INFRASTRUCTURE ONLY
(see oracle/__init__.py).

On grid points x_0 < x_1 < ... < x_{N-1} the l-marginal L1 cost of a tuple i is
    c(i) = sum_{p<q} |x_{i_p} - x_{i_q}|
and, splitting every |x_a - x_b| into the grid edges it crosses, c(i) = sum_e h_e * n_e(i) (l - n_e(i))
where h_e = x_e - x_{e-1} is the length of edge e (between points e-1 and e) and n_e(i) the number
of marginals of the tuple left of edge e.  Hence K = exp(-C/eta) is a product over edges of
lambda_e^{n(l-n)} with lambda_e = exp(-h_e/eta): the paper's separation goes through with one decay
per edge instead of one lambda (the footnote's variant).

* ``cost_tensor`` / ``marginal_dense`` / ``cost_dense`` -- the definitions on the N**l tensor (tiny N).
* ``product`` -- J_k by the forward / backward subset recursion over the bound marginals with
  per-edge weights (the paper's prefix / suffix chains P:243-350 and P:1088-1101 written over
  subsets of marginals instead of the l! orderings), with the cost tangent (hatJ = sum c K prod phi)
  carried alongside.
* ``sinkhorn`` / ``marginals`` / ``cost`` -- the Gauss-Seidel driver on top.
Pinned in tests/test_oracle_points.py: brute force at tiny N, the uniform-grid oracle
(regions.c) when the spacing is constant, and grid refinement with zero scalings at inserted points.
"""
from __future__ import annotations

import itertools
import math
from typing import Optional, Sequence

import numpy as np

from . import dense


def cost_tensor(l: int, x: np.ndarray) -> np.ndarray:
    """C_i = sum_{p<q} |x_{i_p} - x_{i_q}| on the N**l tensor (P:992-995 with grid coordinates)."""
    N = len(x)
    dense._check_budget(l, N)
    C = np.zeros((N,) * l)
    for p in range(l):
        for q in range(p + 1, l):
            sp = [1] * l
            sq = [1] * l
            sp[p] = N
            sq[q] = N
            C = C + np.abs(x.reshape(sp) - x.reshape(sq))
    return C


def marginal_dense(phis: Sequence[np.ndarray], x: np.ndarray, eta: float, k: int) -> np.ndarray:
    """J_k = (K x_{q != k} phi_q), K = exp(-C/eta)."""
    K = np.exp(-cost_tensor(len(phis), x) / eta)
    return dense.contract(K, phis, k)


def cost_dense(phis: Sequence[np.ndarray], x: np.ndarray, eta: float) -> float:
    """W = sum_i c_i K_i prod_q phi_q[i_q]."""
    l = len(phis)
    C = cost_tensor(l, x)
    T = np.exp(-C / eta)
    for q in range(l):
        s = [1] * l
        s[q] = len(x)
        T = T * phis[q].reshape(s)
    return float((C * T).sum())


def product(phis: Sequence[np.ndarray], x: np.ndarray, eta: float, k: int, want_hat: bool = False):
    """J_k (and hatJ_k = sum_i c_i K_i prod_{q != k} phi_q with i_k = m) in O(N 2^{l-1} l).

    Bound marginals B = all q != k, states over subsets S of B:
      prefix  F_m[S]: tuples of S on points <= m, weighted by the edges among points <= m;
      suffix  B_m[R]: tuples of R on points >= m, weighted by the edges among points >= m;
      J_k[m] = sum_S F_m[S] * lambda_{m+1}^{(|S|+1)(l-|S|-1)} * B_{m+1}[B \\ S]
    (edge m+1 between m and m+1 has S and k on its left).  Step at point m (prefix): every state
    crosses edge m -- F[S] *= lambda_m^{|S|(l-|S|)} -- then the marginals placed at m:
    F[S u {q}] += phi_q[m] F[S] for each q in turn.  Tangent: an edge factor w contributes
    (w F, w Fhat + n(l-n) h_e w F)."""
    l = len(phis)
    N = len(x)
    bound = [q for q in range(l) if q != k]
    nb = len(bound)
    M = 1 << nb
    size = np.array([bin(S).count("1") for S in range(M)])
    h = np.diff(x)                       # h[e-1] = length of edge e, e = 1..N-1

    def edge(e, n):
        """weight lambda_e^{n(l-n)} and its cost coefficient n(l-n) h_e for edge e."""
        ex = n * (l - n) * h[e - 1]
        return math.exp(-ex / eta), ex

    def sweep(order, edge_of):
        st = np.zeros(M)
        st[0] = 1.0
        sh = np.zeros(M)
        out = np.zeros((N, M))
        outh = np.zeros((N, M))
        first = True
        for m in order:
            if not first:
                e = edge_of(m)
                for S in range(M):
                    w, c = edge(e, size[S])
                    sh[S] = w * sh[S] + c * w * st[S]
                    st[S] = w * st[S]
            first = False
            for j, q in enumerate(bound):
                b = 1 << j
                for S in range(M):
                    if not S & b:
                        st[S | b] += phis[q][m] * st[S]
                        sh[S | b] += phis[q][m] * sh[S]
            out[m] = st
            outh[m] = sh
        return out, outh

    F, Fh = sweep(range(N), lambda m: m)              # edge m between m-1 and m
    B, Bh = sweep(range(N - 1, -1, -1), lambda m: m + 1)  # edge m+1 between m and m+1
    full = M - 1
    J = np.zeros(N)
    Jh = np.zeros(N)
    for m in range(N):
        for S in range(M):
            if m + 1 < N:
                w, c = edge(m + 1, size[S] + 1)
                J[m] += F[m, S] * w * B[m + 1, full ^ S]
                Jh[m] += w * (Fh[m, S] * B[m + 1, full ^ S] + F[m, S] * Bh[m + 1, full ^ S]
                              + c * F[m, S] * B[m + 1, full ^ S])
            elif S == full:
                J[m] += F[m, S]
                Jh[m] += Fh[m, S]
    return (J, Jh) if want_hat else J


def marginals(phis, x, eta):
    return np.stack([phis[k] * product(phis, x, eta, k) for k in range(len(phis))])


def cost(phis, x, eta, k: Optional[int] = None) -> float:
    """W = <phi_k, hatJ_k> for any k (default l-1)."""
    l = len(phis)
    k = l - 1 if k is None else k
    _, jh = product(phis, x, eta, k, want_hat=True)
    return float(np.dot(phis[k], jh))


def sinkhorn(mus: np.ndarray, x: np.ndarray, eta: float, iters: int):
    """Gauss-Seidel Sinkhorn, init phi = 1/N, plain fp64."""
    l, N = mus.shape
    phis = [np.full(N, 1.0 / N) for _ in range(l)]
    for _ in range(iters):
        for k in range(l):
            phis[k] = mus[k] / product(phis, x, eta, k)
    return np.stack(phis)
