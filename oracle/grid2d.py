"""O6 -- 2-D grids (§4.1), l = 3 marginals (TEST INFRASTRUCTURE ONLY).

Problem.  Three distributions u, v, w on an N x M uniform mesh (vertical spacing h1,
horizontal spacing h2), flattened COLUMN-MAJOR: x[i1 + N i2] is the value at row i1, column i2
(the paper's phi = (phi_1, ..., phi_M), phi_{i2} in R^N).  Cost
    c = (|i1-j1| + |i1-k1| + |j1-k1|) h1 + (|i2-j2| + |i2-k2| + |j2-k2|) h2
kernel K = lambda1^{E1} lambda2^{E2}, lambda_d = exp(-h_d / eps), Sinkhorn updates
phi <- u / (K x psi x varphi) etc. (eqs. 2D 1-3), W = <varphi, (C.K) x phi x psi>
(eq. mmot distance 2d).

* ``dense_product`` -- the tensor-vector product written out (eq. Jk1k2): the O((NM)^3)
  definition, tiny grids only.
* ``ftvp_2d``       -- Algorithm 6 (FTVP_2d) step by step in the paper's notation, with
  Algorithm 2 (FTVP-1, oracle/paper3.py) as the inner 1-D product along columns.
* ``cost_2d``       -- W.  The paper omits the 2-D cost product ("similar idea ... omitted");
  reading (A21): C.K = (C1.K1) (x) K2 + K1 (x) (C2.K2), so the first term is Algorithm 6
  with the inner FTVP-1 replaced by a 1-D cost-weighted product (the role of Algorithm 3, P:555-594;
  evaluated by O4's positive tangent because Algorithm 3 cancels for small lambda) and the second is
  the same on the transposed mesh (rows <-> columns, h1 <-> h2).
* ``sinkhorn_2d``   -- the generalized Sinkhorn iteration, Gauss-Seidel order.
"""
from __future__ import annotations

import math

import numpy as np

from . import paper3


def _cols(x: np.ndarray, N: int, M: int) -> np.ndarray:
    """column-major flat vector -> [M][N] array of columns (phi_{i2} = row i2 of the result)."""
    return np.asarray(x, dtype=np.float64).reshape(M, N)


def dense_product(phis, k: int, N: int, M: int, h1: float, h2: float, eps: float) -> np.ndarray:
    """J_k[k1 + N k2] = sum over the other two marginals' indices of
    lambda1^{E1} lambda2^{E2} prod phi, for l = 3; O((NM)^3)."""
    if (N * M) ** 3 > 2e8:
        raise ValueError("dense 2-D product too large")
    i = np.arange(N)
    j = np.arange(M)
    E1 = (np.abs(i[:, None, None] - i[None, :, None]) + np.abs(i[:, None, None] - i[None, None, :])
          + np.abs(i[None, :, None] - i[None, None, :]))
    E2 = (np.abs(j[:, None, None] - j[None, :, None]) + np.abs(j[:, None, None] - j[None, None, :])
          + np.abs(j[None, :, None] - j[None, None, :]))
    K1 = np.exp(-h1 / eps * E1)           # [i1, j1, k1]  (symmetric under any permutation)
    K2 = np.exp(-h2 / eps * E2)           # [i2, j2, k2]
    a, b = [q for q in range(3) if q != k]
    A = np.asarray(phis[a], dtype=np.float64).reshape(M, N)   # A[i2, i1]
    B = np.asarray(phis[b], dtype=np.float64).reshape(M, N)
    J = np.einsum("ijk,mnl,mi,nj->lk", K1, K2, A, B)        # [k2, k1]
    return J.reshape(-1)


def dense_cost(phis, N: int, M: int, h1: float, h2: float, eps: float) -> float:
    """W = sum c t over the explicit plan; O((NM)^3)."""
    i = np.arange(N)
    j = np.arange(M)
    E1 = (np.abs(i[:, None, None] - i[None, :, None]) + np.abs(i[:, None, None] - i[None, None, :])
          + np.abs(i[None, :, None] - i[None, None, :]))
    E2 = (np.abs(j[:, None, None] - j[None, :, None]) + np.abs(j[:, None, None] - j[None, None, :])
          + np.abs(j[None, :, None] - j[None, None, :]))
    K1 = np.exp(-h1 / eps * E1)
    K2 = np.exp(-h2 / eps * E2)
    P = [np.asarray(p, dtype=np.float64).reshape(M, N) for p in phis]
    t1 = np.einsum("ijk,mnl,mi,nj,lk->", h1 * E1 * K1, K2, P[0], P[1], P[2])
    t2 = np.einsum("ijk,mnl,mi,nj,lk->", K1, h2 * E2 * K2, P[0], P[1], P[2])
    return float(t1 + t2)


def _ftvp_2d(phi, psi, lam1: float, lam2: float, N: int, M: int, inner) -> np.ndarray:
    """Algorithm 6 with the inner 1-D product `inner(x, y, lam1)` (FTVP-1 or FTVP-2)."""
    ph = _cols(phi, N, M)
    ps = _cols(psi, N, M)
    l2 = lam2 * lam2
    l4 = l2 * l2
    # paper indices 1..M -> python 0..M-1
    P1 = np.zeros((M, N)); P2 = np.zeros((M, N)); P3 = np.zeros((M, N)); Q3 = np.zeros((M, N))
    P4 = np.zeros((M, N)); Q4 = np.zeros((M, N)); P5 = np.zeros((M, N)); P6 = np.zeros((M, N))
    J1 = np.zeros((M, N)); J2 = np.zeros((M, N)); J3 = np.zeros((M, N)); J4 = np.zeros((M, N))
    J5 = np.zeros((M, N)); J6 = np.zeros((M, N))
    J1[0] = inner(ph[0], ps[0], lam1)                                  # line 2
    P1[0] = ph[0]; P2[0] = l2 * ps[0]; P3[0] = ph[0]; Q3[M - 1] = l2 * ps[M - 1]        # line 3
    P4[0] = ps[0]; Q4[M - 1] = l2 * ph[M - 1]; P5[M - 1] = l2 * ps[M - 1]; P6[M - 1] = l4 * ph[M - 1]  # line 4
    for k in range(1, M):                                              # lines 5-14 (k = 1..M-1)
        P1[k] = l2 * P1[k - 1] + ph[k]
        P2[k] = l2 * P2[k - 1] + l2 * ps[k]
        P3[k] = l2 * P3[k - 1] + ph[k]
        Q3[M - 1 - k] = l2 * Q3[M - k] + l2 * ps[M - 1 - k]
        P4[k] = l2 * P4[k - 1] + ps[k]
        Q4[M - 1 - k] = l2 * Q4[M - k] + l2 * ph[M - 1 - k]
        P5[M - 1 - k] = l2 * P5[M - k] + l2 * ps[M - 1 - k]
        P6[M - 1 - k] = l2 * P6[M - k] + l4 * ph[M - 1 - k]
    for k in range(1, M):                                              # lines 15-20
        J1[k] = l2 * J1[k - 1] + inner(P1[k], ps[k], lam1)
        J2[k] = l2 * J2[k - 1] + inner(ph[k], P2[k - 1], lam1)
        J3[k - 1] = inner(P3[k - 1], Q3[k], lam1)
        J4[k - 1] = inner(Q4[k], P4[k - 1], lam1)
    for k in range(M - 1, 0, -1):                                      # lines 21-23 (k = M..2)
        J5[k - 1] = l2 * J5[k] + inner(ph[k], P5[k], lam1)
    for k in range(M - 2, 0, -1):                                      # lines 24-26 (k = M-1..2)
        J6[k - 1] = l2 * J6[k] + inner(P6[k + 1], ps[k], lam1)
    J = J1 + J2 + J3 + J4 + J5 + J6                                    # lines 27-29
    return J.reshape(-1)


def ftvp_2d(phi, psi, lam1: float, lam2: float, N: int, M: int) -> np.ndarray:
    """Algorithm 6 FTVP_2d: K x_i phi x_j psi on the N x M mesh (column-major)."""
    return _ftvp_2d(phi, psi, lam1, lam2, N, M, lambda x, y, lam: paper3.ftvp1(x, y, lam))


def product(phis, k: int, N: int, M: int, h1: float, h2: float, eps: float) -> np.ndarray:
    """J_k by Algorithm 6 (K is symmetric in its three index pairs, so the free marginal may be any)."""
    a, b = [q for q in range(3) if q != k]
    return ftvp_2d(phis[a], phis[b], math.exp(-h1 / eps), math.exp(-h2 / eps), N, M)


def _transpose(x, N: int, M: int) -> np.ndarray:
    """column-major N x M flat -> column-major M x N flat (rows <-> columns)."""
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(M, N).T).reshape(-1)


def _cost_inner(h: float):
    """1-D cost-weighted product h sum E lambda^E x_i y_j (the role of Algorithm 3's FTVP-2).  Algorithm 3
    forms the E-weights from absolute index sums and loses all accuracy for small lambda (1 - 3e-8 at
    lambda = e^-10, 90 % at e^-50; tests/test_oracle_grid2d.py), so the positive tangent recursion of
    O4 (oracle/subset.c, pinned against the dense (E.K) product) serves as the inner product."""
    from . import regions, subset

    def inner(x, y, lam):
        w = regions.edge_weights_lambda(3, lam)
        _, jh = subset.marginal_product([x, y, np.ones_like(x)], 2, w, want_hat=True)
        return h * jh
    return inner


def cost_2d(phis, N: int, M: int, h1: float, h2: float, eps: float) -> float:
    """W = <varphi, (C.K) x phi x psi> in O(NM): C.K = (C1.K1)(x)K2 + K1(x)(C2.K2)
    (reading A21); each term is Algorithm 6 with a cost-weighted inner product (`_cost_inner`), the
    second on the transposed mesh."""
    lam1, lam2 = math.exp(-h1 / eps), math.exp(-h2 / eps)
    t1 = _ftvp_2d(phis[0], phis[1], lam1, lam2, N, M, _cost_inner(h1))
    tr = [_transpose(p, N, M) for p in phis]
    t2 = _ftvp_2d(tr[0], tr[1], lam2, lam1, M, N, _cost_inner(h2))
    return float(np.dot(phis[2], t1) + np.dot(tr[2], t2))


def marginals(phis, N: int, M: int, h1: float, h2: float, eps: float) -> np.ndarray:
    return np.stack([np.asarray(phis[k]) * product(phis, k, N, M, h1, h2, eps) for k in range(3)])


def sinkhorn_2d(mus, N: int, M: int, h1: float, h2: float, eps: float, iters: int) -> np.ndarray:
    """Generalized Sinkhorn from phi = 1/(NM), Gauss-Seidel order."""
    x = [np.full(N * M, 1.0 / (N * M)) for _ in range(3)]
    for _ in range(iters):
        for k in range(3):
            x[k] = np.asarray(mus[k]) / product(x, k, N, M, h1, h2, eps)
    return np.stack(x)
