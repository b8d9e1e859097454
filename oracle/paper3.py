"""O2 -- the paper's l = 3 algorithms, step by step (TEST INFRASTRUCTURE ONLY).

Transcribed in the paper's 1-based notation (arrays of length N+2, index 0
and N+1 unused) so that a reader can check each line against PAPER.md:

* ftvp1     -- Algorithm 2 "FTVP-1", exact as printed.
* ftvp2     -- Algorithm 3 "FTVP-2" with the init fix
               R_{N,5} = 2N lambda^2 psi_N, R_{N,6} = 2N lambda^4 phi_N (printed without the
               factor N at P:567; the recurrence displays P:537/P:544 share the typo).
               ``paper_typos=True`` reproduces the printed lines (used by a test that
               shows they are wrong).
* ftvp_log  -- Algorithm 5 "FTVP-LOG" with five fixes (A11):
               (i) J_{1,1} = phi_1 psi_1 e^{(a_1+b_1+g_1)/eps} (P:668 omits the factor);
               (ii) Q_{N-k,3} recurs on Q_{N-k+1,3} (P:676-677 prints ",4");
               (iii) P_{k+1,4} recurs on P_{k,4} (P:678 prints P_{k,2});
               (iv) the P_{N-k,5} ratio uses beta (P:680 prints alpha);
               (v) the P_{N-k,6} ratio uses alpha (P:681-682 print beta).
* fast_sinkhorn_3 -- Algorithm 4: Sinkhorn with FTVP-1 in every update
               (mode permutation trick P:618-630: K is fully symmetric, so
               K x_j psi x_k varphi = FTVP-1(psi, varphi)), residual line 7, and the
               distance with a SINGLE factor h (P:652 applies h twice; A8).

Pure-Python loops: O(N) per call, intended for N up to a few thousand.
"""
from __future__ import annotations

import math

import numpy as np


def _one_based(v):
    a = np.zeros(len(v) + 2)
    a[1:len(v) + 1] = v
    return a


def ftvp1(phi, psi, lam, return_parts=False):
    """Algorithm 2 (FTVP-1): (K x_i phi x_j psi)_k for k = 1..N."""
    N = len(phi)
    f = _one_based(phi)
    s = _one_based(psi)
    l2 = lam * lam
    l4 = l2 * l2
    J = [np.zeros(N + 2) for _ in range(7)]   # J[1..6]
    P = [np.zeros(N + 2) for _ in range(7)]   # P[1..6]
    Q = [np.zeros(N + 2) for _ in range(7)]   # Q[3], Q[4]
    # line 2-4
    J[1][1] = f[1] * s[1]
    P[1][1] = f[1]
    P[2][1] = l2 * s[1]
    P[3][1] = f[1]
    Q[3][N] = l2 * s[N]
    P[4][1] = s[1]
    Q[4][N] = l2 * f[N]
    P[5][N] = l2 * s[N]
    P[6][N] = l4 * f[N]
    # lines 5-14
    for k in range(1, N):
        P[1][k + 1] = l2 * P[1][k] + f[k + 1]
        P[2][k + 1] = l2 * P[2][k] + l2 * s[k + 1]
        P[3][k + 1] = l2 * P[3][k] + f[k + 1]
        Q[3][N - k] = l2 * Q[3][N - k + 1] + l2 * s[N - k]
        P[4][k + 1] = l2 * P[4][k] + s[k + 1]
        Q[4][N - k] = l2 * Q[4][N - k + 1] + l2 * f[N - k]
        P[5][N - k] = l2 * P[5][N - k + 1] + l2 * s[N - k]
        P[6][N - k] = l2 * P[6][N - k + 1] + l4 * f[N - k]
    # lines 15-20
    for k in range(1, N):
        J[1][k + 1] = l2 * J[1][k] + s[k + 1] * P[1][k + 1]
        J[2][k + 1] = l2 * J[2][k] + f[k + 1] * P[2][k]
        J[3][k] = P[3][k] * Q[3][k + 1]
        J[4][k] = P[4][k] * Q[4][k + 1]
    # lines 21-23
    for k in range(N, 1, -1):
        J[5][k - 1] = l2 * J[5][k] + f[k] * P[5][k]
    # lines 24-26
    for k in range(N - 1, 1, -1):
        J[6][k - 1] = l2 * J[6][k] + s[k] * P[6][k + 1]
    out = sum(J[p][1:N + 1] for p in range(1, 7))
    if return_parts:
        return out, [J[p][1:N + 1].copy() for p in range(1, 7)], (J, P, Q)
    return out


def ftvp2(phi, psi, lam, h, paper_typos=False):
    """Algorithm 3 (FTVP-2): ((C . K) x_i phi x_j psi)_k, including the factor h."""
    N = len(phi)
    f = _one_based(phi)
    s = _one_based(psi)
    l2 = lam * lam
    l4 = l2 * l2
    _, _, (J, P, Q) = ftvp1(phi, psi, lam, return_parts=True)
    Jh = [np.zeros(N + 2) for _ in range(7)]
    R = [np.zeros(N + 2) for _ in range(7)]
    S = [np.zeros(N + 2) for _ in range(7)]
    nfac = 1.0 if paper_typos else float(N)
    # lines 2-4
    R[1][1] = -2 * f[1]
    R[2][1] = -2 * l2 * s[1]
    R[3][1] = -2 * f[1]
    S[3][N] = 2 * N * l2 * s[N]
    R[4][1] = -2 * s[1]
    S[4][N] = 2 * N * l2 * f[N]
    R[5][N] = 2 * nfac * l2 * s[N]   # fix: 2 N lambda^2 psi_N (P:567 prints 2 lambda^2 psi_N)
    R[6][N] = 2 * nfac * l4 * f[N]   # fix: 2 N lambda^4 phi_N (P:567 prints 2 lambda^4 phi_N)
    # lines 5-14
    for k in range(1, N):
        R[1][k + 1] = l2 * R[1][k] - 2 * (k + 1) * f[k + 1]
        R[2][k + 1] = l2 * R[2][k] - 2 * (k + 1) * l2 * s[k + 1]
        R[3][k + 1] = l2 * R[3][k] - 2 * (k + 1) * f[k + 1]
        S[3][N - k] = l2 * S[3][N - k + 1] + 2 * (N - k) * l2 * s[N - k]
        R[4][k + 1] = l2 * R[4][k] - 2 * (k + 1) * s[k + 1]
        S[4][N - k] = l2 * S[4][N - k + 1] + 2 * (N - k) * l2 * f[N - k]
        R[5][N - k] = l2 * R[5][N - k + 1] + 2 * (N - k) * l2 * s[N - k]
        R[6][N - k] = l2 * R[6][N - k + 1] + 2 * (N - k) * l4 * f[N - k]
    # lines 15-20
    for k in range(1, N):
        Jh[1][k + 1] = (l2 * Jh[1][k] + 2 * l2 * J[1][k] + s[k + 1] * R[1][k + 1]
                        + 2 * (k + 1) * s[k + 1] * P[1][k + 1])
        Jh[2][k + 1] = (l2 * Jh[2][k] + 2 * l2 * J[2][k] + f[k + 1] * R[2][k]
                        + 2 * (k + 1) * f[k + 1] * P[2][k])
        Jh[3][k] = R[3][k] * Q[3][k + 1] + P[3][k] * S[3][k + 1]
        Jh[4][k] = R[4][k] * Q[4][k + 1] + P[4][k] * S[4][k + 1]
    # lines 21-23
    for k in range(N, 1, -1):
        Jh[5][k - 1] = (l2 * Jh[5][k] + 2 * l2 * J[5][k] + f[k] * R[5][k]
                        - 2 * (k - 1) * f[k] * P[5][k])
    # lines 24-26
    for k in range(N - 1, 1, -1):
        Jh[6][k - 1] = (l2 * Jh[6][k] + 2 * l2 * J[6][k] + s[k] * R[6][k + 1]
                        - 2 * (k - 1) * s[k] * P[6][k + 1])
    return h * sum(Jh[p][1:N + 1] for p in range(1, 7))


def ftvp_log(phi, psi, alpha, beta, gamma, lam, eps, paper_typos=False):
    """Algorithm 5 (FTVP-LOG): (Khat x_i phi x_j psi)_k with
    Khat_{ijk} = e^{(alpha_i + beta_j + gamma_k)/eps} K_{ijk} (Remark 1)."""
    N = len(phi)
    f = _one_based(phi)
    s = _one_based(psi)
    a = _one_based(alpha)
    b = _one_based(beta)
    g = _one_based(gamma)
    l2 = lam * lam
    l4 = l2 * l2
    E = lambda x: math.exp(x / eps)  # noqa: E731
    J = [np.zeros(N + 2) for _ in range(7)]
    P = [np.zeros(N + 2) for _ in range(7)]
    Q = [np.zeros(N + 2) for _ in range(7)]
    # line 2 (fix (i): the e^{(a1+b1+g1)/eps} factor)
    J[1][1] = f[1] * s[1] * (1.0 if paper_typos else E(a[1] + b[1] + g[1]))
    P[1][1] = f[1]
    P[2][1] = l2 * s[1]
    P[3][1] = f[1]
    Q[3][N] = l2 * s[N]
    P[4][1] = s[1]
    Q[4][N] = l2 * f[N]
    P[5][N] = l2 * s[N]
    P[6][N] = l4 * f[N]
    for k in range(1, N):
        P[1][k + 1] = l2 * E(a[k] - a[k + 1]) * P[1][k] + f[k + 1]
        P[2][k + 1] = l2 * E(b[k] - b[k + 1]) * P[2][k] + l2 * s[k + 1]
        P[3][k + 1] = l2 * E(a[k] - a[k + 1]) * P[3][k] + f[k + 1]
        q3src = Q[4] if paper_typos else Q[3]                       # fix (ii)
        Q[3][N - k] = l2 * E(b[N - k + 1] - b[N - k]) * q3src[N - k + 1] + l2 * s[N - k]
        p4src = P[2] if paper_typos else P[4]                       # fix (iii)
        P[4][k + 1] = l2 * E(b[k] - b[k + 1]) * p4src[k] + s[k + 1]
        Q[4][N - k] = l2 * E(a[N - k + 1] - a[N - k]) * Q[4][N - k + 1] + l2 * f[N - k]
        r5 = (a[N - k + 1] - a[N - k]) if paper_typos else (b[N - k + 1] - b[N - k])  # fix (iv)
        P[5][N - k] = l2 * E(r5) * P[5][N - k + 1] + l2 * s[N - k]
        r6 = (b[N - k + 1] - b[N - k]) if paper_typos else (a[N - k + 1] - a[N - k])  # fix (v)
        P[6][N - k] = l2 * E(r6) * P[6][N - k + 1] + l4 * f[N - k]
    for k in range(1, N):
        J[1][k + 1] = (l2 * E(g[k + 1] - g[k]) * J[1][k]
                       + s[k + 1] * E(a[k + 1] + b[k + 1] + g[k + 1]) * P[1][k + 1])
        J[2][k + 1] = (l2 * E(g[k + 1] - g[k]) * J[2][k]
                       + f[k + 1] * E(a[k + 1] + b[k] + g[k + 1]) * P[2][k])
        J[3][k] = E(a[k] + b[k + 1] + g[k]) * P[3][k] * Q[3][k + 1]
        J[4][k] = E(a[k + 1] + b[k] + g[k]) * P[4][k] * Q[4][k + 1]
    for k in range(N, 1, -1):
        J[5][k - 1] = l2 * E(g[k - 1] - g[k]) * J[5][k] + f[k] * E(a[k] + b[k] + g[k - 1]) * P[5][k]
    for k in range(N - 1, 1, -1):
        J[6][k - 1] = (l2 * E(g[k - 1] - g[k]) * J[6][k]
                       + s[k] * E(a[k + 1] + b[k] + g[k - 1]) * P[6][k + 1])
    return sum(J[p][1:N + 1] for p in range(1, 7))


def fast_sinkhorn_3(u, v, w, h, eps, itr_max, tol, paper_double_h=False):
    """Algorithm 4 for l = 3.  Returns (phi, psi, varphi, t, Res, W)."""
    N = len(u)
    lam = math.exp(-h / eps)
    phi = np.full(N, 1.0 / N)
    psi = np.full(N, 1.0 / N)
    vphi = np.full(N, 1.0 / N)
    t = 0
    res = math.inf
    while t < itr_max and res > tol:
        t += 1
        phi = u / ftvp1(psi, vphi, lam)
        psi = v / ftvp1(phi, vphi, lam)
        vphi = w / ftvp1(phi, psi, lam)
        res = float(np.sum(np.abs(phi * ftvp1(psi, vphi, lam) - u))
                    + np.sum(np.abs(psi * ftvp1(phi, vphi, lam) - v)))
    W = float(np.dot(vphi, ftvp2(phi, psi, lam, h)))
    if paper_double_h:          # the printed return line
        W *= h
    return phi, psi, vphi, t, res, W
