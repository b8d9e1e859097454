"""Closed-form unregularised optimum W_0 of 1-D pairwise-L1 MMOT (TEST INFRASTRUCTURE ONLY).

For the cost c = h sum_{p<q} |i_p - i_q| on a line the optimal
coupling of the unregularised problem is the comonotone
(quantile) coupling, so

    W_0 = integral_0^1 sum_{p<q} | F_p^{-1}(t) - F_q^{-1}(t) | dt .

Used only as a sanity pin: the entropic plan's linear cost satisfies
W_eta >= W_0 (the plan is feasible for the LP once the marginals are met),
and W_eta -> W_0 as eta -> 0.  W_0 itself is pinned against scipy's LP
solver on tiny instances (tests/test_oracle_sinkhorn.py).
"""
from __future__ import annotations

import numpy as np


def w0(mus: np.ndarray, h: float) -> float:
    l, N = mus.shape
    cums = [np.cumsum(m / m.sum()) for m in mus]
    bps = np.unique(np.concatenate([np.array([0.0, 1.0])] + [np.clip(c, 0.0, 1.0) for c in cums]))
    total = 0.0
    for a, b in zip(bps[:-1], bps[1:]):
        if b <= a:
            continue
        t = 0.5 * (a + b)
        pos = [int(np.searchsorted(c, t, side="left")) for c in cums]
        pos = [min(p, N - 1) for p in pos]
        s = 0.0
        for p in range(l):
            for q in range(p + 1, l):
                s += abs(pos[p] - pos[q])
        total += (b - a) * s
    return h * total
