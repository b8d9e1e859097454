"""O5 -- Gauss-Seidel Sinkhorn driver over the region-chain products (TEST INFRASTRUCTURE ONLY).

Generalized Sinkhorn for l marginals (Algorithm 1 P:153-172;
Algorithm 4):

    init phi_q = 1/N
    for t = 1..T:  for k = 1..l:  phi_k <- mu_k / J_k(phi_{-k})   (freshest peers)
    Res_t = sum_{k=1}^{l-1} || phi_k * J_k - mu_k ||_1   on end-of-sweep vectors
            (Algorithm 1 line 7, generalised: DESIGN.md A6)
    stop at the first t with Res_t <= tol (tol <= 0: run exactly T)
    W = h * <phi_l, hatJ_l>,  hatJ = sum E lambda^E prod phi          (single h: A8)

``domain="plain"`` uses linear fp64 scalings; ``domain="log"`` carries
g_q = log phi_q and the log-domain region chains (Remark 1's purpose,
P:138-151, realised as a pure log domain -- DESIGN.md A13).
"""
from __future__ import annotations

import math
from typing import Callable, Optional, Sequence

import numpy as np

from . import regions, subset

# product engine: "regions" (O3, the paper's §4.2 recursion) or "subset" (O4, subset-lattice DP,
# pinned against O1 and O3 by tests/test_oracle_subset.py; several times faster at l >= 5)
_ENGINES = {"regions": regions, "subset": subset}


def _weights(l, h, eta):
    return regions.edge_weights(l, h, eta)


def product(phis, k, h, eta, engine: str = "regions"):
    """J_k by region chains (plain fp64), or by the subset DP (engine="subset")."""
    return _ENGINES[engine].marginal_product(list(phis), k, _weights(len(phis), h, eta))


def marginals(phis, h, eta):
    """m_k = phi_k * J_k for every k."""
    return np.stack([phis[k] * product(phis, k, h, eta) for k in range(len(phis))])


def log_product(gs, k, h, eta, engine: str = "regions"):
    l = len(gs)
    lw = np.array([-(a * (l - a)) * h / eta for a in range(l + 1)])
    return _ENGINES[engine].marginal_product_log(list(gs), k, lw)


def cost(phis, h, eta, k: Optional[int] = None):
    """W = sum_i c_i t_i = h * <phi_k, hatJ_k> for any k (default l-1)."""
    l = len(phis)
    k = l - 1 if k is None else k
    _, jh = regions.marginal_product(list(phis), k, _weights(l, h, eta), want_hat=True)
    return float(h * np.dot(phis[k], jh))


def residual(phis, mus, h, eta, engine: str = "regions"):
    l = len(phis)
    return float(sum(np.abs(phis[k] * product(phis, k, h, eta, engine) - mus[k]).sum() for k in range(l - 1)))


def sinkhorn(mus: np.ndarray, h: float, eta: float, iters: int, tol: float = 0.0,
             phis0: Optional[np.ndarray] = None, domain: str = "plain",
             record: Optional[Callable] = None, check_every: int = 1, engine: str = "regions"):
    """Run Sinkhorn; returns (scalings, t, Res).  Scalings are phi (plain) or g = log phi (log).
    engine: "regions" (O3) or "subset" (O4) products."""
    l, N = mus.shape
    if domain == "plain":
        x = [np.full(N, 1.0 / N) for _ in range(l)] if phis0 is None else [p.astype(np.float64).copy() for p in phis0]
    else:
        x = [np.full(N, -math.log(N)) for _ in range(l)] if phis0 is None else [p.astype(np.float64).copy() for p in phis0]
        with np.errstate(divide="ignore"):
            logmu = np.log(mus)
    res = math.inf
    t = 0
    while t < iters and (tol <= 0 or res > tol):
        t += 1
        for k in range(l):
            if domain == "plain":
                x[k] = mus[k] / product(x, k, h, eta, engine)
            else:
                x[k] = logmu[k] - log_product(x, k, h, eta, engine)
        if tol > 0 and (t % check_every == 0 or t == iters):
            if domain == "plain":
                res = residual(x, mus, h, eta, engine)
            else:
                res = float(sum(np.abs(np.exp(x[k] + log_product(x, k, h, eta, engine)) - mus[k]).sum()
                                for k in range(l - 1)))
        if record is not None:
            record(t, [v.copy() for v in x])
    return np.stack(x), t, res
