"""Seeded synthetic inputs for the five BASELINE configs (and small parity cases).

This module is shared by the oracle side (tests, ``bench.py --impl reference``)
and the CUDA side (tests, bench, smoke).  It holds NO arithmetic of the method:
only random draws, Gaussian bumps, box filtering and normalisation of the
input marginals, i.e. the recipes stated in SURVEY.md §8(d) / DESIGN.md §3.

The paper's own inputs are unseeded U[0,1] vectors (§5.1),
Ricker wavelets (§5.2) and DOTmark images (§5.4, not in this container).
These generators stand in for them with the shapes/sizes of BASELINE.json's
configs.  Every array is produced in fp64 on the host with
``numpy.random.default_rng(seed)`` (PCG64), ``seed = 1000*c + b`` for config
``c`` and instance ``b``.  fp32 variants round the same fp64 arrays.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional

import numpy as np

__all__ = [
    "Config", "CONFIGS", "config", "grid_h", "gaussian_bump", "mixture",
    "c1_marginals", "c2_marginals", "c3_marginals", "c4_marginals",
    "c5_marginals", "c5_etas", "c5_batch_marginals", "random_marginals", "random_positive",
    "make_marginals", "ricker_marginals",
]


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    l: int
    N: int
    eta: Optional[float]       # None for C5 (per-instance eta)
    dtype: str                 # "f64" | "f32"
    iters: int
    tol: float
    batch: int = 1
    x_min: float = 0.0
    x_max: float = 1.0


# BASELINE.json "configs".
CONFIGS = {
    "C1": Config("C1", 3, 64, 0.05, "f64", 200, 0.0),
    "C2": Config("C2", 4, 1000, 0.01, "f64", 2000, 1e-9),
    "C3": Config("C3", 6, 100_000, 1e-3, "f64", 500, 0.0),
    "C3f": Config("C3f", 6, 100_000, 1e-3, "f32", 500, 0.0),
    "C4": Config("C4", 4, 100_000_000, 1e-4, "f64", 100, 0.0),
    "C5": Config("C5", 5, 4096, None, "f32", 300, 0.0, batch=8192),
}


def config(name: str) -> Config:
    return CONFIGS[name]


def grid_h(N: int, x_min: float = 0.0, x_max: float = 1.0) -> float:
    """Grid spacing of the endpoint-inclusive uniform grid (reading A1)."""
    return (x_max - x_min) / (N - 1) if N > 1 else 1.0


def _grid(N: int) -> np.ndarray:
    return np.arange(N, dtype=np.float64) / max(N - 1, 1)


def gaussian_bump(N: int, mu: float, sd: float) -> np.ndarray:
    x = _grid(N)
    return np.exp(-((x - mu) ** 2) / (2.0 * sd * sd))


def _normalise(u: np.ndarray) -> np.ndarray:
    return u / u.sum()


def mixture(rng: np.random.Generator, N: int, ncomp: int) -> np.ndarray:
    """Gaussian mixture, weights ~ Dirichlet(1), means ~ U[0.2,0.8], sds ~ U[0.05,0.15]."""
    wts = rng.dirichlet(np.ones(ncomp))
    mus = rng.uniform(0.2, 0.8, size=ncomp)
    sds = rng.uniform(0.05, 0.15, size=ncomp)
    u = np.zeros(N)
    for a, m, s in zip(wts, mus, sds):
        u += a * gaussian_bump(N, m, s)
    return u


def c1_marginals(seed_instance: int = 0, N: int = 64, l: int = 3) -> np.ndarray:
    """C1: normalised Gaussians (mu~U[.2,.8], sd~U[.05,.15]) + 1e-6 floor, renormalised."""
    rng = np.random.default_rng(1000 * 1 + seed_instance)
    out = np.empty((l, N))
    for q in range(l):
        mu = rng.uniform(0.2, 0.8)
        sd = rng.uniform(0.05, 0.15)
        u = _normalise(gaussian_bump(N, mu, sd))
        u = u + 1e-6
        out[q] = _normalise(u)
    return out


def c2_marginals(seed_instance: int = 0, N: int = 1000, l: int = 4) -> np.ndarray:
    """C2: 3-component Gaussian mixtures, normalised."""
    rng = np.random.default_rng(1000 * 2 + seed_instance)
    return np.stack([_normalise(mixture(rng, N, 3)) for _ in range(l)])


def c3_marginals(seed_instance: int = 0, N: int = 100_000, l: int = 6) -> np.ndarray:
    """C3: 5-component mixtures + 1e-4 * U[0,1] i.i.d. noise, normalised."""
    rng = np.random.default_rng(1000 * 3 + seed_instance)
    out = np.empty((l, N))
    for q in range(l):
        u = _normalise(mixture(rng, N, 5)) + 1e-4 * rng.uniform(0.0, 1.0, size=N)
        out[q] = _normalise(u)
    return out


def c4_marginals(seed_instance: int = 0, N: int = 100_000_000, l: int = 4,
                 width: int = 1000) -> np.ndarray:
    """C4: i.i.d. U[0,1] convolved with a width-`width` box filter (valid mode), normalised."""
    rng = np.random.default_rng(1000 * 4 + seed_instance)
    out = np.empty((l, N))
    for q in range(l):
        r = rng.uniform(0.0, 1.0, size=N + width - 1)
        c = np.empty(N + width)
        c[0] = 0.0
        np.cumsum(r, out=c[1:])
        u = c[width:] - c[:-width]
        del c, r
        out[q] = u / u.sum()
    return out


def c5_etas(batch: int = 8192, seed_base: int = 5000) -> np.ndarray:
    """C5: eta_b = 10**U[-3,-1], one draw per instance (seed 1000*5 + b)."""
    return np.array([10.0 ** np.random.default_rng(seed_base + b).uniform(-3.0, -1.0)
                     for b in range(batch)])


def c5_marginals(b: int, N: int = 4096, l: int = 5) -> np.ndarray:
    """C5 instance b: l 3-component Gaussian mixtures (the eta draw comes first)."""
    rng = np.random.default_rng(1000 * 5 + b)
    rng.uniform(-3.0, -1.0)  # eta draw (see c5_etas) keeps the stream aligned
    return np.stack([_normalise(mixture(rng, N, 3)) for _ in range(l)])


def c5_batch_marginals(b0: int, nb: int, N: int = 4096, l: int = 5) -> np.ndarray:
    """C5 instances b0 .. b0+nb-1 as [l][nb][N] planes; identical values to c5_marginals(b)
    (same per-instance draws, Gaussians evaluated in the same order, vectorised over instances)."""
    x = _grid(N)
    wts = np.empty((l, nb, 3))
    mus = np.empty((l, nb, 3))
    sds = np.empty((l, nb, 3))
    for i in range(nb):
        rng = np.random.default_rng(1000 * 5 + b0 + i)
        rng.uniform(-3.0, -1.0)
        for q in range(l):
            wts[q, i] = rng.dirichlet(np.ones(3))
            mus[q, i] = rng.uniform(0.2, 0.8, size=3)
            sds[q, i] = rng.uniform(0.05, 0.15, size=3)
    out = np.zeros((l, nb, N))
    for q in range(l):
        u = out[q]
        for c in range(3):
            m = mus[q, :, c][:, None]
            sd = sds[q, :, c][:, None]
            u += wts[q, :, c][:, None] * np.exp(-((x[None, :] - m) ** 2) / (2.0 * sd * sd))
        u /= u.sum(axis=1, keepdims=True)
    return out


def random_marginals(seed: int, l: int, N: int, floor: float = 0.0) -> np.ndarray:
    """Paper §5.1 style: i.i.d. U[0,1] entries, normalised."""
    rng = np.random.default_rng(seed)
    u = rng.uniform(0.0, 1.0, size=(l, N)) + floor
    return u / u.sum(axis=1, keepdims=True)


def random_positive(seed: int, l: int, N: int, lo: float = 0.1, hi: float = 1.0) -> np.ndarray:
    """Random positive scaling vectors phi_q ~ U[lo,hi] (single-product tests)."""
    rng = np.random.default_rng(seed)
    return rng.uniform(lo, hi, size=(l, N))


def make_marginals(name: str, instance: int = 0, N: Optional[int] = None) -> np.ndarray:
    """Marginals of config `name` (optionally at a reduced N for parity cases)."""
    cfg = CONFIGS[name]
    n = cfg.N if N is None else N
    if name == "C1":
        return c1_marginals(instance, n, cfg.l)
    if name == "C2":
        return c2_marginals(instance, n, cfg.l)
    if name in ("C3", "C3f"):
        return c3_marginals(instance, n, cfg.l)
    if name == "C4":
        return c4_marginals(instance, n, cfg.l, width=min(1000, max(1, n // 10)))
    if name == "C5":
        return c5_marginals(instance, n, cfg.l)
    raise KeyError(name)


def ricker_marginals(N: int = 100, taus=(0.0, 0.75, 1.5), delta: float = 1e-3, x_min: float = -2.0,
                     x_max: float = 2.0, A: float = 1.0, F0: float = 1.0) -> np.ndarray:
    """The paper's Ricker-wavelet marginals (§5.2), one per shift tau_j:
    R(t) = A (1 - 2 pi^2 F0^2 t^2) exp(-pi^2 F0^2 t^2), f_j(t) = R(t - tau_j) on N uniform points of
    [x_min, x_max], mu_j = (f_j^2 / ||f_j^2||_1 + delta) / (1 + L delta).  Deterministic (no draws).
    Reading: ||.||_1 is the discrete sum and L = N, so every mu_j sums to one."""
    t = np.linspace(x_min, x_max, N)
    out = []
    for tau in taus:
        a = (math.pi * F0 * (t - tau)) ** 2
        f = A * (1.0 - 2.0 * a) * np.exp(-a)
        p = f * f / np.sum(f * f)
        out.append((p + delta) / (1.0 + N * delta))
    return np.stack(out)
