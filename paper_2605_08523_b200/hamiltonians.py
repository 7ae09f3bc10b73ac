"""Synthetic Hamiltonians for the benchmark configs.

2-D periodic square lattice, nearest-neighbour hopping t = -1, on-site energies
eps_i ~ U(-0.5, 0.5) drawn from ``numpy.random.default_rng(seed)``; site
i = x*Ly + y.  Gershgorin bounds lie inside [-4.5, 4.5].
"""
from __future__ import annotations

import numpy as np

LATTICE = {256: (16, 16), 512: (32, 16), 1024: (32, 32), 2048: (64, 32), 4096: (64, 64),
           8192: (128, 64), 16384: (128, 128)}


def lattice_shape(n: int) -> tuple[int, int]:
    if n in LATTICE:
        return LATTICE[n]
    lx = 1
    while lx * lx < n:
        lx *= 2
    while n % lx:
        lx //= 2
    return lx, n // lx


def tight_binding(n: int, seed: int = 1234, t: float = -1.0, dtype=np.float64) -> np.ndarray:
    """Dense fp64 H of the periodic 2-D tight-binding model (exactly symmetric)."""
    lx, ly = lattice_shape(n)
    rng = np.random.default_rng(seed)
    H = np.zeros((n, n), dtype=np.float64)
    H[np.diag_indices(n)] = rng.uniform(-0.5, 0.5, size=n)
    for x in range(lx):
        for y in range(ly):
            i = x * ly + y
            for j in (((x + 1) % lx) * ly + y, x * ly + (y + 1) % ly):
                if j != i:
                    H[i, j] = t
                    H[j, i] = t
    return H.astype(dtype, copy=False)


def goe(n: int, seed: int = 0) -> np.ndarray:
    """Dense GOE (A + A^T)/sqrt(2N): the secondary (ungated) stress family."""
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((n, n))
    H = (A + A.T) / np.sqrt(2.0 * n)
    return np.triu(H) + np.triu(H, 1).T


def batch_params(batch: int, seed: int = 777, kT_range=(0.010, 0.0125), mu_range=(-0.5, 0.25)):
    """Per-matrix (mu_k, kT_k) of config 4."""
    rng = np.random.default_rng(seed)
    mu = rng.uniform(mu_range[0], mu_range[1], size=batch)
    kT = rng.uniform(kT_range[0], kT_range[1], size=batch)
    return mu, kT
