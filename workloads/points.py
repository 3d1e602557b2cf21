"""Seeded evaluation points (SURVEY §8(d) "Concrete synthetic inputs").

x_j = exp(rho + i*theta) with rho ~ U[-rho_max, rho_max], theta ~ U[-pi, pi);
tau ~ U[tau_lo, 0], t = exp(tau) in (0, 1] (ledger A16: t real).
These are inputs only; generating them is not part of the method.
"""
from __future__ import annotations

import numpy as np

from .systems import MASTER_SEED


def random_log_points(p: int, n: int, *, seed: int = MASTER_SEED, rho_max: float = 1.0,
                      tau_lo: float = -3.0):
    """Return (z complex128[p,n], tau float64[p]) with z = rho + i theta."""
    rng = np.random.Generator(np.random.PCG64(seed + 7))
    rho = rng.uniform(-rho_max, rho_max, size=(p, n))
    th = rng.uniform(-np.pi, np.pi, size=(p, n))
    tau = rng.uniform(tau_lo, 0.0, size=p)
    return rho + 1j * th, tau


def random_points(p: int, n: int, *, seed: int = MASTER_SEED, rho_max: float = 1.0,
                  tau_lo: float = -3.0):
    """Return (x complex128[p,n], t float64[p], tau float64[p])."""
    z, tau = random_log_points(p, n, seed=seed, rho_max=rho_max, tau_lo=tau_lo)
    return np.exp(z), np.exp(tau), tau
