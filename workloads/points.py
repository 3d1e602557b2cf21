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


def random_extended_points(p: int, n: int, *, seed: int = MASTER_SEED, rho_max: float = 100.0,
                           tau_lo: float = -5.0):
    """Points beyond double range given EXACTLY in extended form (SURVEY §8(d) C5 range-stress
    set: Re z ~ U[-rho_max, rho_max], tau ~ U[tau_lo, 0]): x_j = xm_j 2^xe_j with |xm_j| in
    [1, 2), t = tm 2^te, together with their logarithms z = log x, tau = log t computed in long
    double and rounded once.  The oracle evaluates at the exact (xm, xe, tm, te); the CUDA path
    takes (z, tau), whose only error is that final rounding (u/2 relative).
    Returns (xm complex128[p,n], xe int64[p,n], tm float64[p], te int64[p], z complex128[p,n],
    tau float64[p])."""
    rng = np.random.Generator(np.random.PCG64(seed + 11))
    rho = rng.uniform(-rho_max, rho_max, size=(p, n))
    th = rng.uniform(-np.pi, np.pi, size=(p, n))
    xe = np.floor(rho / np.log(2)).astype(np.int64)
    mag = np.exp(rho - xe * np.log(2))                     # ~[1, 2): any value is an exact input
    mag = np.clip(mag, 1.0, np.nextafter(2.0, 0.0))
    xm = mag * np.exp(1j * th)
    taur = rng.uniform(tau_lo, 0.0, size=p)
    te = np.floor(taur / np.log(2)).astype(np.int64)
    tm = np.clip(np.exp(taur - te * np.log(2)), 1.0, np.nextafter(2.0, 0.0))
    L2 = np.log(np.longdouble(2))
    zr = np.log(np.abs(xm).astype(np.longdouble)) + xe.astype(np.longdouble) * L2
    zi = np.arctan2(xm.imag.astype(np.longdouble), xm.real.astype(np.longdouble))
    z = zr.astype(np.float64) + 1j * zi.astype(np.float64)
    tau = (np.log(tm.astype(np.longdouble)) + te.astype(np.longdouble) * L2).astype(np.float64)
    return xm, xe, tm, te, z, tau
