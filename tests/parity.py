"""Parity metrics (readings R9/R10).  Test infrastructure only."""
import numpy as np


def eval_err(gpu, orc, scale):
    """max |gpu - oracle| / S over entries, S = the oracle's absolute term sum of the entry
    (summation condition scale, reading R9).  Structurally zero entries (S == 0) must be 0."""
    gpu = np.asarray(gpu)
    orc = np.asarray(orc)
    scale = np.asarray(scale, float)
    zero = scale == 0
    if np.any(gpu[zero] != 0):
        return np.inf
    d = np.abs(gpu - orc)
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.where(zero, 0.0, d / np.where(zero, 1.0, scale))
    return float(np.max(r)) if r.size else 0.0


def backward_err(A, v, rhs):
    """||A v - rhs|| / (||A|| ||v|| + ||rhs||) per point (A: [p,n,n], v/rhs: [p,n])."""
    res = np.einsum("pkj,pj->pk", A, v) - rhs
    den = np.linalg.norm(A, axis=(1, 2)) * np.linalg.norm(v, axis=1) + np.linalg.norm(rhs, axis=1)
    return np.linalg.norm(res, axis=1) / den


def rel_err(a, b):
    return np.linalg.norm(a - b, axis=-1) / np.maximum(np.linalg.norm(b, axis=-1), 1e-300)


def skeel_cond(A):
    """Skeel's condition number || |A^-1| |A| ||_inf per matrix (invariant under row scaling; it
    bounds the forward error of Gaussian elimination with partial pivoting)."""
    Ai = np.linalg.inv(A)
    return np.max(np.einsum("pij,pjk->pik", np.abs(Ai), np.abs(A)).sum(axis=2), axis=1)
