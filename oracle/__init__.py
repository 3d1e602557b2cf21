"""ctypes front end for the C oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs are the only permitted callers.  The product
package (paper_2111_14317_b200) never imports this module.

Functions mirror oracle.c; see there for the paper passage each one follows.
Parity-unpinned items: none of the evaluation/direction/step functions (all pinned in
tests/test_oracle_*.py); the adaptive tracker's accept/reject decisions are pinned only
through endpoints and counts (DESIGN.md ledger R14).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liborc.so")

PT_OK, PT_ZERO_COORD, PT_NONFINITE, PT_SINGULAR = 0, 1, 2, 4
PT_STEP_UNDERFLOW, PT_MAX_STEPS, PT_DIVERGED = 8, 16, 32


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE, "liborc.so"], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB_PATH)
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def set_threads(nt: int = 0) -> int:
    return int(lib().orc_set_threads(ctypes.c_int(nt)))


def _c2(a):
    """complex128 array -> contiguous float64 view [..., 2]."""
    a = np.ascontiguousarray(a, np.complex128)
    return a


class Oracle:
    """Oracle bound to one system (workloads.System)."""

    def __init__(self, system):
        self.system = system
        self.n = int(system.n)
        self.off = np.ascontiguousarray(system.offsets, np.int64)
        self.exps = np.ascontiguousarray(system.exps, np.int32)
        self.coeffs = np.ascontiguousarray(system.coeffs, np.complex128)
        lift = np.asarray(system.lifting, np.float64)
        if np.any(lift != np.round(lift)) or np.any(lift < 0):
            raise ValueError("oracle requires non-negative integer liftings (ledger R4)")
        self.w = np.ascontiguousarray(lift.astype(np.int64))

    def _sys_args(self):
        return (ctypes.c_int(self.n), _p(self.off), _p(self.exps), _p(self.coeffs), _p(self.w))

    # --- O1: evaluation by the definition -------------------------------
    def evaluate(self, x, t):
        x = _c2(x)
        t = np.ascontiguousarray(t, np.float64)
        p, n = x.shape[0], self.n
        H = np.zeros((p, n), np.complex128)
        Jx = np.zeros((p, n, n), np.complex128)
        Jt = np.zeros((p, n), np.complex128)
        SH = np.zeros((p, n))
        SJx = np.zeros((p, n, n))
        SJt = np.zeros((p, n))
        st = np.zeros(p, np.uint8)
        rc = lib().orc_evaluate(*self._sys_args(), ctypes.c_int64(p), _p(x), _p(t), _p(H), _p(Jx),
                                _p(Jt), _p(SH), _p(SJx), _p(SJt), _p(st))
        assert rc == 0
        return dict(H=H, Jx=Jx, Jt=Jt, SH=SH, SJx=SJx, SJt=SJt, status=st)

    # --- O2: extended range ---------------------------------------------------------
    def evaluate_x(self, xm, xe, tm, te):
        """x = xm * 2**xe, t = tm * 2**te; returns mantissas, exponents, log2 term sums."""
        xm = _c2(xm)
        xe = np.ascontiguousarray(xe, np.int64)
        tm = np.ascontiguousarray(tm, np.float64)
        te = np.ascontiguousarray(te, np.int64)
        p, n = xm.shape[0], self.n
        out = dict(Hm=np.zeros((p, n), np.complex128), He=np.zeros((p, n), np.int64),
                   Jxm=np.zeros((p, n, n), np.complex128), Jxe=np.zeros((p, n, n), np.int64),
                   Jtm=np.zeros((p, n), np.complex128), Jte=np.zeros((p, n), np.int64),
                   LSH=np.zeros((p, n)), LSJx=np.zeros((p, n, n)), LSJt=np.zeros((p, n)))
        rc = lib().orc_evaluate_x(*self._sys_args(), ctypes.c_int64(p), _p(xm), _p(xe), _p(tm), _p(te),
                                  *[_p(out[k]) for k in ("Hm", "He", "Jxm", "Jxe", "Jtm", "Jte",
                                                         "LSH", "LSJx", "LSJt")])
        assert rc == 0
        return out

    # --- O3: directions --------------------------------------------------
    def euler_newton(self, x, t):
        x = _c2(x)
        t = np.ascontiguousarray(t, np.float64)
        p, n = x.shape[0], self.n
        dE = np.zeros((p, n), np.complex128)
        dN = np.zeros((p, n), np.complex128)
        st = np.zeros(p, np.uint8)
        rc = lib().orc_euler_newton(*self._sys_args(), ctypes.c_int64(p), _p(x), _p(t), _p(dE),
                                    _p(dN), _p(st))
        assert rc == 0
        return dE, dN, st

    # --- O4: the paper's Euler-Newton step ------------------------------
    def pc_step(self, x, tau, dtau, K=1):
        x = _c2(x).copy()
        tau = np.ascontiguousarray(tau, np.float64).copy()
        p = x.shape[0]
        dtau = np.ascontiguousarray(np.broadcast_to(np.asarray(dtau, np.float64), (p,)))
        st = np.zeros(p, np.uint8)
        dn = np.zeros(p)
        rc = lib().orc_pc_step(*self._sys_args(), ctypes.c_int64(p), _p(x), _p(tau), _p(dtau),
                               ctypes.c_int(K), _p(st), _p(dn))
        assert rc == 0
        return x, tau, st, dn

    def track(self, x, tau, *, dtau_init=0.05, dtau_min=1e-12, dtau_max=0.5, newton_tol=1e-10,
              shrink=0.5, grow=2.0, final_tol=1e-13, inf_norm=1e8, K=4, grow_after=3,
              max_steps=10000, final_iters=5, pred_log=0, pred_tol=0.0, reuse_tangent=0):
        x = _c2(x).copy()
        tau = np.ascontiguousarray(tau, np.float64).copy()
        p = x.shape[0]
        opt = np.array([dtau_init, dtau_min, dtau_max, newton_tol, shrink, grow, final_tol, inf_norm, pred_tol])
        iopt = np.array([K, grow_after, max_steps, final_iters, pred_log, reuse_tangent], np.int32)
        st = np.zeros(p, np.uint8)
        stats = np.zeros((p, 4), np.int64)
        rc = lib().orc_track(*self._sys_args(), ctypes.c_int64(p), _p(x), _p(tau), _p(opt), _p(iopt),
                             _p(st), _p(stats))
        assert rc == 0
        return x, tau, st, stats


    def track_x(self, xm, xe, tau, *, dtau_init=0.05, dtau_min=1e-12, dtau_max=0.5, newton_tol=1e-10,
                shrink=0.5, grow=2.0, final_tol=1e-13, inf_norm=1e8, K=4, grow_after=3,
                max_steps=10000, final_iters=5, pred_log=1, cell_lift=None, path_cell=None, pred_tol=0.0,
                predictor=0, reuse_tangent=0):
        """orc_track_x: the tracker with extended-range state x = xm * 2**xe; with cell_lift
        [ncells, M] / path_cell [p] it tracks in cell coordinates (pht_track_cells)."""
        xm = _c2(xm).copy()
        xe = np.ascontiguousarray(xe, np.int64).copy()
        tau = np.ascontiguousarray(tau, np.float64).copy()
        p = xm.shape[0]
        opt = np.array([dtau_init, dtau_min, dtau_max, newton_tol, shrink, grow, final_tol, inf_norm, pred_tol])
        iopt = np.array([K, grow_after, max_steps, final_iters, pred_log, predictor, reuse_tangent], np.int32)
        st = np.zeros(p, np.uint8)
        stats = np.zeros((p, 4), np.int64)
        cw = None if cell_lift is None else np.ascontiguousarray(cell_lift, np.float64)
        pc = None if path_cell is None else np.ascontiguousarray(path_cell, np.int32)
        rc = lib().orc_track_x(*self._sys_args(), ctypes.c_int64(p), _p(xm), _p(xe), _p(tau), _p(opt),
                               _p(iopt), _p(st), _p(stats), _p(cw) if cw is not None else None,
                               _p(pc) if pc is not None else None)
        assert rc == 0
        return xm, xe, tau, st, stats


    # --- projective formulation -------------------------
    def proj_evaluate(self, y, t):
        """H^, dH^/dy [p, n, n+1], dH^/dt of the homogenised system (Eq. (3)) at y in C^{n+1}."""
        y = _c2(y)
        t = np.ascontiguousarray(t, np.float64)
        p, n = y.shape[0], self.n
        assert y.shape[1] == n + 1
        out = dict(H=np.zeros((p, n), np.complex128), Jy=np.zeros((p, n, n + 1), np.complex128),
                   Jt=np.zeros((p, n), np.complex128), SH=np.zeros((p, n)), SJy=np.zeros((p, n, n + 1)),
                   SJt=np.zeros((p, n)), status=np.zeros(p, np.uint8))
        rc = lib().orc_proj_evaluate(*self._sys_args(), ctypes.c_int64(p), _p(y), _p(t),
                                     *[_p(out[k]) for k in ("H", "Jy", "Jt", "SH", "SJy", "SJt", "status")])
        assert rc == 0
        return out

    def proj_euler_newton(self, y, t):
        """Projective Euler E = dy/dtau and Newton N directions."""
        y = _c2(y)
        t = np.ascontiguousarray(t, np.float64)
        p, m = y.shape
        E = np.zeros((p, m), np.complex128)
        N = np.zeros((p, m), np.complex128)
        st = np.zeros(p, np.uint8)
        rc = lib().orc_proj_euler_newton(*self._sys_args(), ctypes.c_int64(p), _p(y), _p(t), _p(E), _p(N), _p(st))
        assert rc == 0
        return E, N, st

    def proj_pc_step(self, y, tau, dtau, K=1):
        y = _c2(y).copy()
        tau = np.ascontiguousarray(tau, np.float64).copy()
        dtau = np.ascontiguousarray(dtau, np.float64)
        p = y.shape[0]
        st = np.zeros(p, np.uint8)
        dn = np.zeros(p)
        rc = lib().orc_proj_pc_step(*self._sys_args(), ctypes.c_int64(p), _p(y), _p(tau), _p(dtau),
                                    ctypes.c_int(K), _p(st), _p(dn))
        assert rc == 0
        return y, tau, st, dn

    def proj_track(self, y, tau, *, dtau_init=0.05, dtau_min=1e-12, dtau_max=0.5, newton_tol=1e-10,
                   shrink=0.5, grow=2.0, final_tol=1e-13, inf_norm=1e8, K=4, grow_after=3,
                   max_steps=10000, final_iters=5, pred_tol=0.0):
        y = _c2(y).copy()
        tau = np.ascontiguousarray(tau, np.float64).copy()
        p = y.shape[0]
        opt = np.array([dtau_init, dtau_min, dtau_max, newton_tol, shrink, grow, final_tol, inf_norm, pred_tol])
        iopt = np.array([K, grow_after, max_steps, final_iters, 0], np.int32)
        st = np.zeros(p, np.uint8)
        stats = np.zeros((p, 4), np.int64)
        rc = lib().orc_proj_track(*self._sys_args(), ctypes.c_int64(p), _p(y), _p(tau), _p(opt), _p(iopt),
                                  _p(st), _p(stats))
        assert rc == 0
        return y, tau, st, stats


# --- test plumbing (not the oracle): log coordinates <-> extended-range (mantissa, exponent) ---
def z_to_x(z):
    """z = log x  ->  (m, e) with x = m * 2**e, |m| in [1, 2)."""
    z = np.asarray(z, np.complex128)
    e = np.floor(z.real / np.log(2)).astype(np.int64)
    m = np.exp(z.real - e * np.log(2)) * np.exp(1j * z.imag)
    return m, e


def x_to_z(m, e):
    """(m, e) -> z = log m + e ln 2 (principal branch of log m)."""
    return np.log(np.asarray(m, np.complex128)) + np.asarray(e, np.float64) * np.log(2)


def lu_solve(A, B):
    """Route 1 (Gaussian elimination, partial pivoting): returns (X, status)."""
    A = _c2(A)
    B = _c2(B)
    n = A.shape[0]
    B2 = B.reshape(n, -1)
    X = np.zeros_like(B2)
    st = lib().orc_lu_solve(ctypes.c_int(n), ctypes.c_int(B2.shape[1]), _p(A), _p(np.ascontiguousarray(B2)), _p(X))
    return X.reshape(B.shape), int(st)


def dirs_qr(J):
    """Route 2, the paper's QR null space: J n x (n+2) -> (dE, dN, status)."""
    J = _c2(J)
    n = J.shape[0]
    dE = np.zeros(n, np.complex128)
    dN = np.zeros(n, np.complex128)
    st = lib().orc_dirs_qr(ctypes.c_int(n), _p(J), _p(dE), _p(dN))
    return dE, dN, int(st)
