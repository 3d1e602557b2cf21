"""Start points of the polyhedral homotopy for small systems (workload preparation).

The paper assumes the start points are given ("we simply assume the set of all
solutions to H(x, t0) = 0 ... is readily available").  This module produces them the standard
way (Huber-Sturmfels), for SMALL systems only (brute force over edge tuples):

1. Fine mixed cells: one pair {a_k, a'_k} of S_k per equation with an inner normal (alpha, 1):
   <a_k, alpha> + w(a_k) = <a'_k, alpha> + w(a'_k) = beta_k  and  <b, alpha> + w(b) > beta_k
   for every other b in S_k.  Exact rational arithmetic.  Volume |det V|, V = [a_k - a'_k]_k.
2. Binomial start system per cell: c_k y^{a_k} + c'_k y^{a'_k} = 0  <=>  y^{V} = -c'/c, solved in
   log coordinates via a Hermite normal form U V = T (all |det V| branches).
3. Start point on the path at tau0 (per cell): x = exp(tau0 alpha + log y), tau0 = -L / gap with
   gap = the smallest lifting gap of the cell, so the neglected terms are O(e^{-L}).

No evaluation of H or its derivatives happens here (nothing of the method's arithmetic).
"""
from __future__ import annotations

import itertools
from fractions import Fraction
from typing import List, Tuple

import numpy as np

import os

DATA_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data")


def _solve_rational(V: List[List[int]], b: List[Fraction]):
    """Gaussian elimination over Q; returns x or None if singular."""
    n = len(V)
    M = [[Fraction(V[i][j]) for j in range(n)] + [Fraction(b[i])] for i in range(n)]
    for c in range(n):
        p = next((r for r in range(c, n) if M[r][c] != 0), None)
        if p is None:
            return None
        M[c], M[p] = M[p], M[c]
        for r in range(n):
            if r != c and M[r][c] != 0:
                f = M[r][c] / M[c][c]
                M[r] = [M[r][j] - f * M[c][j] for j in range(n + 1)]
    return [M[i][n] / M[i][i] for i in range(n)]


def _det_int(V: List[List[int]]) -> int:
    M = [[Fraction(v) for v in row] for row in V]
    n = len(M)
    det = Fraction(1)
    for c in range(n):
        p = next((r for r in range(c, n) if M[r][c] != 0), None)
        if p is None:
            return 0
        if p != c:
            M[c], M[p] = M[p], M[c]
            det = -det
        det *= M[c][c]
        for r in range(c + 1, n):
            f = M[r][c] / M[c][c]
            M[r] = [M[r][j] - f * M[c][j] for j in range(n)]
    return int(det)


def mixed_cells(system) -> List[dict]:
    """All fine mixed cells of the lifted supports (brute force over pair tuples)."""
    n = system.n
    sup = []
    for k in range(n):
        rows = [(tuple(int(v) for v in system.exps[i]), Fraction(system.lifting[i]).limit_denominator(10**9), i)
                for i in system.terms_of(k)]
        sup.append(rows)
    cells = []
    for pairs in itertools.product(*[list(itertools.combinations(range(len(s)), 2)) for s in sup]):
        V = [[sup[k][pairs[k][0]][0][j] - sup[k][pairs[k][1]][0][j] for j in range(n)] for k in range(n)]
        rhs = [sup[k][pairs[k][1]][1] - sup[k][pairs[k][0]][1] for k in range(n)]
        alpha = _solve_rational(V, rhs)
        if alpha is None:
            continue
        ok = True
        gap = None
        for k in range(n):
            a0, w0, _ = sup[k][pairs[k][0]]
            beta = sum(Fraction(a0[j]) * alpha[j] for j in range(n)) + w0
            for idx, (b, wb, _) in enumerate(sup[k]):
                if idx in pairs[k]:
                    continue
                d = sum(Fraction(b[j]) * alpha[j] for j in range(n)) + wb - beta
                if d <= 0:
                    ok = False
                    break
                gap = d if gap is None else min(gap, d)
            if not ok:
                break
        if not ok:
            continue
        cells.append({"pairs": [(sup[k][pairs[k][0]][2], sup[k][pairs[k][1]][2]) for k in range(n)],
                      "V": V, "alpha": alpha, "gap": gap, "volume": abs(_det_int(V))})
    return cells


def mixed_cells_fast(system, max_cells: int = 2_000_000) -> List[dict]:
    """Same cells as mixed_cells(), via the C++ enumerator (lower edges, pairwise compatibility,
    LP-pruned depth-first search; workloads/mixedcell.cpp).  Cell records carry exact rational
    alpha/gap recomputed from the pairs."""
    import ctypes
    import os
    import subprocess
    here = os.path.dirname(os.path.abspath(__file__))
    lib_path = os.path.join(here, "libmixedcell.so")
    src = os.path.join(here, "mixedcell.cpp")
    if not os.path.exists(lib_path) or os.path.getmtime(lib_path) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", here, "libmixedcell.so"], check=True)
    lib = ctypes.CDLL(lib_path)
    lib.mc_cells.restype = ctypes.c_int64
    n = system.n
    off = np.ascontiguousarray(system.offsets, np.int64)
    ex = np.ascontiguousarray(system.exps, np.int32)
    lift = np.ascontiguousarray(system.lifting, np.float64)
    pairs = np.zeros((max_cells, n, 2), np.int32)
    alpha = np.zeros((max_cells, n))
    gap = np.zeros(max_cells)
    stats = np.zeros(4, np.int64)
    P = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    cnt = lib.mc_cells(ctypes.c_int(n), P(off), P(ex), P(lift), ctypes.c_int64(max_cells), P(pairs), P(alpha),
                       P(gap), P(stats))
    if cnt < 0:
        raise RuntimeError("too many mixed cells")
    cells = []
    for c in range(cnt):
        pr = [(int(pairs[c, k, 0]), int(pairs[c, k, 1])) for k in range(n)]
        V = [[int(system.exps[p][j]) - int(system.exps[q][j]) for j in range(n)] for (p, q) in pr]
        rhs = [Fraction(system.lifting[q]).limit_denominator(10**9) - Fraction(system.lifting[p]).limit_denominator(10**9)
               for (p, q) in pr]
        al = _solve_rational(V, rhs)
        g = None
        for k in range(n):
            p0, q0 = pr[k]
            beta = sum(Fraction(int(system.exps[p0][j])) * al[j] for j in range(n)) + \
                Fraction(system.lifting[p0]).limit_denominator(10**9)
            for i in system.terms_of(k):
                if i in (p0, q0):
                    continue
                d = sum(Fraction(int(system.exps[i][j])) * al[j] for j in range(n)) + \
                    Fraction(system.lifting[i]).limit_denominator(10**9) - beta
                if d <= 0:
                    raise RuntimeError("enumerated cell fails the exact check")
                g = d if g is None else min(g, d)
        cells.append({"pairs": pr, "V": V, "alpha": al, "gap": g, "volume": abs(_det_int(V))})
    mixed_cells_fast.last_stats = stats.copy()
    return cells


def mixed_volume(system) -> int:
    return sum(c["volume"] for c in mixed_cells(system))


def _hnf_rows(V: List[List[int]]) -> Tuple[List[List[int]], List[List[int]]]:
    """Row-style Hermite reduction: unimodular U with U V = T upper triangular."""
    n = len(V)
    T = [list(r) for r in V]
    U = [[int(i == j) for j in range(n)] for i in range(n)]
    r = 0
    for c in range(n):
        # Euclid on column c among rows r..n-1
        while True:
            nz = [i for i in range(r, n) if T[i][c] != 0]
            if len(nz) <= 1:
                break
            p = min(nz, key=lambda i: abs(T[i][c]))
            for i in nz:
                if i != p:
                    q = T[i][c] // T[p][c]
                    T[i] = [T[i][j] - q * T[p][j] for j in range(n)]
                    U[i] = [U[i][j] - q * U[p][j] for j in range(n)]
        nz = [i for i in range(r, n) if T[i][c] != 0]
        if not nz:
            continue
        p = nz[0]
        T[r], T[p] = T[p], T[r]
        U[r], U[p] = U[p], U[r]
        if T[r][c] < 0:
            T[r] = [-v for v in T[r]]
            U[r] = [-v for v in U[r]]
        r += 1
    return U, T


def cell_start_points(system, cell, L: float = 37.0, tau_cap: float | None = None,
                      zmax: float | None = None):
    """All |det V| start points of one cell: returns (x [vol, n] complex128, tau0, z [vol, n]).

    tau0 = -L / gap (neglected terms O(e^{-L})), optionally capped so that |tau0| <= tau_cap
    and |tau0 * alpha_j| <= zmax (keeps |x| inside double range at the price of a larger start
    residual, which the tracker's first corrections remove)."""
    n = system.n
    V = cell["V"]
    U, T = _hnf_rows(V)
    c = system.coeffs
    logb = np.array([np.log(-c[j1] / c[j0]) for (j0, j1) in cell["pairs"]], np.complex128)
    w = np.array([sum(U[k][l] * logb[l] for l in range(n)) for k in range(n)], np.complex128)
    sols = [np.zeros(n, np.complex128)]
    for row in range(n - 1, -1, -1):
        new = []
        d = T[row][row]
        for z in sols:
            rest = w[row] - sum(T[row][j] * z[j] for j in range(row + 1, n))
            for m in range(abs(d)):
                zz = z.copy()
                zz[row] = (rest + 2j * np.pi * m) / d
                new.append(zz)
        sols = new
    Z = np.array(sols)
    alpha = np.array([float(a) for a in cell["alpha"]])
    tau0 = -L / float(cell["gap"])
    if tau_cap is not None:
        tau0 = max(tau0, -tau_cap)
    if zmax is not None and np.max(np.abs(alpha)) > 0:
        tau0 = max(tau0, -zmax / float(np.max(np.abs(alpha))))
    Zt = Z + tau0 * alpha[None, :]
    with np.errstate(over="ignore", under="ignore"):
        X = np.exp(Zt)  # inf/0 where x leaves double range: use the log coordinates Zt there
    return X, tau0, Zt


def start_points(system, L: float = 37.0, tau_cap: float | None = None, zmax: float | None = None,
                 fast: bool = False):
    """Start points of every mixed cell: (x [MV, n], tau0 [MV], cell id [MV], z [MV, n])."""
    xs, taus, ids, zs = [], [], [], []
    cells = mixed_cells_fast(system) if fast else mixed_cells(system)
    for ci, cell in enumerate(cells):
        x, t0, z = cell_start_points(system, cell, L, tau_cap, zmax)
        xs.append(x)
        zs.append(z)
        taus.append(np.full(len(x), t0))
        ids.append(np.full(len(x), ci))
    return (np.concatenate(xs), np.concatenate(taus), np.concatenate(ids), np.concatenate(zs))


def load_cells(name: str, lift_max: int):
    """Cells stored by workloads.make_starts (exact rational alpha/gap restored)."""
    d = np.load(os.path.join(DATA_DIR, f"{name}_L{lift_max}.npz"), allow_pickle=False)
    cells = []
    for c in range(len(d["volume"])):
        pr = [(int(a), int(b)) for a, b in d["pairs"][c]]
        al = [Fraction(int(nu), int(de)) for nu, de in zip(d["alpha_num"][c], d["alpha_den"][c])]
        cells.append({"pairs": pr, "alpha": al, "gap": Fraction(d["gap"][c]).limit_denominator(10**12),
                      "volume": int(d["volume"][c]), "V": None})
    return cells


def start_points_from_cells(system, cells, L: float = 37.0):
    """Start points (log coordinates z, tau0 per path, cell ids) from stored cells."""
    n = system.n
    zs, taus, ids = [], [], []
    for ci, cell in enumerate(cells):
        if cell.get("V") is None:
            cell = dict(cell)
            cell["V"] = [[int(system.exps[p][j]) - int(system.exps[q][j]) for j in range(n)]
                         for (p, q) in cell["pairs"]]
        _, t0, z = cell_start_points(system, cell, L)
        zs.append(z)
        taus.append(np.full(len(z), t0))
        ids.append(np.full(len(z), ci))
    return np.concatenate(zs), np.concatenate(taus), np.concatenate(ids)


def cell_lifts_fast(system, cells) -> np.ndarray:
    """cell_lifts() with exact integer arithmetic over a common denominator per cell (numpy
    object ints; integer liftings required)."""
    import math
    n, M = system.n, system.M
    E = system.exps.astype(object)
    w = np.array([int(v) for v in system.lifting], dtype=object)
    eq = np.zeros(M, np.int64)
    for k in range(n):
        eq[system.terms_of(k)] = k
    W = np.zeros((len(cells), M))
    for ci, cell in enumerate(cells):
        al = cell["alpha"]
        D = 1
        for a in al:
            D = D * a.denominator // math.gcd(D, a.denominator)
        num = np.array([int(a.numerator * (D // a.denominator)) for a in al], dtype=object)
        val = E.dot(num) + w * D                     # (<a_i, alpha> + omega_i) * D, exact
        beta = np.array([val[cell["pairs"][k][0]] for k in range(n)], dtype=object)
        sh = val - beta[eq]
        if any(v < 0 for v in sh):
            raise RuntimeError("negative shifted lifting: not a lower cell")
        W[ci] = [float(v) / D for v in sh]
    return W


def cell_lifts(system, cells) -> np.ndarray:
    """Cell-shifted liftings omega'_i = omega_i + <a_i, alpha> - beta_k(i) of every term, per cell
    ([ncells, M], exact rationals rounded once).  In cell coordinates x = e^{tau alpha} y the scaled
    homotopy e^{-tau beta_k} h_k is again polyhedral with these liftings (include/pht.h
    pht_track_cells); they are >= 0, = 0 on the cell's two terms of each equation."""
    n = system.n
    M = system.M
    W = np.zeros((len(cells), M))
    lift = [Fraction(v).limit_denominator(10**9) for v in system.lifting]
    for ci, cell in enumerate(cells):
        al = cell["alpha"]
        for k in range(n):
            p0 = cell["pairs"][k][0]
            beta = sum(Fraction(int(system.exps[p0][j])) * al[j] for j in range(n)) + lift[p0]
            for i in system.terms_of(k):
                v = sum(Fraction(int(system.exps[i][j])) * al[j] for j in range(n)) + lift[i] - beta
                if v < 0:
                    raise RuntimeError("negative shifted lifting: not a lower cell")
                W[ci, i] = float(v)
    return W


def start_points_cells(system, cells, L: float = 37.0):
    """Start data for cell-coordinate tracking: (w0 = log y [P, n], tau0 [P], cell id [P])."""
    n = system.n
    ws, taus, ids = [], [], []
    for ci, cell in enumerate(cells):
        if cell.get("V") is None:
            cell = dict(cell)
            cell["V"] = [[int(system.exps[p][j]) - int(system.exps[q][j]) for j in range(n)]
                         for (p, q) in cell["pairs"]]
        _, t0, z = cell_start_points(system, cell, L)
        alpha = np.array([float(a) for a in cell["alpha"]])
        ws.append(z - t0 * alpha[None, :])
        taus.append(np.full(len(z), t0))
        ids.append(np.full(len(z), ci, np.int32))
    return np.concatenate(ws), np.concatenate(taus), np.concatenate(ids)
