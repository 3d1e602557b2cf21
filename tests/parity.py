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


def solve_bound(J, SJ, d, Srhs):
    """Componentwise forward-error scale of the solution d of J d = rhs when every entry of J and
    rhs carries an error bounded by eps x its term sum (SJ, Srhs; reading R9/A25):
    |delta d| <= eps |J^-1| (SJ |d| + Srhs) to first order.  Returns that vector per point
    (J, SJ: [p,n,n]; d, Srhs: [p,n]).  Invariant under row scaling; it is Skeel's condition
    number measured against the evaluation's own error model instead of |J|."""
    Ai = np.linalg.inv(J)
    return np.einsum("pij,pj->pi", np.abs(Ai), np.einsum("pjk,pk->pj", np.asarray(SJ, float), np.abs(d)) + Srhs)


def coord_err_ratio(got, ref, bound, eps):
    """max_j |got_j - ref_j| / (eps * bound_j) per point (<= 1 passes)."""
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.abs(got - ref) / (eps * bound)
    r = np.where(np.abs(got - ref) == 0, 0.0, r)
    return np.max(r, axis=-1)


def xeval_errs(o, xm, xe, tm, te, H, Jz, Jtau, e2):
    """Term-sum errors (reading R9) of a row-scaled log-coordinate evaluation against the oracle's
    extended-range evaluation o = Oracle.evaluate_x(xm, xe, tm, te) at x = xm 2^xe, t = tm 2^te.
    GPU rows are [Jz | Jtau | H] * 2^-e2 with Jz = Jx diag(x), Jtau = t Jt.  The
    SURVEY A25 floor applies: an entry's scale is max(S, 2^-960 S_row), S_row = the term sum of
    the row's h (entries flushed that far below their row are zero for the solve).  Structurally
    zero entries (S = 0) must be exactly 0.  Returns the maxima (errH, errJz, errJtau)."""
    e2 = np.asarray(e2, np.float64)
    xe = np.asarray(xe, np.float64)
    te = np.asarray(te, np.float64)
    lsh = o["LSH"]

    def err(got, gexp, ref_m, ref_e, ls, row_ls):
        ls_eff = np.maximum(ls, row_ls - 960.0)
        zero = np.isneginf(ls)
        if np.any(zero & (got != 0)):
            return np.inf
        ls_eff = np.where(zero, 0.0, ls_eff)
        d = np.abs(got * np.exp2(gexp - ls_eff) - ref_m * np.exp2(ref_e - ls_eff))
        return float(np.max(np.where(zero, 0.0, d)))

    eH = err(H, e2, o["Hm"], o["He"].astype(float), lsh, lsh)
    lt = np.log2(np.abs(tm)) + te                                    # log2 t
    eT = err(Jtau, e2, o["Jtm"] * tm[:, None], o["Jte"] + te[:, None], o["LSJt"] + lt[:, None], lsh)
    lx = np.log2(np.abs(xm)) + xe                                    # log2 |x_j|
    eJ = err(Jz, e2[:, :, None], o["Jxm"] * xm[:, None, :], o["Jxe"] + xe[:, None, :],
             o["LSJx"] + lx[:, None, :], lsh[:, :, None])
    return eH, eJ, eT


# Per-coordinate direction / step parity (VERDICT r1 "next" 1(iv)).  EPS_SOLVE multiplies the
# componentwise forward-error scale solve_bound(): the first-order error of a solution computed
# from entries carrying errors <= eps x their term sums.  At the parity points (|rho| <= 1,
# |omega tau| <= 5, degree <= 14) the GPU evaluation is within ~6e-15 of the term sums (SURVEY A27:
# 2.7 u Phi + (m + 2) u), the oracle's repeated multiplication within ~3e-15, and both
# eliminations add ~n u times the pivot growth: EPS_SOLVE = 1e-12 leaves a margin of ~50.
EPS_SOLVE = 1e-12
U = 2.0 ** -53


def dirs_parity(o, x, t, dE, dN, st):
    """Directions from the CUDA path (dE = dx/dt, dN) against oracle.euler_newton on the same
    points.  Returns (status sets equal, max backward errors (E, N), max coordinate ratios (E, N))
    over EVERY status-0 point; the ratio is |gpu_j - oracle_j| / (EPS_SOLVE * bound_j)."""
    r = o.evaluate(x, t)
    oE, oN, ost = o.euler_newton(x, t)
    good = st == 0
    same = bool(np.array_equal(good, ost == 0))
    J, SJ = r["Jx"][good], r["SJx"][good]
    be = (backward_err(J, dE[good], -r["Jt"][good]).max(initial=0.0),
          backward_err(J, dN[good], -r["H"][good]).max(initial=0.0))
    bE = solve_bound(J, SJ, oE[good], r["SJt"][good])
    bN = solve_bound(J, SJ, oN[good], r["SH"][good])
    ratio = (coord_err_ratio(dE[good], oE[good], bE, EPS_SOLVE).max(initial=0.0),
             coord_err_ratio(dN[good], oN[good], bN, EPS_SOLVE).max(initial=0.0))
    return same, be, ratio


def step_parity(o, x, tau, dtau, K, xg, stg, taug):
    """Euler-Newton step of the CUDA path (xg, stg, taug after pht_pc_step) against oracle.pc_step.
    The coordinate bound accumulates the solve bounds of the Euler direction (times h t, since
    dx/dtau = t dx/dt) and of each Newton direction at the oracle's own intermediate points,
    plus the rounding of the updates (8 u |x_j|).  Returns (statuses equal, tau equal,
    max coordinate ratio over every status-0 point)."""
    xo, tauo, sto, _ = o.pc_step(x, tau, dtau, K=K)
    good = (stg == 0) & (sto == 0)
    t = np.exp(tau)
    r0 = o.evaluate(x, t)
    oE, _, _ = o.euler_newton(x, t)
    h = np.broadcast_to(np.asarray(dtau, float), (len(x),))
    with np.errstate(all="ignore"):
        bound = (h * t)[:, None] * solve_bound(r0["Jx"], r0["SJx"], oE, r0["SJt"])
        xt = x + (h * t)[:, None] * oE
        tt = np.exp(tau + h)
        for _ in range(K):
            r = o.evaluate(xt, tt)
            _, oN, _ = o.euler_newton(xt, tt)
            bound = bound + solve_bound(r["Jx"], r["SJx"], oN, r["SH"])
            xt = xt + oN
    d = np.abs(xg[good] - xo[good])
    den = EPS_SOLVE * bound[good] + 8 * U * np.abs(xo[good])
    ratio = float(np.max(np.where(d == 0, 0.0, d / den), initial=0.0))
    return bool(np.array_equal(stg == 0, sto == 0)), bool(np.array_equal(taug, tauo)), ratio
