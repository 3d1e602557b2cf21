"""Pins for the oracle's projective formulation (Eq. (3)) and projective directions
(P:237-252), SURVEY §8(f) f1.  Each pin follows from the mathematics, not from
the oracle's code: dehomogenisation, Euler's homogeneous-function theorem, homogeneity under
scaling, the closed-form relation between projective and affine Newton directions for systems
of equal degree, the closed-form Euler direction on a diagonal system's path, and a target
with a solution at infinity at a known point of P^n."""
import numpy as np

import oracle
import workloads as W
from workloads import param as PH
from workloads import startsys as SS


def _deg(sysm):
    return np.array([sysm.exps[sysm.terms_of(k)].sum(axis=1).max() for k in range(sysm.n)])


def test_dehomogenisation_and_euler_theorem():
    for sysm in (W.cyclic(5, lift_max=20), W.katsura(4, lift_max=20), W.chandra(5, lift_max=20)):
        o = oracle.Oracle(sysm)
        n = sysm.n
        x, t, _ = W.random_points(40, n, seed=5)
        ra = o.evaluate(x, t)
        y = np.concatenate([x, np.ones((40, 1))], axis=1)
        rp = o.proj_evaluate(y, t)
        # y = (x, 1): H^ = H, dH^/dy_j = dH/dx_j (j < n), dH^/dt = dH/dt
        assert np.max(np.abs(rp["H"] - ra["H"]) / ra["SH"]) < 1e-14
        assert np.max(np.abs(rp["Jy"][:, :, :n] - ra["Jx"]) / np.maximum(ra["SJx"], 1e-300)) < 1e-14
        assert np.max(np.abs(rp["Jt"] - ra["Jt"]) / np.maximum(ra["SJt"], 1e-300)) < 1e-14
        # Euler's theorem at arbitrary y: sum_j y_j dh^_k/dy_j = deg_k h^_k
        z, _ = W.random_log_points(40, n + 1, seed=6)
        y = np.exp(z)
        rp = o.proj_evaluate(y, t)
        lhs = np.einsum("pkj,pj->pk", rp["Jy"], y)
        scale = np.einsum("pkj,pj->pk", rp["SJy"], np.abs(y)) + rp["SH"]
        assert np.max(np.abs(lhs - _deg(sysm)[None] * rp["H"]) / scale) < 1e-13
        # homogeneity: H^(l y) = l^deg H^(y)
        lam = 0.7 - 1.3j
        r2 = o.proj_evaluate(lam * y, t)
        assert np.max(np.abs(r2["H"] - lam ** _deg(sysm)[None] * rp["H"]) / (np.abs(lam) ** _deg(sysm)[None] * rp["SH"])) < 1e-13


def test_projective_newton_closed_form_equal_degree():
    """All equations of degree d (noon-4: d = 3).  At y = (x, 1), with N_a the affine Newton
    direction: N = mu (N_a, 0) - lam y, lam = mu x^* N_a / ||y||^2, mu = 1 / (1 + d x^* N_a / ||y||^2)
    (from dH^/dy y = d H^ and y^* N = 0)."""
    sysm = W.noon(4, lift_max=20)
    assert np.all(_deg(sysm) == 3)
    o = oracle.Oracle(sysm)
    x, t, _ = W.random_points(30, 4, seed=8, tau_lo=-0.05)
    _, Na, sa = o.euler_newton(x, t)
    y = np.concatenate([x, np.ones((30, 1))], axis=1)
    E, N, sp = o.proj_euler_newton(y, t)
    assert np.all(sa == 0) and np.all(sp == 0)
    y2 = np.sum(np.abs(y) ** 2, axis=1)
    xn = np.sum(np.conj(x) * Na, axis=1)
    mu = 1.0 / (1.0 + 3 * xn / y2)
    lam = mu * xn / y2
    Nref = mu[:, None] * np.concatenate([Na, np.zeros((30, 1))], axis=1) - lam[:, None] * y
    assert np.max(np.linalg.norm(N - Nref, axis=1) / np.linalg.norm(Nref, axis=1)) < 1e-10


def test_projective_euler_on_diagonal_path():
    """h_k = x_k^d - b_k t^{w_k} (all degree d): on the path x_k = (b_k t^{w_k})^{1/d} the affine
    Euler direction is dx_k/dtau = (w_k / d) x_k; the projective one is its projection onto y^perp
    at y = (x, 1) (dH^/dy y = d H^ = 0 on the path)."""
    d, b, w = 3, [0.5 + 1j, -2.0, 1j], [3, 5, 2]
    sysm = W.diagonal([d] * 3, b, w)
    o = oracle.Oracle(sysm)
    tau = -0.7
    x = np.array([[(complex(b[k]) * np.exp(w[k] * tau)) ** (1.0 / d) for k in range(3)]])
    Ea = np.array([[w[k] / d * x[0, k] for k in range(3)]])
    y = np.concatenate([x, np.ones((1, 1))], axis=1)
    E, N, st = o.proj_euler_newton(y, np.array([np.exp(tau)]))
    v = np.concatenate([Ea, np.zeros((1, 1))], axis=1)
    Eref = v - y * (np.sum(np.conj(y) * v) / np.sum(np.abs(y) ** 2))
    assert st[0] == 0
    assert np.max(np.abs(E - Eref)) < 1e-13 * np.abs(Eref).max()
    assert np.max(np.abs(N)) < 1e-13


def test_projective_step_stays_on_sphere_and_newton_converges():
    """Projective Newton (h = 0, K iterations) from a perturbed solution of cyclic-5 returns to the
    projective point of that solution (quadratic convergence); every update stays on ||y|| = 1."""
    c5 = W.cyclic(5, lift_max=100)
    x, tau0, _, _ = SS.start_points(c5, zmax=20)
    o = oracle.Oracle(c5)
    xs, _, st, _ = o.track(x[:20], tau0[:20])
    assert np.all(st == 0)
    y = np.concatenate([xs, np.ones((20, 1))], axis=1)
    y /= np.linalg.norm(y, axis=1, keepdims=True)
    rng = np.random.default_rng(2)
    yp = y + 1e-4 * (rng.normal(size=y.shape) + 1j * rng.normal(size=y.shape))
    yp /= np.linalg.norm(yp, axis=1, keepdims=True)
    y2, t2, st, dn = o.proj_pc_step(yp, np.zeros(20), np.zeros(20), K=4)
    assert np.all(st == 0)
    assert np.allclose(np.linalg.norm(y2, axis=1), 1.0, atol=1e-15)
    assert np.max(dn) < 1e-12                      # last correction at rounding level
    x2 = y2[:, :5] / y2[:, 5:]
    assert np.max(np.abs(x2 - xs) / np.abs(xs)) < 1e-12


def test_projective_tracker_solution_at_infinity():
    """F = {x1 + x2 - 1, x1^2 + x1 x2 + x1 + x2 - 3}: mixed volume 2, one finite solution
    (2, -1) and one at infinity, the common zero (1 : -1 : 0) of the leading forms x1 + x2 and
    x1 (x1 + x2).  The projective second stage reaches both; the affine one loses the second."""
    eqs = [[((1, 0), 1.0), ((0, 1), 1.0), ((0, 0), -1.0)],
           [((2, 0), 1.0), ((1, 1), 1.0), ((1, 0), 1.0), ((0, 1), 1.0), ((0, 0), -3.0)]]
    F = W.from_terms("inf2", 2, eqs, coeffs="native", lift_max=100)
    G = W.from_terms("inf2", 2, eqs, coeffs="random", lift_max=100)
    cells = SS.mixed_cells(G)
    assert sum(c["volume"] for c in cells) == 2
    Wc = SS.cell_lifts(G, cells)
    w0, tau0, cid = SS.start_points_cells(G, cells)
    m, e = oracle.z_to_x(w0)
    xm, xe, _, s1, _ = oracle.Oracle(G).track_x(m, e, tau0, cell_lift=Wc, path_cell=cid)
    x1 = xm * np.exp2(xe.astype(float))
    assert np.all(s1 == 0)
    H2 = PH.parameter_homotopy(G, F.coeffs)
    y1 = np.concatenate([x1, np.ones((2, 1))], axis=1)
    y1 /= np.linalg.norm(y1, axis=1, keepdims=True)
    y2, _, s2, _ = oracle.Oracle(H2).proj_track(y1, np.full(2, PH.TAU0))
    fin = s2 == 0
    assert fin.sum() == 1 and np.sum(s2 == oracle.PT_DIVERGED) == 1
    xf = y2[fin, :2] / y2[fin, 2:]
    assert np.allclose(xf, [[2.0, -1.0]], atol=1e-12)
    yi = y2[~fin][0]
    yi = yi / yi[0]
    assert np.allclose(yi, [1.0, -1.0, 0.0], atol=1e-12)
    _, _, sa, _ = oracle.Oracle(H2).track(x1, np.full(2, PH.TAU0))
    assert np.sum(sa == 0) == 1
