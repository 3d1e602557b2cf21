"""Pins for the oracle's directions, Euler-Newton step and tracker (oracle.c O3/O4)."""
import json
import os
from fractions import Fraction

import numpy as np

import oracle
import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _cx(v):
    return complex(float(Fraction(v[0])), float(Fraction(v[1])))


def test_worked_example_directions():
    """cyclic-3 worked example: dE = Jx^{-1}(-Jt), dN = Jx^{-1}(-H) are dyadic."""
    with open(os.path.join(GOLD, "cyclic3_worked_example.json")) as f:
        g = json.load(f)
    eqs = [[(tuple(a), complex(*c), w) for a, c, w in eq] for eq in g["equations"]]
    o = oracle.Oracle(W.from_terms("g", 3, eqs, coeffs="native"))
    x = np.array([[_cx(v) for v in g["x"]]])
    dE, dN, st = o.euler_newton(x, np.array([g["t"]]))
    assert st[0] == 0
    assert np.allclose(dE[0], [_cx(v) for v in g["dE"]], rtol=0, atol=1e-15)
    assert np.allclose(dN[0], [_cx(v) for v in g["dN"]], rtol=0, atol=1e-15)


def test_spec_affine_examples():
    """h = x - e^tau gives E = 1, N = 0 at x = 1 and N = -1 at x = 2 (tau = 0)."""
    sysm = W.from_terms("lin", 1, [[((1,), 1.0, 0), ((0,), -1.0, 1)]], coeffs="native")
    o = oracle.Oracle(sysm)
    dE, dN, st = o.euler_newton(np.array([[1.0 + 0j], [2.0 + 0j]]), np.ones(2))
    assert np.allclose(dE[:, 0] * 1.0, [1.0, 1.0]) and np.allclose(dN[:, 0], [0.0, -1.0])


def test_lu_route_equals_paper_qr_route():
    """LU (route 1) == the paper's QR null space (route 2) on random well-conditioned
    extended Jacobians, and both satisfy the defining residuals."""
    rng = np.random.default_rng(7)
    for n in (1, 2, 5, 10, 16):
        for _ in range(5):
            J = rng.normal(size=(n, n + 2)) + 1j * rng.normal(size=(n, n + 2))
            J[:, :n] += 2 * np.sqrt(n) * np.eye(n)
            X, st = oracle.lu_solve(J[:, :n], -J[:, n:])
            dE, dN, st2 = oracle.dirs_qr(J)
            assert st == 0 and st2 == 0
            assert np.allclose(X[:, 0], dE, rtol=1e-12, atol=1e-12)
            assert np.allclose(X[:, 1], dN, rtol=1e-12, atol=1e-12)
            A = J[:, :n]
            for v, rhs in ((dE, J[:, n]), (dN, J[:, n + 1])):
                res = np.linalg.norm(A @ v + rhs)
                assert res <= 1e-12 * (np.linalg.norm(A) * np.linalg.norm(v) + np.linalg.norm(rhs))


def test_lu_singular_flag():
    A = np.array([[1, 2], [2, 4]], np.complex128)
    _, st = oracle.lu_solve(A, np.ones((2, 1)))
    assert st == oracle.PT_SINGULAR
    _, st = oracle.lu_solve(np.zeros((3, 3), np.complex128), np.ones((3, 1)))
    assert st == oracle.PT_SINGULAR


def test_row_scaling_invariance():
    """Scaling a row of [Jx | Jt | H] leaves dE and dN unchanged — the property the
    GPU's row_exp2 convention relies on."""
    rng = np.random.default_rng(8)
    n = 6
    J = rng.normal(size=(n, n + 2)) + 1j * rng.normal(size=(n, n + 2)) + 3 * np.eye(n, n + 2)
    X0, _ = oracle.lu_solve(J[:, :n], -J[:, n:])
    s = 2.0 ** rng.integers(-300, 300, size=n)
    Js = J * s[:, None]
    X1, _ = oracle.lu_solve(Js[:, :n], -Js[:, n:])
    assert np.allclose(X0, X1, rtol=1e-13, atol=1e-13)


def test_diagonal_closed_form_directions():
    """h_k = x_k^d - b_k t^w: on the path x_k^d = b_k t^w, dx_k/dtau = (w/d) x_k; off the path
    the Newton step is -(x^d - b t^w)/(d x^{d-1}) (SURVEY §8(c) O3 closed form)."""
    d, b, w = [2, 3, 1], [0.5 + 1j, -2.0, 1j], [3, 5, 2]
    o = oracle.Oracle(W.diagonal(d, b, w))
    t = 0.4
    x_on = np.array([[(complex(b[k]) * t ** w[k]) ** (1.0 / d[k]) for k in range(3)]])
    dE, dN, st = o.euler_newton(x_on, np.array([t]))
    assert np.allclose(t * dE[0], [w[k] / d[k] * x_on[0, k] for k in range(3)], rtol=1e-13)
    assert np.allclose(dN[0], 0, atol=1e-15)
    x_off = x_on * 1.1
    _, dN, _ = o.euler_newton(x_off, np.array([t]))
    ref = [-(x_off[0, k] ** d[k] - b[k] * t ** w[k]) / (d[k] * x_off[0, k] ** (d[k] - 1)) for k in range(3)]
    assert np.allclose(dN[0], ref, rtol=1e-13)


def test_pc_step_linear_path_is_exact():
    """h = x - t (x = e^tau): an Euler step plus one Newton iteration lands exactly on the path
    because h is linear in x (the protocol of P:911-920)."""
    sysm = W.from_terms("lin", 1, [[((1,), 1.0, 0), ((0,), -1.0, 1)]], coeffs="native")
    o = oracle.Oracle(sysm)
    tau = np.array([-2.0, -0.7, -0.01])
    x = np.exp(tau)[:, None].astype(np.complex128)
    x1, tau1, st, dn = o.pc_step(x, tau, np.array([0.3, 0.5, 0.01]), K=1)
    assert np.allclose(x1[:, 0], np.exp(tau1), rtol=1e-14)


def test_pc_step_diagonal_newton_converges():
    d, b, w = [2, 3], [0.5 + 1j, -2.0], [3, 5]
    o = oracle.Oracle(W.diagonal(d, b, w))
    tau = np.array([-1.0])
    t = np.exp(tau[0])
    x = np.array([[(complex(b[k]) * t ** w[k]) ** (1.0 / d[k]) for k in range(2)]])
    x1, tau1, st, dn = o.pc_step(x, tau, np.array([0.05]), K=4)
    t1 = np.exp(tau1[0])
    assert np.allclose(x1[0] ** np.array(d), [b[k] * t1 ** w[k] for k in range(2)], rtol=1e-13)
    assert dn[0] < 1e-12


def test_track_diagonal_all_roots():
    """Tracking tau0 -> 0 on a diagonal system reaches every root b_k^{1/d_k} (closed form paths),
    finite count = prod d_k = the mixed volume."""
    d, b, w = [2, 3], [0.5 + 1j, -2.0], [3, 5]
    o = oracle.Oracle(W.diagonal(d, b, w))
    tau0 = -4.0
    t0 = np.exp(tau0)
    r0 = [np.roots([1] + [0] * (d[k] - 1) + [-b[k] * t0 ** w[k]]) for k in range(2)]
    starts = np.array([[u, v] for u in r0[0] for v in r0[1]], np.complex128)
    x, tau, st, stats = o.track(starts, np.full(len(starts), tau0))
    assert np.all(st == 0) and np.all(tau == 0)
    roots = [np.roots([1] + [0] * (d[k] - 1) + [-b[k]]) for k in range(2)]
    for k in range(2):
        for q in range(len(starts)):
            assert np.min(np.abs(roots[k] - x[q, k])) < 1e-12
    ends = {(round(v[0].real, 8), round(v[0].imag, 8), round(v[1].real, 8), round(v[1].imag, 8)) for v in x}
    assert len(ends) == int(np.prod(d))
    # each path's continuation is the closed form (b t^w)^{1/d} on the branch of its start
    for q in range(len(starts)):
        for k in range(2):
            ratio = x[q, k] / starts[q, k]
            ref = (1.0 / t0 ** w[k]) ** (1.0 / d[k])
            assert abs(ratio - ref) < 1e-9 * abs(ref)


def test_track_one_variable_closed_form_path():
    """h = x - e^tau tracked from tau0 = -20 reaches x = 1."""
    sysm = W.from_terms("lin", 1, [[((1,), 1.0, 0), ((0,), -1.0, 1)]], coeffs="native")
    o = oracle.Oracle(sysm)
    x, tau, st, stats = o.track(np.array([[np.exp(-20.0) + 0j]]), np.array([-20.0]))
    assert st[0] == 0 and abs(x[0, 0] - 1) < 1e-13


def test_track_status_isolation():
    """a poisoned start (zero coordinate) fails alone; siblings converge."""
    sysm = W.from_terms("lin", 1, [[((1,), 1.0, 0), ((0,), -1.0, 1)]], coeffs="native")
    o = oracle.Oracle(sysm)
    starts = np.full((8, 1), np.exp(-5.0) + 0j)
    starts[3, 0] = 0
    x, tau, st, stats = o.track(starts, np.full(8, -5.0))
    assert st[3] != 0 and np.sum(st == 0) == 7
