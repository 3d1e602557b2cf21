"""Pins for the oracle's evaluation (oracle.c orc_evaluate / orc_evaluate_x).

Each test fixes the oracle against something other than itself (task rule ③):
hand-computed worked examples, closed forms, complex-step and Cauchy-contour
derivatives, finite differences, exact rational arithmetic and known roots.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _cx(v):
    return complex(float(Fraction(v[0])), float(Fraction(v[1])))


def _system_from_golden(g):
    eqs = [[(tuple(a), complex(*c), w) for a, c, w in eq] for eq in g["equations"]]
    return W.from_terms("golden", len(eqs), eqs, coeffs="native")


def test_worked_example_cyclic3_exact():
    """cyclic-3 at x=(1+i, 2, -1), t=2 — all values exact."""
    g = _golden("cyclic3_worked_example.json")
    o = oracle.Oracle(_system_from_golden(g))
    x = np.array([[_cx(v) for v in g["x"]]])
    r = o.evaluate(x, np.array([g["t"]]))
    assert np.array_equal(r["H"][0], np.array([_cx(v) for v in g["H"]]))
    assert np.array_equal(r["Jx"][0], np.array([[_cx(v) for v in row] for row in g["Jx"]]))
    assert np.array_equal(r["Jt"][0], np.array([_cx(v) for v in g["Jt"]]))
    # dH/dtau = t dH/dt (Eq. (2))
    assert np.array_equal(g["t"] * r["Jt"][0], np.array([_cx(v) for v in g["dH_dtau"]]))


def test_spec_extended_jacobian_blocks():
    """S:222 [2,3,8,5] and S:232 [2,3,10,7]: h = 2 y1 t + 3 yh t^2 (tau-derivative via t dh/dt)."""
    g = _golden("spec_examples.json")
    terms = [(tuple(a), complex(*c), w) for a, c, w in g["block_system"]["terms"]]
    sysm = W.from_terms("spec", 2, [terms, [((0, 1), 1.0, 0), ((0, 0), -1.0, 0)]], coeffs="native")
    o = oracle.Oracle(sysm)
    for case in g["block_cases"]:
        t = np.exp(case["tau"])
        r = o.evaluate(np.array([case["y"]], np.complex128), np.array([t]))
        got = [r["Jx"][0, 0, 0], r["Jx"][0, 0, 1], t * r["Jt"][0, 0], r["H"][0, 0]]
        assert np.allclose(got, case["block"], rtol=0, atol=1e-15), (case, got)


def test_cyclic_native_at_ones_closed_form():
    """cyclic-n at x = 1: f_k = n (k<n), f_n = 0; df_k/dx_j = k (each variable lies in
    exactly k of the n cyclic windows of length k), last row all ones."""
    for n in (3, 5, 7, 10):
        o = oracle.Oracle(W.cyclic(n, coeffs="native"))
        r = o.evaluate(np.ones((1, n), np.complex128), np.ones(1))
        H = np.full(n, float(n))
        H[-1] = 0.0
        J = np.array([[k + 1] * n for k in range(n - 1)] + [[1] * n], float)
        assert np.array_equal(r["H"][0], H)
        assert np.array_equal(r["Jx"][0], J)


def test_cyclic_odd_roots_of_unity_are_roots():
    """x_j = w^j, w = e^{2 pi i/n}, is a root of cyclic-n for odd n (F = H(.,1))."""
    for n in (3, 5, 7, 9):
        o = oracle.Oracle(W.cyclic(n, coeffs="native"))
        x = np.exp(2j * np.pi * np.arange(n) / n)[None, :]
        r = o.evaluate(x, np.ones(1))
        assert np.max(np.abs(r["H"])) <= 1e-13 * np.max(r["SH"])


def _rand_small_system(rng, n, terms, emin=-2, emax=3, lmax=5, real=False):
    eqs = []
    for _ in range(n):
        seen = {}
        while len(seen) < terms:
            a = tuple(int(v) for v in rng.integers(emin, emax + 1, size=n))
            c = complex(int(rng.integers(-3, 4)), 0 if real else int(rng.integers(-3, 4)))
            if c == 0:
                c = 1
            seen[a] = (c, int(rng.integers(0, lmax + 1)))
        eqs.append([(a, c, w) for a, (c, w) in seen.items()])
    return W.from_terms("rand", n, eqs, coeffs="native")


def _exact_eval(system, x, t):
    """Exact rational evaluation of Eq. (1) and its derivatives (Gaussian rationals as pairs)."""
    def cm(a, b):
        return (a[0] * b[0] - a[1] * b[1], a[0] * b[1] + a[1] * b[0])

    def cinv(a):
        d = a[0] * a[0] + a[1] * a[1]
        return (a[0] / d, -a[1] / d)

    def cpow(a, e):
        r = (Fraction(1), Fraction(0))
        base = a if e >= 0 else cinv(a)
        for _ in range(abs(e)):
            r = cm(r, base)
        return r

    n = system.n
    X = [(Fraction(v.real), Fraction(v.imag)) for v in x]
    T = Fraction(t)
    H, Jx, Jt = [], [], []
    for k in range(n):
        h = (Fraction(0), Fraction(0))
        hx = [(Fraction(0), Fraction(0))] * n
        ht = (Fraction(0), Fraction(0))
        for i in system.terms_of(k):
            a = [int(v) for v in system.exps[i]]
            c = (Fraction(system.coeffs[i].real), Fraction(system.coeffs[i].imag))
            w = int(system.lifting[i])
            mono = (Fraction(1), Fraction(0))
            for j in range(n):
                mono = cm(mono, cpow(X[j], a[j]))
            term = cm(c, mono)
            tw = T ** w
            h = (h[0] + term[0] * tw, h[1] + term[1] * tw)
            if w >= 1:
                f = w * T ** (w - 1)
                ht = (ht[0] + term[0] * f, ht[1] + term[1] * f)
            for j in range(n):
                if a[j]:
                    d = cm(c, (Fraction(a[j]), Fraction(0)))
                    for l in range(n):
                        d = cm(d, cpow(X[l], a[l] - (1 if l == j else 0)))
                    hx[j] = (hx[j][0] + d[0] * tw, hx[j][1] + d[1] * tw)
        H.append(h)
        Jx.append(hx)
        Jt.append(ht)
    return H, Jx, Jt


def test_exact_gaussian_rational_cases():
    """Gaussian-integer coefficients, points in {+-1, +-i, +-2, 1+-i}, t in {1, 2, 1/2}: every
    entry is a dyadic Gaussian rational representable in double, so the oracle must equal
    exact rational arithmetic bit for bit (SURVEY §8(c) O1 pin)."""
    rng = np.random.default_rng(5)
    pts = [1, -1, 1j, -1j, 2, -2, 1 + 1j, 1 - 1j]
    for trial in range(12):
        n = int(rng.integers(1, 4))
        sysm = _rand_small_system(rng, n, int(rng.integers(1, 5)))
        o = oracle.Oracle(sysm)
        x = np.array([[pts[int(i)] for i in rng.integers(0, len(pts), size=n)]], np.complex128)
        t = float([1.0, 2.0, 0.5][trial % 3])
        r = o.evaluate(x, np.array([t]))
        H, Jx, Jt = _exact_eval(sysm, x[0], t)
        for k in range(n):
            assert r["H"][0, k] == complex(float(H[k][0]), float(H[k][1]))
            assert r["Jt"][0, k] == complex(float(Jt[k][0]), float(Jt[k][1]))
            for j in range(n):
                assert r["Jx"][0, k, j] == complex(float(Jx[k][j][0]), float(Jx[k][j][1]))


def test_complex_step_derivatives_real_systems():
    """Complex step: for real coefficients at real (x, t), df/dx_j = Im f(x + i h e_j)/h,
    h = 1e-30, exact to rounding — independent of the symbolic derivative."""
    for sysm in (W.cyclic(5, coeffs="native"), W.katsura(4, coeffs="native"),
                 W.noon(4, coeffs="native"), W.chandra(5, coeffs="native")):
        sysm = sysm.with_lifting(np.random.default_rng(1).integers(0, 6, sysm.M))
        o = oracle.Oracle(sysm)
        n = sysm.n
        rng = np.random.default_rng(2)
        x = rng.uniform(0.5, 1.5, (3, n)) * rng.choice([-1, 1], (3, n))
        t = rng.uniform(0.2, 1.0, 3)
        r = o.evaluate(x.astype(np.complex128), t)
        for j in range(n):
            xs = x.astype(np.complex128)
            xs[:, j] += 1e-30j
            Hs = o.evaluate(xs, t)["H"]
            d = Hs.imag / 1e-30
            assert np.allclose(d, r["Jx"][:, :, j].real, rtol=1e-13, atol=1e-13 * r["SJx"][:, :, j].max())


def test_cauchy_contour_derivatives_complex_points():
    """df/dx_j = (1/2 pi i) contour integral f(zeta)/(zeta - x_j)^2 on |zeta - x_j| = 0.1|x_j|;
    the trapezoid rule with 64 nodes converges geometrically (holomorphic Laurent terms)."""
    rng = np.random.default_rng(3)
    sysm = _rand_small_system(rng, 3, 5)
    o = oracle.Oracle(sysm)
    n = 3
    z = rng.uniform(-0.5, 0.5, (2, n)) + 1j * rng.uniform(-np.pi, np.pi, (2, n))
    x = np.exp(z)
    t = np.array([0.7, 0.3])
    r = o.evaluate(x, t)
    N = 64
    th = 2 * np.pi * np.arange(N) / N
    for j in range(n):
        acc = np.zeros((2, n), np.complex128)
        for q in range(N):
            xs = x.copy()
            rad = 0.1 * np.abs(x[:, j]) * np.exp(1j * th[q])
            xs[:, j] = x[:, j] + rad
            acc += o.evaluate(xs, t)["H"] / rad[:, None]
        d = acc / N
        assert np.allclose(d, r["Jx"][:, :, j], rtol=1e-11, atol=1e-11 * r["SJx"].max())


def test_finite_difference_t_derivative():
    """Central differences in t (S:242 tolerance 1e-6) pin dH/dt."""
    sysm = W.cyclic(5, lift_max=7)
    o = oracle.Oracle(sysm)
    x, t, _ = W.random_points(4, 5, seed=11)
    r = o.evaluate(x, t)
    h = 1e-6
    d = (o.evaluate(x, t * (1 + h))["H"] - o.evaluate(x, t * (1 - h))["H"]) / (2 * h * t[:, None])
    assert np.allclose(d, r["Jt"], rtol=1e-6, atol=1e-6 * r["SJt"].max())


def test_target_identity_H_at_t1_equals_F():
    """H(x,1) = F(x), F written separately with numpy powers."""
    for sysm in (W.cyclic(5), W.katsura(5), W.noon(5)):
        o = oracle.Oracle(sysm)
        x, _, _ = W.random_points(6, sysm.n, seed=4)
        H = o.evaluate(x, np.ones(6))["H"]
        F = np.zeros_like(H)
        for k in range(sysm.n):
            for i in sysm.terms_of(k):
                F[:, k] += sysm.coeffs[i] * np.prod(x ** sysm.exps[i][None, :], axis=1)
        assert np.allclose(H, F, rtol=1e-13, atol=1e-13)


def test_t_zero_keeps_only_unlifted_terms():
    """t -> 0: H(x,0) = sum of the omega = 0 terms (0^0 = 1)."""
    sysm = W.cyclic(5, lift_max=3)
    o = oracle.Oracle(sysm)
    x, _, _ = W.random_points(3, 5, seed=8)
    H = o.evaluate(x, np.zeros(3))["H"]
    ref = np.zeros_like(H)
    for k in range(5):
        for i in sysm.terms_of(k):
            if sysm.lifting[i] == 0:
                ref[:, k] += sysm.coeffs[i] * np.prod(x ** sysm.exps[i][None, :], axis=1)
    assert np.allclose(H, ref, rtol=1e-14, atol=1e-14)


def test_weighted_sum_identities():
    """Euler-type identities of the log formulation: sum_j x_j dh_k/dx_j =
    sum_i (1^T a_i) T_i and t dh_k/dt = sum_i omega_i T_i, checked with per-term values
    computed by numpy powers."""
    sysm = W.random_dense(4, 6, seed=2)
    o = oracle.Oracle(sysm)
    x, t, _ = W.random_points(5, 4, seed=9, rho_max=0.3)
    r = o.evaluate(x, t)
    for k in range(4):
        lhs1 = np.einsum("pj,pj->p", x, r["Jx"][:, k, :])
        lhs2 = t * r["Jt"][:, k]
        rhs1 = np.zeros(5, np.complex128)
        rhs2 = np.zeros(5, np.complex128)
        for i in sysm.terms_of(k):
            T = sysm.coeffs[i] * np.prod(x ** sysm.exps[i][None, :], axis=1) * t ** sysm.lifting[i]
            rhs1 += sysm.exps[i].sum() * T
            rhs2 += sysm.lifting[i] * T
        assert np.allclose(lhs1, rhs1, rtol=1e-12, atol=1e-12 * r["SH"].max() * 10)
        assert np.allclose(lhs2, rhs2, rtol=1e-12, atol=1e-12 * r["SH"].max() * 10)


def test_extended_range_matches_double_in_range():
    """O2: in range the extended-range evaluation equals the double evaluation bit for bit,
    and x_j <- 2^s x_j shifts every monomial's binary exponent by s a_j exactly."""
    sysm = W.noon(4, lift_max=20)
    o = oracle.Oracle(sysm)
    x, t, _ = W.random_points(4, 4, seed=21)
    r = o.evaluate(x, t)
    xm, xe = x.copy(), np.zeros(x.shape, np.int64)
    rx = o.evaluate_x(xm, xe, t, np.zeros(4, np.int64))
    for key, m, e in (("H", "Hm", "He"), ("Jx", "Jxm", "Jxe"), ("Jt", "Jtm", "Jte")):
        v = rx[m] * np.exp2(rx[e].astype(float))
        assert np.array_equal(v, r[key]), key
    # exponent shift: scale x_0 by 2^s; a pure-monomial system makes the shift exact per entry
    mono = W.from_terms("mono", 2, [[((3, -2), 1.0, 4)], [((-1, 5), 1.0 + 1j, 2)]], coeffs="native")
    om = oracle.Oracle(mono)
    xm = np.array([[0.75 + 0.25j, -0.5 + 0.625j]])
    base = om.evaluate_x(xm, np.zeros((1, 2), np.int64), np.array([0.5]), np.zeros(1, np.int64))
    s = 10_000
    sh = om.evaluate_x(xm, np.array([[s, 0]]), np.array([0.5]), np.zeros(1, np.int64))
    assert np.array_equal(sh["Hm"], base["Hm"])
    assert sh["He"][0, 0] - base["He"][0, 0] == 3 * s
    assert sh["He"][0, 1] - base["He"][0, 1] == -1 * s


def test_extended_range_large_lifting_against_exact_logs():
    """Large liftings (noon-style, omega ~ 1e4, t = 2^-k): log2|h_k| of a one-term equation is
    known in closed form: log2|c| + sum a_j log2|x_j| + omega log2 t."""
    mono = W.from_terms("mono", 2, [[((2, 1), 1.0, 9000)], [((0, 3), 2.0, 12345)]], coeffs="native")
    om = oracle.Oracle(mono)
    xm = np.array([[0.5 + 0.5j, 0.5 - 0.25j]])
    r = om.evaluate_x(xm, np.zeros((1, 2), np.int64), np.array([0.5]), np.array([-3], np.int64))
    l2 = np.log2(np.abs(r["Hm"][0])) + r["He"][0]
    lx = np.log2(np.abs(xm[0]))
    ref0 = 2 * lx[0] + lx[1] + 9000 * (-4)
    ref1 = 1 + 3 * lx[1] + 12345 * (-4)
    assert abs(l2[0] - ref0) < 1e-9 and abs(l2[1] - ref1) < 1e-9


def test_generator_monomial_counts():
    """P:901 (cyclic-14: 184 monomials), P:928 (chandra-24: 324); SURVEY §8 table."""
    assert W.cyclic(14).union_support_size() == 184
    assert W.chandra(24).union_support_size() == 324
    assert W.cyclic(5).M == 22 and W.cyclic(10).M == 92
    assert W.katsura(10).M == 107 and W.noon(10).M == 110
    assert W.random_dense().M == 1000
