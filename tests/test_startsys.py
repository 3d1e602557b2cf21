"""Pins for the start-system generator (workload prep) and for the oracle
tracker's solution count (Bernshtein: generic coefficients -> #solutions = mixed volume)."""
import numpy as np
import pytest

import oracle
import workloads as W
from workloads import startsys as SS


def _hull_area(pts):
    pts = sorted(set(map(tuple, pts)))
    if len(pts) < 3:
        return 0.0

    def cross(o, a, b):
        return (a[0] - o[0]) * (b[1] - o[1]) - (a[1] - o[1]) * (b[0] - o[0])
    lower, upper = [], []
    for p in pts:
        while len(lower) >= 2 and cross(lower[-2], lower[-1], p) <= 0:
            lower.pop()
        lower.append(p)
    for p in reversed(pts):
        while len(upper) >= 2 and cross(upper[-2], upper[-1], p) <= 0:
            upper.pop()
        upper.append(p)
    h = lower[:-1] + upper[:-1]
    return 0.5 * abs(sum(h[i][0] * h[(i + 1) % len(h)][1] - h[(i + 1) % len(h)][0] * h[i][1] for i in range(len(h))))


def test_mixed_volume_n2_area_formula():
    """MV(P1, P2) = area(P1 + P2) - area(P1) - area(P2) for n = 2 (independent of the cells)."""
    rng = np.random.default_rng(3)
    cases = [[[(2, 0), (0, 1), (0, 0)], [(1, 1), (1, 0), (0, 2), (0, 0)]]]  # MV = 4
    for _ in range(6):
        cases.append([[tuple(int(v) for v in rng.integers(0, 4, 2)) for _ in range(4)] for _ in range(2)])
    for sup in cases:
        sup = [sorted(set(s)) for s in sup]
        if min(len(s) for s in sup) < 2:
            continue
        sysm = W.from_terms("mv2", 2, [[(a, 1.0) for a in s] for s in sup], lift_max=10**6, seed=11)
        mink = [(a[0] + b[0], a[1] + b[1]) for a in sup[0] for b in sup[1]]
        ref = _hull_area(mink) - _hull_area(sup[0]) - _hull_area(sup[1])
        assert SS.mixed_volume(sysm) == round(ref), (sup, ref)


def test_cyclic5_mixed_volume_is_70():
    """BASELINE.json configs[0]: cyclic-5 has 70 solutions (= its mixed volume)."""
    assert SS.mixed_volume(W.cyclic(5, lift_max=1000)) == 70


def test_start_points_solve_the_binomial_systems():
    sysm = W.cyclic(4, lift_max=1000)
    for cell in SS.mixed_cells(sysm):
        x, tau0, z = SS.cell_start_points(sysm, cell)
        alpha = np.array([float(a) for a in cell["alpha"]])
        y = np.exp(z - tau0 * alpha[None, :])
        assert len(x) == cell["volume"]
        for (j0, j1) in cell["pairs"]:
            a0, a1 = sysm.exps[j0], sysm.exps[j1]
            lhs = sysm.coeffs[j0] * np.prod(y ** a0, axis=1) + sysm.coeffs[j1] * np.prod(y ** a1, axis=1)
            assert np.max(np.abs(lhs)) < 1e-10
        # all |det V| solutions are distinct
        assert len({tuple(np.round(v, 8)) for v in y}) == len(y)


def test_oracle_tracker_finds_all_cyclic5_solutions():
    """70 start paths -> 70 distinct finite endpoints with H(x, 1) = F(x) ~ 0."""
    c5 = W.cyclic(5, lift_max=100)
    x, tau0, _, _ = SS.start_points(c5, zmax=20)
    assert len(x) == 70
    o = oracle.Oracle(c5)
    xe, te, st, stats = o.track(x, tau0)
    assert np.all(st == 0) and np.all(te == 0)
    r = o.evaluate(xe, np.ones(70))
    assert np.max(np.abs(r["H"]) / r["SH"]) < 1e-13
    assert len({tuple(np.round(v, 7)) for v in xe}) == 70


def test_fast_enumerator_equals_brute_force():
    """The LP-pruned C++ enumerator (workloads/mixedcell.cpp) finds exactly the brute-force cells."""
    for sysm in (W.cyclic(5, lift_max=100), W.cyclic(4, lift_max=1000), W.noon(3, lift_max=100),
                 W.katsura(3, lift_max=100), W.random_dense(3, 5, seed=4, lift_max=10**4)):
        a = {tuple(c["pairs"]) for c in SS.mixed_cells(sysm)}
        b = {tuple(c["pairs"]) for c in SS.mixed_cells_fast(sysm)}
        assert a == b, sysm.name


def test_known_mixed_volumes():
    """Published torus root counts [ext]: noon-n = 3^n - 2n, cyclic-7 = 924 (generic lifting)."""
    assert sum(c["volume"] for c in SS.mixed_cells_fast(W.noon(4, lift_max=1000))) == 3 ** 4 - 8
    assert sum(c["volume"] for c in SS.mixed_cells_fast(W.noon(5, lift_max=1000))) == 3 ** 5 - 10
    assert sum(c["volume"] for c in SS.mixed_cells_fast(W.cyclic(7, lift_max=10 ** 4))) == 924


def test_extended_range_tracker_matches_double_tracker_in_range():
    """orc_track_x (extended range) follows the same algorithm as orc_track: same endpoints when
    the data fit in double (the only difference is the representation)."""
    c5 = W.cyclic(5, lift_max=100)
    x, tau0, _, z = SS.start_points(c5, zmax=20)
    o = oracle.Oracle(c5)
    xa, ta, sa, _ = o.track(x, tau0)
    m, e = oracle.z_to_x(z)
    xm, xe, tb, sb, _ = o.track_x(m, e, tau0, pred_log=0)
    xb = xm * np.exp2(xe.astype(float))
    assert np.array_equal(sa, sb)
    assert np.max(np.abs(xa - xb) / np.abs(xa)) < 1e-10


def test_extended_range_tracker_uncapped_start_points():
    """Start points at the full tau0 = -37/gap (|Re z| up to ~350, outside double range for the
    monomials) -> 70 distinct finite solutions of cyclic-5."""
    c5 = W.cyclic(5, lift_max=100)
    _, tau0, _, z = SS.start_points(c5)
    assert np.abs(z.real).max() > 300
    o = oracle.Oracle(c5)
    m, e = oracle.z_to_x(z)
    xm, xe, te, st, _ = o.track_x(m, e, tau0)
    assert np.all(st == 0)
    xend = xm * np.exp2(xe.astype(float))
    r = o.evaluate(xend, np.ones(70))
    assert np.max(np.abs(r["H"]) / r["SH"]) < 1e-13
    assert len({tuple(np.round(v, 7)) for v in xend}) == 70


def test_log_chart_predictor_same_solutions_fewer_steps():
    """The log-chart Euler predictor (reading R25) reaches the same 70 solutions of cyclic-5 in far
    fewer steps than the affine one (toric paths x ~ e^{tau alpha} y near tau0)."""
    c5 = W.cyclic(5, lift_max=100)
    _, tau0, _, z = SS.start_points(c5)
    o = oracle.Oracle(c5)
    m, e = oracle.z_to_x(z)
    xa, ea, _, sa, sta = o.track_x(m, e, tau0, pred_log=0)
    xb, eb, _, sb, stb = o.track_x(m, e, tau0, pred_log=1)
    assert np.all(sa == 0) and np.all(sb == 0)
    A = xa * np.exp2(ea.astype(float))
    B = xb * np.exp2(eb.astype(float))
    assert np.max(np.abs(A - B) / np.abs(A)) < 1e-10
    assert stb[:, 0].sum() * 5 < sta[:, 0].sum()
