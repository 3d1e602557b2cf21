"""Pins for the second-stage coefficient-parameter homotopy (workloads.param):
H(x, 1) = F(x), H(x, 0) = G(x), and the oracle's two-stage solve of the NATIVE cyclic-5 system
reaches its 70 isolated solutions (a known count) with F-residuals at rounding level."""
import numpy as np

import oracle
import workloads as W
from workloads import param as PH
from workloads import startsys as SS


def _two_stage_oracle(n):
    G = W.cyclic(n, lift_max=100)                          # stage 1: generic coefficients
    F = W.cyclic(n, lift_max=100, coeffs="native")         # target: same supports, native c
    cells = SS.mixed_cells_fast(G)
    Wc = SS.cell_lifts(G, cells)
    w0, tau0, cid = SS.start_points_cells(G, cells)
    m, e = oracle.z_to_x(w0)
    xm, xe, _, s1, _ = oracle.Oracle(G).track_x(m, e, tau0, cell_lift=Wc, path_cell=cid)
    x1 = xm * np.exp2(xe.astype(float))
    H2 = PH.parameter_homotopy(G, F.coeffs)
    ok = s1 == 0
    x2, t2, s2, _ = oracle.Oracle(H2).track(x1[ok], np.full(ok.sum(), PH.TAU0))
    return G, F, H2, x1, s1, x2, s2


def test_parameter_homotopy_end_values():
    G = W.cyclic(6, lift_max=10)
    F = W.cyclic(6, lift_max=10, coeffs="native")
    H2 = PH.parameter_homotopy(G, F.coeffs)
    x, _, _ = W.random_points(50, 6, seed=9)
    one, tiny = np.ones(50), np.full(50, 1e-300)
    rH, rF = oracle.Oracle(H2).evaluate(x, one), oracle.Oracle(F).evaluate(x, one)
    assert np.max(np.abs(rH["H"] - rF["H"]) / rF["SH"]) < 1e-14
    assert np.max(np.abs(rH["Jx"] - rF["Jx"]) / np.maximum(rF["SJx"], 1e-300)) < 1e-14
    rG = oracle.Oracle(G.with_lifting(np.zeros(G.M))).evaluate(x, one)
    r0 = oracle.Oracle(H2).evaluate(x, tiny)
    assert np.max(np.abs(r0["H"] - rG["H"]) / rG["SH"]) < 1e-14
    # two terms per monomial only where the coefficients differ
    assert H2.M == G.M + int(np.count_nonzero(F.coeffs - G.coeffs))


def test_two_stage_oracle_solves_native_cyclic5():
    G, F, H2, x1, s1, x2, s2 = _two_stage_oracle(5)
    assert np.sum(s1 == 0) == 70 and np.sum(s2 == 0) == 70
    xs = x2[s2 == 0]
    r = oracle.Oracle(F).evaluate(xs, np.ones(len(xs)))
    assert np.max(np.abs(r["H"]) / r["SH"]) < 1e-12
    assert len({tuple(np.round(v, 7)) for v in xs}) == 70
    # the cyclic-5 solutions are invariant under the cyclic shift x_i -> x_{i+1}
    key = {tuple(np.round(v, 6)) for v in xs}
    assert all(tuple(np.round(np.roll(v, 1), 6)) in key for v in xs)
