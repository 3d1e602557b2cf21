"""Pin for the oracle's Hermite predictor (orc_track_x predictor = 1): it is only a
different predictor, so the tracked endpoints are the same solutions as with the Euler predictor
(to rounding) and every start path of cyclic-5 / katsura-6 converges."""
import numpy as np

import oracle
import workloads as W
from workloads import startsys as SS


def test_hermite_predictor_same_endpoints_as_euler():
    for s, count in ((W.cyclic(5, lift_max=100), 70), (W.katsura(6, lift_max=10 ** 4), 54)):
        cells = SS.mixed_cells_fast(s)
        Wc = SS.cell_lifts(s, cells)
        w0, tau0, cid = SS.start_points_cells(s, cells)
        m, e = oracle.z_to_x(w0)
        o = oracle.Oracle(s)
        xa, ea, _, sa, _ = o.track_x(m, e, tau0, cell_lift=Wc, path_cell=cid, predictor=0)
        xb, eb, _, sb, stb = o.track_x(m, e, tau0, cell_lift=Wc, path_cell=cid, predictor=1)
        assert np.sum(sb == 0) == count
        ok = (sa == 0) & (sb == 0)
        A, B = xa * np.exp2(ea.astype(float)), xb * np.exp2(eb.astype(float))
        assert np.max(np.linalg.norm(A[ok] - B[ok], axis=1) / np.linalg.norm(A[ok], axis=1)) < 1e-10
        r = o.evaluate(B, np.ones(len(B)))
        assert np.max(np.abs(r["H"]) / r["SH"]) < 1e-12
