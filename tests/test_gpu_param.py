"""Two-stage solve on the GPU (polyhedral stage 1 with pht_track_cells, then the coefficient-
parameter homotopy (1 - t) G + t F with pht_track in log state) against the
oracle's two-stage solve from the same workload inputs: identical finite counts (the known
solution counts of native cyclic-5 / cyclic-7: 70 / 924), endpoints <= 1e-8."""
import numpy as np
import pytest

import oracle
import workloads as W
from workloads import param as PH
from workloads import startsys as SS

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    import paper_2111_14317_b200 as P
    return P


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("n,L,count", [(5, 100, 70), (7, 10 ** 4, 924)])
def test_two_stage_native_cyclic(P, n, L, count):
    G = W.cyclic(n, lift_max=L)
    F = W.cyclic(n, lift_max=L, coeffs="native")
    H2 = PH.parameter_homotopy(G, F.coeffs)
    cells = SS.mixed_cells_fast(G)
    Wc = SS.cell_lifts_fast(G, cells)
    w0, tau0, cid = SS.start_points_cells(G, cells)
    # GPU: stage 1 in cell coordinates, stage 2 in log state from the stage-1 endpoints (z = log x)
    g1, g2 = P.System.from_workload(G), P.System.from_workload(H2)
    wd, td = _cuda(w0), _cuda(tau0)
    s1, _ = g1.track_cells(wd, td, _cuda(Wc), _cuda(cid))
    ok = s1 == 0
    z = wd[ok].contiguous()
    t2 = torch.full((z.shape[0],), PH.TAU0, dtype=torch.float64, device="cuda")
    s2, _ = g2.track(z, t2, log_state=1)
    zg, sg = z.cpu().numpy(), s2.cpu().numpy()
    # oracle: the same two stages (extended-range state, same predictor chart)
    m, e = oracle.z_to_x(w0)
    xm, xe, _, so1, _ = oracle.Oracle(G).track_x(m, e, tau0, cell_lift=Wc, path_cell=cid)
    assert np.array_equal(so1 == 0, ok.cpu().numpy())
    k = so1 == 0
    xm2, xe2, _, so2, _ = oracle.Oracle(H2).track_x(xm[k], xe[k], np.full(k.sum(), PH.TAU0))
    assert np.sum(sg == 0) == np.sum(so2 == 0) == count
    both = (sg == 0) & (so2 == 0)
    xo = xm2[both] * np.exp2(xe2[both].astype(float))
    xg = np.exp(zg[both])
    rel = np.linalg.norm(xg - xo, axis=1) / np.linalg.norm(xo, axis=1)
    assert rel.max() <= 1e-8, rel.max()
    # property: the endpoints solve the native system and are distinct
    r = oracle.Oracle(F).evaluate(xg, np.ones(len(xg)))
    assert np.max(np.abs(r["H"]) / r["SH"]) < 1e-10
    assert len({tuple(np.round(v, 7)) for v in xg}) == count
