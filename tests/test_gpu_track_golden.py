"""Every start path of katsura-10 (990), cyclic-10 (35,940) and noon-10 (59,029) tracked on the
GPU in one launch (the bench.py tracking configuration) against the CPU oracle's tracking of the
same paths (tests/golden/track_<name>.npz, written by tools/make_track_golden.py, which calls only
oracle/).  BASELINE.json north_star: identical finite counts and endpoints <= 1e-8.

The oracle's finite rule is ledger A24 (refined to final_tol = 1e-13).  The device refines with a
compensated stage 2 (reading R30) and reaches final_tol on exactly the oracle's finite
paths: the statuses are identical.  (PHT_PT_FLOOR -- finite, refined only to newton_tol -- remains
possible where no compensated evaluation exists, the specialised trackers; it would count as
finite.)"""
import os

import numpy as np
import pytest

from workloads import startsys as SS
from workloads.make_starts import CONFIGS

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
LIFT = {"katsura-10": 10_000, "noon-10": 10_000, "cyclic-10": 1_000_000}


@pytest.fixture(scope="module")
def P():
    import paper_2111_14317_b200 as P
    return P


@pytest.mark.parametrize("name", ["katsura-10", "cyclic-10", "noon-10"])
def test_all_paths_against_oracle(P, name):
    gold = np.load(os.path.join(GOLDEN, f"track_{name}.npz"))
    L = LIFT[name]
    s = CONFIGS[name](L)
    cells = SS.load_cells(name, L)
    Wc = SS.cell_lifts_fast(s, cells)
    w0, tau0, cid = SS.start_points_cells(s, cells)
    assert len(w0) == len(gold["status"])
    g = P.System.from_workload(s)
    wd, td = torch.from_numpy(w0.copy()).cuda(), torch.from_numpy(tau0.copy()).cuda()
    st, stats = g.track_cells(wd, td, torch.from_numpy(Wc).cuda(), torch.from_numpy(cid).cuda())
    sg = st.cpu().numpy()
    so = gold["status"]
    fin_g = (sg == P.PT_OK) | (sg == P.PT_FLOOR)
    fin_o = so == 0
    n_floor = int((sg == P.PT_FLOOR).sum())
    print(f"{name}: oracle finite {fin_o.sum()}, GPU OK {(sg == 0).sum()} + FLOOR {n_floor}")
    assert fin_g.sum() == fin_o.sum()            # identical finite counts
    assert np.array_equal(fin_g, fin_o)          # ... on the same paths
    assert np.array_equal(sg, so)                # identical statuses (no FLOOR: compensated refinement)
    xo = gold["xm"] * np.exp2(gold["xe"].astype(float))
    xg = np.exp(wd.cpu().numpy())
    rel = np.linalg.norm(xg[fin_o] - xo[fin_o], axis=1) / np.linalg.norm(xo[fin_o], axis=1)
    assert rel.max() <= 1e-8, (rel.max(), int(np.argmax(rel)))
    # work statistics agree as statistics (ledger A23: decisions may flip at rounding level)
    ev_g, ev_o = int(stats[:, 2].sum()), int(gold["stats"][:, 2].sum())
    assert abs(ev_g - ev_o) <= 0.02 * ev_o, (ev_g, ev_o)
