"""Parity at BASELINE.json's full sizes in the launch configurations bench.py times (task rule:
full-size runs compared on outputs the oracle can compute one by one): the cyclic-10 step on
2^22 points (bench.py value), the cyclic-10 evaluation on 2^21 points and the random dense n=20
DMMA evaluation on 2^18 points (bench.py evaluation section).  A seeded sample of 256 points
of each launch is recomputed by the oracle."""
import numpy as np
import pytest

import bench
import oracle
import workloads as W
from tests.parity import eval_err, rel_err, skeel_cond

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    import paper_2111_14317_b200 as P
    return P


def _sample(p, k=256, seed=0):
    return np.sort(np.random.default_rng(seed).choice(p, k, replace=False))


def test_step_full_size_sampled(P):
    sysm = bench._system()
    Pn = 1 << 22
    x, _, tau = W.random_points(Pn, bench.N_VARS, seed=1000, tau_lo=bench.TAU_LO)   # bench.py rank 0
    g = P.System.from_workload(sysm)
    xd, td = torch.from_numpy(x).cuda(), torch.from_numpy(tau).cuda()
    dt = torch.full((Pn,), bench.DTAU, dtype=torch.float64, device="cuda")
    st, dn = g.pc_step(xd, td, dt, 1)
    pick = _sample(Pn, seed=1)
    xg, tg, sg = xd[pick].cpu().numpy(), td[pick].cpu().numpy(), st[pick].cpu().numpy()
    o = oracle.Oracle(sysm)
    xo, to, so, _ = o.pc_step(x[pick], tau[pick], np.full(len(pick), bench.DTAU), K=1)
    assert np.array_equal(tg, to)
    cond = skeel_cond(o.evaluate(x[pick], np.exp(tau[pick]))["Jx"])
    well = (sg == 0) & (so == 0) & (cond <= 1e3)
    assert well.sum() >= 0.9 * len(pick)
    assert rel_err(xg[well], xo[well]).max() <= 1e-9
    assert np.array_equal(sg == 0, so == 0)


@pytest.mark.parametrize("name,Pn", [("cyclic-10", 1 << 21), ("random-20x50", 1 << 18)])
def test_evaluation_full_size_sampled(P, name, Pn):
    sysm = W.cyclic(10, lift_max=bench.LIFT_MAX) if name == "cyclic-10" else W.random_dense(20, 50)
    x, t, _ = W.random_points(Pn, sysm.n, seed=2000, rho_max=0.5 if sysm.n > 12 else 1.0)  # bench.py rank 0
    g = P.System.from_workload(sysm)
    H, J, Jt, st = g.evaluate(torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda())
    pick = _sample(Pn, seed=2)
    r = oracle.Oracle(sysm).evaluate(x[pick], t[pick])
    assert np.all(st[pick].cpu().numpy() == 0)
    assert eval_err(H[pick].cpu().numpy(), r["H"], r["SH"]) <= 1e-10
    assert eval_err(J[pick].cpu().numpy(), r["Jx"], r["SJx"]) <= 1e-10
    assert eval_err(Jt[pick].cpu().numpy(), r["Jt"], r["SJt"]) <= 1e-10
    # the rest of the launch: every status clean and every output finite (property at any size)
    assert bool((st == 0).all()) and bool(torch.isfinite(torch.view_as_real(J)).all())


@pytest.mark.parametrize("name,L", [("noon-10", 10_000), ("cyclic-10", 1_000_000)])
def test_tracking_full_launch_sampled(P, name, L):
    """All start paths tracked in one launch (the bench.py tracking configuration); 128 seeded
    paths re-tracked by the oracle: identical statuses, endpoints <= 1e-8."""
    from workloads import startsys as SS
    from workloads.make_starts import CONFIGS
    s = CONFIGS[name](L)
    cells = SS.load_cells(name, L)
    Wc = SS.cell_lifts_fast(s, cells)
    w0, tau0, cid = SS.start_points_cells(s, cells)
    g = P.System.from_workload(s)
    wd, td = torch.from_numpy(w0.copy()).cuda(), torch.from_numpy(tau0.copy()).cuda()
    st, _ = g.track_cells(wd, td, torch.from_numpy(Wc).cuda(), torch.from_numpy(cid).cuda())
    assert int((st == 0).sum()) == len(w0)          # every path finite (the mixed volume)
    pick = _sample(len(w0), 128, seed=4)
    m, e = oracle.z_to_x(w0[pick])
    xm, xe, _, so, _ = oracle.Oracle(s).track_x(m, e, tau0[pick], cell_lift=Wc, path_cell=cid[pick])
    sg = st[pick].cpu().numpy()
    assert np.array_equal(sg, so)
    xg = np.exp(wd[pick].cpu().numpy())
    xo = xm * np.exp2(xe.astype(float))
    rel = np.linalg.norm(xg - xo, axis=1) / np.linalg.norm(xo, axis=1)
    assert rel.max() <= 1e-8, rel.max()
