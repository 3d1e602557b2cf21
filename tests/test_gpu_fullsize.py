"""Parity at BASELINE.json's full sizes in the launch configurations bench.py times (task rule:
full-size runs compared on outputs the oracle can compute one by one): the cyclic-10 step on
2^22 points (bench.py value), the cyclic-10 evaluation on 2^21 points and the random dense n=20
DMMA evaluation on 2^20 points (bench.py evaluation section).  A seeded sample of 256-1024
points of each launch is recomputed by the oracle."""
import numpy as np
import pytest

import bench
import oracle
import workloads as W
from tests.parity import eval_err, step_parity

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
    pick = _sample(Pn, k=1024, seed=1)
    xg, tg, sg = xd[pick].cpu().numpy(), td[pick].cpu().numpy(), st[pick].cpu().numpy()
    o = oracle.Oracle(sysm)
    same, tau_eq, ratio = step_parity(o, x[pick], tau[pick], np.full(len(pick), bench.DTAU), 1, xg, sg, tg)
    assert same and tau_eq and ratio <= 1.0, (same, tau_eq, ratio)
    assert (sg == 0).sum() >= 0.9 * len(pick)
    # the rest of the launch: tau advanced by exactly dtau everywhere, every output finite
    assert torch.equal(td, torch.from_numpy(tau + bench.DTAU).cuda())
    assert bool(torch.isfinite(torch.view_as_real(xd)).all())


@pytest.mark.parametrize("name,Pn", [("cyclic-10", 1 << 21), ("random-20x50", 1 << 20)])
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


# All-path tracking at full size against the oracle: tests/test_gpu_track_golden.py (every path).
