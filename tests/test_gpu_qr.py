"""GPU parity of the QR direction solver (pht_system_set_solver(PHT_SOLVER_QR); the paper's
Householder mechanism P:708-726) against the oracle: its QR null-space route
(oracle.dirs_qr, QR of J^T) and its LU route, the worked example, singular flags, the step and
the tracker."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import workloads as W
from tests.parity import backward_err, rel_err, skeel_cond, step_parity
from workloads import startsys as SS

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    import paper_2111_14317_b200 as P
    return P


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


SYSTEMS = {
    "cyclic-5": lambda: W.cyclic(5),
    "cyclic-10": lambda: W.cyclic(10, lift_max=100),
    "katsura-10": lambda: W.katsura(10, lift_max=100),
    "noon-10": lambda: W.noon(10, lift_max=100),
    "chandra-6": lambda: W.chandra(6),
    "cyclic-14": lambda: W.cyclic(14),
    "random-20x50": lambda: W.random_dense(20, 50),
    "n1": lambda: W.from_terms("n1", 1, [[((2,), 1.0), ((0,), -3.0), ((-1,), 0.5)]]),
}


@pytest.mark.parametrize("name,p", [("cyclic-5", 512), ("cyclic-10", 200), ("katsura-10", 150),
                                    ("noon-10", 129), ("chandra-6", 100), ("cyclic-14", 40),
                                    ("random-20x50", 30), ("n1", 33)])
def test_qr_directions_match_oracle_qr_route(P, name, p):
    sysm = SYSTEMS[name]()
    o = oracle.Oracle(sysm)
    x, t, _ = W.random_points(p, sysm.n, seed=41, tau_lo=-0.05, rho_max=0.5 if sysm.n > 12 else 1.0)
    g = P.System.from_workload(sysm).set_solver("qr")
    dE, dN, st = g.euler_newton(_cuda(x), _cuda(t))
    dE, dN, st = dE.cpu().numpy(), dN.cpu().numpy(), st.cpu().numpy()
    r = o.evaluate(x, t)
    good = st == 0
    assert good.mean() >= 0.9
    # backward error against the oracle's Jacobian (QR is backward stable without pivoting)
    assert backward_err(r["Jx"][good], dE[good], -r["Jt"][good]).max() <= 1e-10
    assert backward_err(r["Jx"][good], dN[good], -r["H"][good]).max() <= 1e-10
    # forward agreement with the oracle's QR null-space route (QR of J^T)
    cond = skeel_cond(r["Jx"])
    for i in np.nonzero(good & (cond <= 1e4))[0][:64]:
        J = np.concatenate([r["Jx"][i], r["Jt"][i][:, None], r["H"][i][:, None]], axis=1)
        qE, qN, qs = oracle.dirs_qr(J)
        assert qs == 0
        assert rel_err(dE[i:i + 1], qE[None]).max() <= 1e-9
        assert rel_err(dN[i:i + 1], qN[None]).max() <= 1e-9


def test_qr_worked_example(P):
    gd = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cyclic3_worked_example.json")))
    eqs = [[(tuple(a), complex(*c), w) for a, c, w in eq] for eq in gd["equations"]]
    sysm = W.from_terms("g", 3, eqs, coeffs="native")
    cx = lambda v: complex(float(Fraction(v[0])), float(Fraction(v[1])))
    x = np.array([[cx(v) for v in gd["x"]]])
    g = P.System.from_workload(sysm).set_solver("qr")
    dE, dN, st = g.euler_newton(_cuda(x), _cuda(np.array([gd["t"]])))
    assert st.cpu().numpy()[0] == 0
    assert np.allclose(dE.cpu().numpy()[0], [cx(v) for v in gd["dE"]], atol=1e-14)
    assert np.allclose(dN.cpu().numpy()[0], [cx(v) for v in gd["dN"]], atol=1e-14)


def test_qr_singular_flag_and_isolation(P):
    sysm = W.from_terms("sing", 2, [[((1, 1), 1.0), ((0, 0), -1.0)], [((1, 1), 2.0), ((0, 0), -2.0)]],
                        coeffs="native")
    g = P.System.from_workload(sysm).set_solver("qr")
    x, t, _ = W.random_points(5, 2, seed=2)
    _, _, st = g.euler_newton(_cuda(x), _cuda(t))
    assert np.all(st.cpu().numpy() & P.PT_SINGULAR)
    # a regular system next to it on the same handle type is unaffected
    g2 = P.System.from_workload(W.cyclic(5)).set_solver("qr")
    x, t, _ = W.random_points(64, 5, seed=2, tau_lo=-0.05)
    _, _, st2 = g2.euler_newton(_cuda(x), _cuda(t))
    assert np.all(st2.cpu().numpy() == 0)
    with pytest.raises(P.PhtError):
        P._lib.check(P._lib.load().pht_system_set_solver(g2._h, 7), "pht_system_set_solver")


def test_qr_ill_conditioned_backward_stable(P):
    """tau down to -3 with liftings up to 100 flattens rows (Skeel cond up to ~1e12): the QR
    route stays backward stable on every point it does not flag."""
    sysm = W.cyclic(10, lift_max=100)
    x, t, _ = W.random_points(400, 10, seed=43, tau_lo=-3.0)
    g = P.System.from_workload(sysm).set_solver("qr")
    dE, dN, st = g.euler_newton(_cuda(x), _cuda(t))
    dE, dN, st = dE.cpu().numpy(), dN.cpu().numpy(), st.cpu().numpy()
    r = oracle.Oracle(sysm).evaluate(x, t)
    good = st == 0
    assert good.mean() >= 0.5
    assert skeel_cond(r["Jx"][good]).max() >= 1e6  # the sample does contain ill-conditioned points
    assert backward_err(r["Jx"][good], dE[good], -r["Jt"][good]).max() <= 1e-10
    assert backward_err(r["Jx"][good], dN[good], -r["H"][good]).max() <= 1e-10


@pytest.mark.parametrize("name,p,K", [("cyclic-5", 512, 1), ("cyclic-10", 200, 1), ("katsura-10", 120, 2)])
def test_qr_pc_step_parity(P, name, p, K):
    sysm = SYSTEMS[name]()
    o = oracle.Oracle(sysm)
    x, _, tau = W.random_points(p, sysm.n, seed=12, tau_lo=-0.05)
    dtau = np.full(p, 0.01)
    g = P.System.from_workload(sysm).set_solver("qr")
    xg, taug = _cuda(x), _cuda(tau)
    st, _ = g.pc_step(xg, taug, _cuda(dtau), newton_iters=K)
    same, tau_eq, ratio = step_parity(o, x, tau, dtau, K, xg.cpu().numpy(), st.cpu().numpy(), taug.cpu().numpy())
    assert same and tau_eq and ratio <= 1.0, (same, tau_eq, ratio)


@pytest.mark.parametrize("spec", [False, True])
def test_qr_track_cells_cyclic5(P, spec):
    s = W.cyclic(5, lift_max=100)
    cells = SS.mixed_cells_fast(s)
    Wc = SS.cell_lifts(s, cells)
    w0, tau0, cid = SS.start_points_cells(s, cells)
    g = P.System.from_workload(s).set_solver("qr")
    if spec:
        g.specialize().set_kernels("specialized")  # also the tracker on small batches
    wd, td = _cuda(w0), _cuda(tau0)
    st, _ = g.track_cells(wd, td, _cuda(Wc), _cuda(cid))
    sg = st.cpu().numpy()
    m, e = oracle.z_to_x(w0)
    xm, xe, _, so, _ = oracle.Oracle(s).track_x(m, e, tau0, cell_lift=Wc, path_cell=cid)
    xo, xg = xm * np.exp2(xe.astype(float)), np.exp(wd.cpu().numpy())
    assert np.sum(sg == 0) == np.sum(so == 0) == 70
    rel = np.linalg.norm(xg - xo, axis=1) / np.linalg.norm(xo, axis=1)
    assert rel.max() <= 1e-8, rel.max()
