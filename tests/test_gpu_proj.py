"""GPU parity of the projective formulation (pht_system_create_projective, SURVEY
§8(f) f1) against the oracle's projective functions (tests/test_oracle_proj.py pins them):
evaluation of the bordered matrix, the projective Euler/Newton directions, the step with
renormalisation, and tracking including a solution at infinity."""
import numpy as np
import pytest

import oracle
import workloads as W
from tests.parity import backward_err, eval_err, rel_err, skeel_cond
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


SYSTEMS = {
    "cyclic-5": lambda: W.cyclic(5, lift_max=20),
    "cyclic-10": lambda: W.cyclic(10, lift_max=100),
    "katsura-10": lambda: W.katsura(10, lift_max=100),
    "noon-10": lambda: W.noon(10, lift_max=100),
    "chandra-6": lambda: W.chandra(6, lift_max=20),
}


def _sphere_points(p, m, seed):
    z, _ = W.random_log_points(p, m, seed=seed, rho_max=0.5)
    y = np.exp(z)
    return y / np.linalg.norm(y, axis=1, keepdims=True)


@pytest.mark.parametrize("name,p", [("cyclic-5", 300), ("cyclic-10", 200), ("katsura-10", 150), ("chandra-6", 100)])
@pytest.mark.parametrize("spec", [False, True])
def test_proj_evaluate_parity(P, name, p, spec):
    sysm = SYSTEMS[name]()
    n = sysm.n
    y = _sphere_points(p, n + 1, seed=51)
    _, t, _ = W.random_points(p, 1, seed=52, tau_lo=-1.0)
    r = oracle.Oracle(sysm).proj_evaluate(y, t)
    g = P.System.from_workload(sysm, projective=True)
    if spec:
        g.specialize()
    assert g.projective and g.n == n + 1
    H, J, Jt, st = g.evaluate(_cuda(y), _cuda(t))
    H, J, Jt, st = H.cpu().numpy(), J.cpu().numpy(), Jt.cpu().numpy(), st.cpu().numpy()
    assert np.all(st == 0)
    assert eval_err(H[:, :n], r["H"], r["SH"]) <= 1e-10
    assert eval_err(J[:, :n, :], r["Jy"], r["SJy"]) <= 1e-10
    assert eval_err(Jt[:, :n], r["Jt"], r["SJt"]) <= 1e-10
    # the bordering row y^* and its zero right-hand sides
    assert np.max(np.abs(J[:, n, :] - np.conj(y))) <= 1e-15
    assert np.all(H[:, n] == 0) and np.all(Jt[:, n] == 0)


@pytest.mark.parametrize("name,p", [("cyclic-5", 300), ("cyclic-10", 200), ("noon-10", 150)])
@pytest.mark.parametrize("solver", ["lu", "qr"])
def test_proj_directions_parity(P, name, p, solver):
    sysm = SYSTEMS[name]()
    n = sysm.n
    y = _sphere_points(p, n + 1, seed=53)
    _, t, _ = W.random_points(p, 1, seed=54, tau_lo=-0.05)
    o = oracle.Oracle(sysm)
    g = P.System.from_workload(sysm, projective=True).set_solver(solver)
    dE, dN, st = g.euler_newton(_cuda(y), _cuda(t))
    dE, dN, st = dE.cpu().numpy(), dN.cpu().numpy(), st.cpu().numpy()
    E, N, so = o.proj_euler_newton(y, t)
    r = o.proj_evaluate(y, t)
    # bordered matrix and right-hand sides from the oracle's evaluation
    A = np.concatenate([r["Jy"], np.conj(y)[:, None, :]], axis=1)
    bE = np.concatenate([-(t[:, None] * r["Jt"]), np.zeros((p, 1))], axis=1)
    bN = np.concatenate([-r["H"], np.zeros((p, 1))], axis=1)
    good = (st == 0) & (so == 0)
    assert good.mean() >= 0.9
    # pht_euler_newton returns dE = dx/dt: the projective Euler direction is dy/dtau = t dy/dt
    dEt = dE * t[:, None]
    assert backward_err(A[good], dEt[good], bE[good]).max() <= 1e-10
    assert backward_err(A[good], dN[good], bN[good]).max() <= 1e-10
    cond = skeel_cond(A)  # row-scaling invariant (degree-10 rows are ~1e-5 of the y^* row)
    well = good & (cond <= 1e4)
    assert well.sum() >= 0.5 * p
    assert rel_err(dEt[well], E[well]).max() <= 1e-9
    assert rel_err(dN[well], N[well]).max() <= 1e-9


@pytest.mark.parametrize("name,p,K", [("cyclic-5", 300, 1), ("cyclic-10", 200, 2)])
def test_proj_pc_step_parity(P, name, p, K):
    sysm = SYSTEMS[name]()
    n = sysm.n
    y = _sphere_points(p, n + 1, seed=55)
    _, _, tau = W.random_points(p, 1, seed=56, tau_lo=-0.05)
    dtau = np.full(p, 0.01)
    yo, tauo, so, dno = oracle.Oracle(sysm).proj_pc_step(y, tau, dtau, K=K)
    g = P.System.from_workload(sysm, projective=True)
    yg, tg = _cuda(y), _cuda(tau)
    st, dn = g.pc_step(yg, tg, _cuda(dtau), newton_iters=K)
    yg, st = yg.cpu().numpy(), st.cpu().numpy()
    assert np.allclose(np.linalg.norm(yg, axis=1), 1.0, atol=1e-14)
    r = oracle.Oracle(sysm).proj_evaluate(y, np.exp(tau))
    A = np.concatenate([r["Jy"], np.conj(y)[:, None, :]], axis=1)
    well = (st == 0) & (so == 0) & (skeel_cond(A) <= 1e3)
    assert well.sum() >= 0.4 * p
    assert rel_err(yg[well], yo[well]).max() <= 1e-9


def _stage1_oracle(G):
    cells = SS.mixed_cells_fast(G)
    Wc = SS.cell_lifts(G, cells)
    w0, tau0, cid = SS.start_points_cells(G, cells)
    m, e = oracle.z_to_x(w0)
    xm, xe, _, s1, _ = oracle.Oracle(G).track_x(m, e, tau0, cell_lift=Wc, path_cell=cid)
    assert np.all(s1 == 0)
    x1 = xm * np.exp2(xe.astype(float))
    y1 = np.concatenate([x1, np.ones((len(x1), 1))], axis=1)
    return y1 / np.linalg.norm(y1, axis=1, keepdims=True)


@pytest.mark.parametrize("spec", [False, True])
def test_proj_track_solution_at_infinity(P, spec):
    """Second stage to F = {x1 + x2 - 1, x1^2 + x1 x2 + x1 + x2 - 3}: one finite solution (2, -1),
    one at the point at infinity (1 : -1 : 0); same statuses and endpoints as the oracle."""
    eqs = [[((1, 0), 1.0), ((0, 1), 1.0), ((0, 0), -1.0)],
           [((2, 0), 1.0), ((1, 1), 1.0), ((1, 0), 1.0), ((0, 1), 1.0), ((0, 0), -3.0)]]
    F = W.from_terms("inf2", 2, eqs, coeffs="native", lift_max=100)
    G = W.from_terms("inf2", 2, eqs, coeffs="random", lift_max=100)
    H2 = PH.parameter_homotopy(G, F.coeffs)
    y1 = _stage1_oracle(G)
    yo, _, so, _ = oracle.Oracle(H2).proj_track(y1, np.full(2, PH.TAU0))
    g = P.System.from_workload(H2, projective=True)
    if spec:
        g.specialize().set_kernels("specialized")  # also the tracker on 2 paths
    yd, td = _cuda(y1), _cuda(np.full(2, PH.TAU0))
    st, _ = g.track(yd, td)
    yg, sg = yd.cpu().numpy(), st.cpu().numpy()
    assert np.array_equal(sg, so)
    assert sorted(sg.tolist()) == [0, P.PT_DIVERGED]
    fin = sg == 0
    assert np.allclose(yg[fin, :2] / yg[fin, 2:], [[2.0, -1.0]], atol=1e-12)
    yi = yg[~fin][0] / yg[~fin][0][0]
    assert np.allclose(yi, [1.0, -1.0, 0.0], atol=1e-10)
    # endpoints agree up to the phase of the projective point
    for i in range(2):
        ph = np.vdot(yo[i], yg[i]) / abs(np.vdot(yo[i], yg[i]))
        assert np.linalg.norm(yg[i] - ph * yo[i]) <= 1e-8


def test_proj_two_stage_cyclic5(P):
    """Native cyclic-5 in homogeneous coordinates: 70 finite solutions, as the oracle."""
    G = W.cyclic(5, lift_max=100)
    F = W.cyclic(5, lift_max=100, coeffs="native")
    H2 = PH.parameter_homotopy(G, F.coeffs)
    y1 = _stage1_oracle(G)
    yo, _, so, _ = oracle.Oracle(H2).proj_track(y1, np.full(len(y1), PH.TAU0))
    g = P.System.from_workload(H2, projective=True)
    yd, td = _cuda(y1), _cuda(np.full(len(y1), PH.TAU0))
    st, _ = g.track(yd, td)
    yg, sg = yd.cpu().numpy(), st.cpu().numpy()
    assert np.sum(sg == 0) == np.sum(so == 0) == 70
    xg, xo = yg[:, :5] / yg[:, 5:], yo[:, :5] / yo[:, 5:]
    assert np.max(np.linalg.norm(xg - xo, axis=1) / np.linalg.norm(xo, axis=1)) <= 1e-8
    with pytest.raises(P.PhtError):
        g.track(_cuda(y1), _cuda(np.full(len(y1), PH.TAU0)), log_state=1)


def test_homogenize_points(P):
    sysm = W.cyclic(5, lift_max=20)
    g = P.System.from_workload(sysm, projective=True)
    z, _ = W.random_log_points(100, 5, seed=61, rho_max=8.0)
    y1 = g.homogenize(_cuda(z), log_input=True).cpu().numpy()
    y2 = g.homogenize(_cuda(np.exp(z)), log_input=False).cpu().numpy()
    assert np.allclose(np.linalg.norm(y1, axis=1), 1.0, atol=1e-15)
    x = np.exp(z)
    assert np.max(np.abs(y1[:, :5] / y1[:, 5:] - x) / np.abs(x)) < 1e-13
    assert np.max(np.abs(y1 - y2)) < 1e-14
