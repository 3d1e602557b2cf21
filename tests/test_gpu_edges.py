"""Edge cases of the CUDA path against the oracle: the largest n with a compiled kernel
(PHT_MAX_N = 24) on every entry point, Laurent (negative-exponent) systems through the step,
projective systems on the QR solver and the specialised kernels, and empty batches everywhere."""
import numpy as np
import pytest

import oracle
import workloads as W
from tests.parity import eval_err, rel_err, skeel_cond, step_parity
from tests.test_gpu_parity import _dirs_check

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    import paper_2111_14317_b200 as P
    return P


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_max_n_24_all_entry_points(P):
    sysm = W.random_dense(24, 6, emax=1, lift_max=5)
    o = oracle.Oracle(sysm)
    x, t, tau = W.random_points(70, 24, seed=71, rho_max=0.3, tau_lo=-0.05)
    g = P.System.from_workload(sysm)
    H, J, Jt, st = g.evaluate(_cuda(x), _cuda(t))
    r = o.evaluate(x, t)
    assert np.all(st.cpu().numpy() == 0)
    assert eval_err(H.cpu().numpy(), r["H"], r["SH"]) <= 1e-10
    assert eval_err(J.cpu().numpy(), r["Jx"], r["SJx"]) <= 1e-10
    dE, dN, st = g.euler_newton(_cuda(x), _cuda(t))
    _dirs_check(o, x, t, dE.cpu().numpy(), dN.cpu().numpy(), st.cpu().numpy())
    for solver in ("lu", "qr"):
        g.set_solver(solver)
        xg, tg = _cuda(x), _cuda(tau)
        sg, _ = g.pc_step(xg, tg, _cuda(np.full(70, 0.01)), 1)
        same, tau_eq, ratio = step_parity(o, x, tau, np.full(70, 0.01), 1, xg.cpu().numpy(), sg.cpu().numpy(),
                                          tg.cpu().numpy())
        assert same and tau_eq and ratio <= 1.0, (solver, same, tau_eq, ratio)


def test_laurent_system_step(P):
    """Negative exponents (Laurent monomials) through the Euler-Newton step."""
    sysm = W.random_dense(6, 9, emax=2, lift_max=20)
    assert (sysm.exps < 0).any()
    o = oracle.Oracle(sysm)
    x, _, tau = W.random_points(300, 6, seed=72, tau_lo=-0.05)
    g = P.System.from_workload(sysm)
    xg, tg = _cuda(x), _cuda(tau)
    sg, _ = g.pc_step(xg, tg, _cuda(np.full(300, 0.01)), 2)
    same, tau_eq, ratio = step_parity(o, x, tau, np.full(300, 0.01), 2, xg.cpu().numpy(), sg.cpu().numpy(),
                                      tg.cpu().numpy())
    assert same and tau_eq and ratio <= 1.0, (same, tau_eq, ratio)


def test_empty_batches_every_entry_point(P):
    g = P.System.from_workload(W.cyclic(5))
    e = torch.empty((0, 5), dtype=torch.complex128, device="cuda")
    f = torch.empty(0, dtype=torch.float64, device="cuda")
    g.evaluate(e, f)
    g.evaluate_log(e, f)
    g.euler_newton(e, f)
    g.pc_step(e, f, f, 1)
    st, _ = g.track(e, f)
    assert st.numel() == 0
    g.specialize(P._lib.SPEC_EVAL)
    g.evaluate(e, f)
    gp = P.System.from_workload(W.cyclic(5), projective=True)
    gp.homogenize(e, log_input=True)
    torch.cuda.synchronize()


def test_projective_specialised_qr_step(P):
    """Projective system on the specialised kernels with the QR solver: the step agrees with the
    oracle's projective step."""
    sysm = W.cyclic(5, lift_max=20)
    z, _ = W.random_log_points(200, 6, seed=73, rho_max=0.5)
    y = np.exp(z)
    y /= np.linalg.norm(y, axis=1, keepdims=True)
    _, _, tau = W.random_points(200, 1, seed=74, tau_lo=-0.05)
    yo, _, so, _ = oracle.Oracle(sysm).proj_pc_step(y, tau, np.full(200, 0.01), K=1)
    g = P.System.from_workload(sysm, projective=True).set_solver("qr").specialize()
    yg, tg = _cuda(y), _cuda(tau)
    sg, _ = g.pc_step(yg, tg, _cuda(np.full(200, 0.01)), 1)
    r = oracle.Oracle(sysm).proj_evaluate(y, np.exp(tau))
    A = np.concatenate([r["Jy"], np.conj(y)[:, None, :]], axis=1)
    well = (sg.cpu().numpy() == 0) & (so == 0) & (skeel_cond(A) <= 1e3)
    assert well.sum() >= 80
    assert rel_err(yg.cpu().numpy()[well], yo[well]).max() <= 1e-9
