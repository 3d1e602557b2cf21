"""GPU parity of the system-specialised kernels (pht_system_specialize: rows generated as
straight-line code and compiled with NVRTC) against the oracle, with the same bars as the
generic kernels (tests/test_gpu_parity.py, tests/test_gpu_track.py)."""
import numpy as np
import pytest

import oracle
import workloads as W
from tests.parity import eval_err, rel_err, step_parity
from tests.test_gpu_parity import _dirs_check
from workloads import startsys as SS

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    import paper_2111_14317_b200 as P
    return P


# The specialised tracker normally needs a full wave of paths and the warp-per-group step is the
# default from n = 10: every handle here selects the specialised kernels explicitly
# (pht_system_set_kernels(PHT_KERNELS_SPECIALIZED)).


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


SYSTEMS = {
    "cyclic-5": lambda: W.cyclic(5),
    "cyclic-10": lambda: W.cyclic(10, lift_max=100),
    "katsura-10": lambda: W.katsura(10, lift_max=100),
    "noon-10": lambda: W.noon(10, lift_max=100),
    "chandra-6": lambda: W.chandra(6),
    "random-6x9": lambda: W.random_dense(6, 9),
    "n1": lambda: W.from_terms("n1", 1, [[((2,), 1.0), ((0,), -3.0), ((-1,), 0.5)]]),
}


def _spec(P, sysm):
    g = P.System.from_workload(sysm).specialize().set_kernels("specialized")
    assert g.specialized
    return g


@pytest.mark.parametrize("name,p", [("cyclic-5", 1024), ("cyclic-10", 333), ("katsura-10", 200),
                                    ("noon-10", 257), ("chandra-6", 100), ("random-6x9", 77), ("n1", 65)])
def test_specialized_evaluate_parity(P, name, p):
    sysm = SYSTEMS[name]()
    x, t, _ = W.random_points(p, sysm.n, seed=3)
    r = oracle.Oracle(sysm).evaluate(x, t)
    g = _spec(P, sysm)
    H, Jx, Jt, st = g.evaluate(_cuda(x), _cuda(t))
    assert np.all(st.cpu().numpy() == 0)
    assert eval_err(H.cpu().numpy(), r["H"], r["SH"]) <= 1e-10
    assert eval_err(Jx.cpu().numpy(), r["Jx"], r["SJx"]) <= 1e-10
    assert eval_err(Jt.cpu().numpy(), r["Jt"], r["SJt"]) <= 1e-10
    # scaled rows: row * 2^row_exp2 is the unscaled row
    Hs, Jxs, Jts, e2, _ = g.evaluate(_cuda(x), _cuda(t), scaled=True)
    sc = np.exp2(e2.cpu().numpy().astype(float))
    assert np.allclose(Hs.cpu().numpy() * sc, H.cpu().numpy(), rtol=1e-15, atol=0)


def test_specialized_log_variant_and_large_liftings(P):
    """evaluate_log with liftings up to 1e4 and tau down to -3 (rows spanning e^3e4) against the
    extended-range oracle: the row exponent is taken from the largest term."""
    sysm = W.noon(10, lift_max=10 ** 4)
    z, tau = W.random_log_points(200, 10, seed=21, tau_lo=-3.0)
    g = _spec(P, sysm)
    H, Jz, Jtau, e2, st = g.evaluate_log(_cuda(z), _cuda(tau))
    ref = P.System.from_workload(sysm)
    H0, Jz0, Jtau0, e20, st0 = ref.evaluate_log(_cuda(z), _cuda(tau))
    # same rows as the generic kernel up to rounding, once both are brought to a common exponent
    d = (e2 - e20).cpu().numpy().astype(float)
    a = H.cpu().numpy() * np.exp2(d)
    b = H0.cpu().numpy()
    scale = np.abs(Jz0.cpu().numpy()).max(axis=2) + np.abs(b)
    assert np.all(np.abs(a - b) <= 1e-10 * scale + 1e-300)
    assert np.array_equal(st.cpu().numpy(), st0.cpu().numpy())


@pytest.mark.parametrize("name,p", [("cyclic-5", 1024), ("cyclic-10", 333), ("katsura-10", 200), ("noon-10", 129)])
def test_specialized_euler_newton_parity(P, name, p):
    sysm = SYSTEMS[name]()
    o = oracle.Oracle(sysm)
    x, t, _ = W.random_points(p, sysm.n, seed=4, tau_lo=-0.05)
    g = _spec(P, sysm)
    dE, dN, st = g.euler_newton(_cuda(x), _cuda(t))
    _dirs_check(o, x, t, dE.cpu().numpy(), dN.cpu().numpy(), st.cpu().numpy())


@pytest.mark.parametrize("name,p,K", [("cyclic-5", 1024, 1), ("cyclic-10", 300, 1), ("katsura-10", 150, 2)])
def test_specialized_pc_step_parity(P, name, p, K):
    sysm = SYSTEMS[name]()
    o = oracle.Oracle(sysm)
    x, _, tau = W.random_points(p, sysm.n, seed=12, tau_lo=-0.05)
    dtau = np.full(p, 0.01)
    g = _spec(P, sysm)
    xg, taug = _cuda(x), _cuda(tau)
    st, dn = g.pc_step(xg, taug, _cuda(dtau), newton_iters=K)
    same, tau_eq, ratio = step_parity(o, x, tau, dtau, K, xg.cpu().numpy(), st.cpu().numpy(), taug.cpu().numpy())
    assert same and tau_eq and ratio <= 1.0, (same, tau_eq, ratio)


def test_specialized_matches_generic_step(P):
    """Specialised and generic kernels agree to rounding on 2^14 cyclic-10 points (statuses equal)."""
    sysm = SYSTEMS["cyclic-10"]()
    x, _, tau = W.random_points(1 << 14, 10, seed=31, tau_lo=-0.05)
    dtau = np.full(len(x), 1e-3)
    res = []
    for spec in (False, True):
        g = P.System.from_workload(sysm)
        if spec:
            g.specialize().set_kernels("specialized")
        xg, tg = _cuda(x), _cuda(tau)
        st, _ = g.pc_step(xg, tg, _cuda(dtau), 1)
        res.append((xg.cpu().numpy(), st.cpu().numpy()))
    assert np.array_equal(res[0][1], res[1][1])
    ok = res[0][1] == 0
    assert rel_err(res[1][0][ok], res[0][0][ok]).max() <= 1e-9


@pytest.mark.parametrize("name", ["cyclic-5", "noon-5"])
def test_specialized_track_cells_parity(P, name):
    s = {"cyclic-5": W.cyclic(5, lift_max=100), "noon-5": W.noon(5, lift_max=1000)}[name]
    cells = SS.mixed_cells_fast(s)
    Wc = SS.cell_lifts(s, cells)
    w0, tau0, cid = SS.start_points_cells(s, cells)
    g = _spec(P, s)
    wd, td = _cuda(w0), _cuda(tau0)
    st, _ = g.track_cells(wd, td, _cuda(Wc), _cuda(cid))
    zg, sg = wd.cpu().numpy(), st.cpu().numpy()
    m, e = oracle.z_to_x(w0)
    xm, xe, _, so, _ = oracle.Oracle(s).track_x(m, e, tau0, cell_lift=Wc, path_cell=cid)
    xo, xg = xm * np.exp2(xe.astype(float)), np.exp(zg)
    assert np.sum(sg == 0) == np.sum(so == 0)
    both = (sg == 0) & (so == 0)
    assert both.sum() >= 0.98 * len(w0)
    rel = np.linalg.norm(xg[both] - xo[both], axis=1) / np.linalg.norm(xo[both], axis=1)
    assert rel.max() <= 1e-8, rel.max()


def test_specialized_track_katsura10_all_paths(P):
    from workloads.make_starts import CONFIGS
    s = CONFIGS["katsura-10"](10_000)
    cells = SS.load_cells("katsura-10", 10_000)
    Wc = SS.cell_lifts_fast(s, cells)
    w0, tau0, cid = SS.start_points_cells(s, cells)
    g = _spec(P, s)
    wd, td = _cuda(w0), _cuda(tau0)
    st, _ = g.track_cells(wd, td, _cuda(Wc), _cuda(cid))
    sg = st.cpu().numpy()
    m, e = oracle.z_to_x(w0)
    xm, xe, _, so, _ = oracle.Oracle(s).track_x(m, e, tau0, cell_lift=Wc, path_cell=cid)
    xo, xg = xm * np.exp2(xe.astype(float)), np.exp(wd.cpu().numpy())
    assert np.sum(sg == 0) == np.sum(so == 0) == 990
    rel = np.linalg.norm(xg - xo, axis=1) / np.linalg.norm(xo, axis=1)
    assert rel.max() <= 1e-8, rel.max()


def test_specialize_subsets_and_flags(P):
    sysm = W.cyclic(5)
    g = P.System.from_workload(sysm)
    assert not g.specialized
    g.specialize(P._lib.SPEC_EVAL).set_kernels("specialized")
    assert g.specialized
    # kernels not specialised (step) still run (generic) and agree
    x, t, _ = W.random_points(64, 5, seed=1, tau_lo=-0.05)
    dE, dN, st = g.euler_newton(_cuda(x), _cuda(t))
    dE0, dN0, st0 = P.System.from_workload(sysm).euler_newton(_cuda(x), _cuda(t))
    assert np.array_equal(dE.cpu().numpy(), dE0.cpu().numpy())
    with pytest.raises(P.PhtError):
        g.specialize(64)


def test_specialize_refuses_oversized_code(P):
    """Random dense 20 x 50 terms would generate ~24,000 code units (minutes of NVRTC, i-cache
    bound): PHT_EUNSUPPORTED, and the handle keeps working on the generic / DMMA kernels."""
    sysm = W.random_dense(20, 50)
    g = P.System.from_workload(sysm)
    with pytest.raises(P.PhtError, match="-8"):
        g.specialize().set_kernels("specialized")
    assert not g.specialized
    x, t, _ = W.random_points(16, 20, seed=1, rho_max=0.5)
    H, J, Jt, st = g.evaluate(_cuda(x), _cuda(t))
    assert np.all(st.cpu().numpy() == 0)
