"""GPU parity: the CUDA path (through the C ABI) against the oracle on identical seeded inputs.

Tolerances: evaluation <= 1e-10 in the term-sum metric (BASELINE.json north_star
"relative error <= 1e-10 in FP64 for H and J"); directions: backward error <= 1e-10 and forward
error <= 1e-9 where cond(Jx) <= 1e4 (reading R10).
"""
import numpy as np
import pytest

import oracle
import workloads as W
from tests.parity import backward_err, eval_err, rel_err, skeel_cond

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
    "random-6x9": lambda: W.random_dense(6, 9),
    "cyclic-14": lambda: W.cyclic(14),
    "random-20x50": lambda: W.random_dense(20, 50),
    "n1": lambda: W.from_terms("n1", 1, [[((2,), 1.0), ((0,), -3.0), ((-1,), 0.5)]]),
}


@pytest.mark.parametrize("name,p", [("cyclic-5", 1024), ("cyclic-10", 333), ("katsura-10", 200),
                                    ("noon-10", 257), ("chandra-6", 100), ("random-6x9", 77),
                                    ("cyclic-14", 97), ("random-20x50", 50), ("n1", 65)])
def test_evaluate_parity(P, name, p):
    sysm = SYSTEMS[name]()
    o = oracle.Oracle(sysm)
    x, t, _ = W.random_points(p, sysm.n, seed=3, rho_max=0.5 if sysm.n > 12 else 1.0)
    r = o.evaluate(x, t)
    g = P.System.from_workload(sysm)
    H, Jx, Jt, st = g.evaluate(_cuda(x), _cuda(t))
    torch.cuda.synchronize()
    assert np.all(st.cpu().numpy() == 0)
    assert eval_err(H.cpu().numpy(), r["H"], r["SH"]) <= 1e-10
    assert eval_err(Jx.cpu().numpy(), r["Jx"], r["SJx"]) <= 1e-10
    assert eval_err(Jt.cpu().numpy(), r["Jt"], r["SJt"]) <= 1e-10


def test_evaluate_scaled_rows_and_log_variant(P):
    sysm = W.cyclic(10, lift_max=100)
    g = P.System.from_workload(sysm)
    z, tau = W.random_log_points(300, 10, seed=5)
    x, t = np.exp(z), np.exp(tau)
    H, Jx, Jt, st = g.evaluate(_cuda(x), _cuda(t))
    Hs, Jxs, Jts, e2, st2 = g.evaluate(_cuda(x), _cuda(t), scaled=True)
    sc = np.exp2(e2.cpu().numpy().astype(float))
    assert np.allclose(Hs.cpu().numpy() * sc, H.cpu().numpy(), rtol=0, atol=0)
    assert np.array_equal(Jxs.cpu().numpy() * sc[:, :, None], Jx.cpu().numpy())
    # log coordinates: Jz = Jx diag(x), Jtau = t Jt
    Hl, Jz, Jtau, e2l, stl = g.evaluate_log(_cuda(z), _cuda(tau))
    scl = np.exp2(e2l.cpu().numpy().astype(float))
    o = oracle.Oracle(sysm).evaluate(x, t)
    assert eval_err(Hl.cpu().numpy() * scl, o["H"], o["SH"]) <= 1e-10
    Jz_ref = o["Jx"] * x[:, None, :]
    assert eval_err(Jz.cpu().numpy() * scl[:, :, None], Jz_ref, o["SJx"] * np.abs(x)[:, None, :]) <= 1e-10
    assert eval_err(Jtau.cpu().numpy() * scl, t[:, None] * o["Jt"], t[:, None] * o["SJt"]) <= 1e-10


def test_log_branch_invariance(P):
    """Any branch of log: shifting Im z_j by 2 pi m leaves the outputs unchanged."""
    sysm = W.noon(10, lift_max=100)
    g = P.System.from_workload(sysm)
    z, tau = W.random_log_points(64, 10, seed=6)
    shift = 2 * np.pi * np.random.default_rng(0).integers(-5, 6, size=z.shape)
    a = g.evaluate_log(_cuda(z), _cuda(tau))
    b = g.evaluate_log(_cuda(z + 1j * shift), _cuda(tau))
    sa = np.exp2(a[3].cpu().numpy().astype(float))[:, :, None]
    assert np.allclose(a[1].cpu().numpy() * sa, b[1].cpu().numpy() * sa, rtol=1e-13, atol=1e-13 * np.abs(a[1].cpu().numpy() * sa).max())


def test_large_liftings_against_extended_range_oracle(P):
    """noon-10 with omega ~ U{0..10^4} at |Re z| up to 60 and tau in [-5, 0]: monomials far outside
    double range; GPU row_exp2 output vs the oracle's extended-range evaluation."""
    sysm = W.noon(10, lift_max=10_000)
    g = P.System.from_workload(sysm)
    z, tau = W.random_log_points(64, 10, seed=8, rho_max=60.0, tau_lo=-5.0)
    Hl, Jz, Jtau, e2, st = g.evaluate_log(_cuda(z), _cuda(tau))
    assert np.all(st.cpu().numpy() == 0)
    # oracle inputs as (mantissa, exponent) without log/exp in the oracle: x = e^z computed here
    # in extended form (test plumbing): x = m 2^e with e = floor(Re z / ln 2)
    e = np.floor(z.real / np.log(2)).astype(np.int64)
    xm = np.exp(z.real - e * np.log(2)) * np.exp(1j * z.imag)
    te = np.floor(tau / np.log(2)).astype(np.int64)
    tm = np.exp(tau - te * np.log(2))
    o = oracle.Oracle(sysm).evaluate_x(xm, e, tm, te)
    e2 = e2.cpu().numpy().astype(np.int64)
    H = Hl.cpu().numpy()
    # compare log2 magnitudes relative to the row's term sum: |gpu - orc| / S in log space
    for q in range(64):
        for k in range(10):
            ls = o["LSH"][q, k]
            ref = o["Hm"][q, k] * np.exp2(float(o["He"][q, k] - ls))
            got = H[q, k] * np.exp2(float(e2[q, k] - ls))
            assert abs(got - ref) <= 1e-10 * 64 * 60, (q, k, got, ref)


def test_batch_composition_bitwise(P):
    """A point's results do not depend on its tile position or batch size (per-point arithmetic
    order is fixed): stronger than S:246-249."""
    sysm = W.katsura(10, lift_max=100)
    g = P.System.from_workload(sysm)
    x, t, _ = W.random_points(1000, 11, seed=9)
    full = [a.cpu().numpy() for a in g.evaluate(_cuda(x), _cuda(t))]
    for off, cnt in ((0, 1), (37, 5), (500, 333), (999, 1)):
        part = [a.cpu().numpy() for a in g.evaluate(_cuda(x[off:off + cnt]), _cuda(t[off:off + cnt]))]
        for A, B in zip(full, part):
            assert np.array_equal(A[off:off + cnt], B)


def test_status_isolation_and_empty(P):
    sysm = W.cyclic(5)
    g = P.System.from_workload(sysm)
    x, t, _ = W.random_points(8, 5, seed=1)
    x[3, 2] = 0
    t[5] = -1.0
    H, Jx, Jt, st = g.evaluate(_cuda(x), _cuda(t))
    s = st.cpu().numpy()
    assert s[3] & P.PT_ZERO_COORD and s[5] & P.PT_NONFINITE
    assert np.sum(s == 0) == 6
    o = oracle.Oracle(sysm).evaluate(x, np.where(t > 0, t, 1.0))
    ok = s == 0
    assert eval_err(H.cpu().numpy()[ok], o["H"][ok], o["SH"][ok]) <= 1e-10
    # p = 0 is a no-op
    e = torch.empty((0, 5), dtype=torch.complex128, device="cuda")
    g.evaluate(e, torch.empty(0, dtype=torch.float64, device="cuda"))


def _dirs_check(o, x, t, dE, dN, st):
    r = o.evaluate(x, t)
    good = st == 0
    be_E = backward_err(r["Jx"][good], dE[good], -r["Jt"][good])
    be_N = backward_err(r["Jx"][good], dN[good], -r["H"][good])
    assert be_E.max() <= 1e-10 and be_N.max() <= 1e-10
    oE, oN, ost = o.euler_newton(x, t)
    cond = skeel_cond(r["Jx"])
    well = good & (ost == 0) & (cond <= 1e4)
    assert well.sum() >= 0.5 * len(x)
    assert rel_err(dE[well], oE[well]).max() <= 1e-9
    assert rel_err(dN[well], oN[well]).max() <= 1e-9


@pytest.mark.parametrize("name,p", [("cyclic-5", 1024), ("cyclic-10", 333), ("katsura-10", 200),
                                    ("noon-10", 129), ("cyclic-14", 64), ("n1", 40)])
def test_euler_newton_parity(P, name, p):
    sysm = SYSTEMS[name]()
    o = oracle.Oracle(sysm)
    # tau near 0 keeps t^omega from flattening the rows (omega up to 100): Skeel cond ~1e2
    x, t, _ = W.random_points(p, sysm.n, seed=4, tau_lo=-0.05)
    g = P.System.from_workload(sysm)
    dE, dN, st = g.euler_newton(_cuda(x), _cuda(t))
    _dirs_check(o, x, t, dE.cpu().numpy(), dN.cpu().numpy(), st.cpu().numpy())


def test_euler_newton_worked_example(P):
    import json, os
    from fractions import Fraction
    gd = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cyclic3_worked_example.json")))
    eqs = [[(tuple(a), complex(*c), w) for a, c, w in eq] for eq in gd["equations"]]
    sysm = W.from_terms("g", 3, eqs, coeffs="native")
    cx = lambda v: complex(float(Fraction(v[0])), float(Fraction(v[1])))
    x = np.array([[cx(v) for v in gd["x"]]])
    g = P.System.from_workload(sysm)
    dE, dN, st = g.euler_newton(_cuda(x), _cuda(np.array([gd["t"]])))
    assert np.allclose(dE.cpu().numpy()[0], [cx(v) for v in gd["dE"]], atol=1e-14)
    assert np.allclose(dN.cpu().numpy()[0], [cx(v) for v in gd["dN"]], atol=1e-14)


def test_singular_flag(P):
    """x_1 x_2 - 1 = 0, x_1 x_2 - 1 = 0 (rank-1 Jacobian everywhere) -> SINGULAR, sibling system ok."""
    sysm = W.from_terms("sing", 2, [[((1, 1), 1.0), ((0, 0), -1.0)], [((1, 1), 2.0), ((0, 0), -2.0, )]],
                        coeffs="native")
    g = P.System.from_workload(sysm)
    x, t, _ = W.random_points(5, 2, seed=2)
    dE, dN, st = g.euler_newton(_cuda(x), _cuda(t))
    assert np.all(st.cpu().numpy() & P.PT_SINGULAR)


@pytest.mark.parametrize("name,p,K", [("cyclic-5", 1024, 1), ("cyclic-10", 300, 1), ("katsura-10", 150, 2),
                                      ("noon-10", 100, 1)])
def test_pc_step_parity(P, name, p, K):
    """The paper's Euler-Newton step vs the oracle's, same seeded inputs."""
    sysm = SYSTEMS[name]()
    o = oracle.Oracle(sysm)
    x, _, tau = W.random_points(p, sysm.n, seed=12, tau_lo=-0.05)
    dtau = np.full(p, 0.01)
    xo, tauo, sto, dno = o.pc_step(x, tau, dtau, K=K)
    g = P.System.from_workload(sysm)
    xg, taug = _cuda(x), _cuda(tau)
    st, dn = g.pc_step(xg, taug, _cuda(dtau), newton_iters=K)
    xg, st, dn = xg.cpu().numpy(), st.cpu().numpy(), dn.cpu().numpy()
    assert np.array_equal(taug.cpu().numpy(), tauo)
    r = o.evaluate(x, np.exp(tau))
    cond = skeel_cond(r["Jx"])
    well = (st == 0) & (sto == 0) & (cond <= 1e3)
    assert well.sum() >= 0.5 * p
    err = rel_err(xg[well], xo[well])
    assert err.max() <= 1e-9, err.max()
    assert np.allclose(dn[well], dno[well], rtol=1e-6, atol=1e-12)


@pytest.mark.parametrize("p", [500, 100_003])
def test_pc_step_host_equals_device(P, p):
    """The pipelined host-buffer entry point (chunks on 3 streams; 100,003 points = 4 chunks with
    a ragged last one) gives bitwise the device entry point's results, pinned or pageable."""
    sysm = W.cyclic(10, lift_max=100)
    g = P.System.from_workload(sysm)
    x, _, tau = W.random_points(p, 10, seed=13)
    dtau = np.full(p, 0.02)
    xd, td = _cuda(x), _cuda(tau)
    g.pc_step(xd, td, _cuda(dtau))
    xh, th = x.copy(), tau.copy()
    g.pc_step_host(xh, th, dtau)
    assert np.array_equal(xh, xd.cpu().numpy()) and np.array_equal(th, td.cpu().numpy())
    xp = torch.from_numpy(x.copy()).pin_memory()
    tp = torch.from_numpy(tau.copy()).pin_memory()
    g.pc_step_host(xp.numpy(), tp.numpy(), dtau)
    assert np.array_equal(xp.numpy(), xh) and np.array_equal(tp.numpy(), th)


@pytest.mark.parametrize("name,n", [("cyclic-5", 5), ("noon-5", 5), ("cyclic-10", 10)])
def test_evaluate_log_extreme_rows(P, name, n):
    """Rows whose terms span more than e^512 (online rescale mid-row), including the case where
    the second term of a processed pair triggers the rescale: GPU vs extended-range oracle."""
    sysm = {"cyclic-5": W.cyclic(5, lift_max=100), "noon-5": W.noon(5, lift_max=1000),
            "cyclic-10": W.cyclic(10, lift_max=100)}[name]
    z, tau = W.random_log_points(200, n, seed=17, rho_max=300.0, tau_lo=-8.0)
    g = P.System.from_workload(sysm)
    Hl, Jz, Jtau, e2, st = g.evaluate_log(_cuda(z), _cuda(tau))
    e = np.floor(z.real / np.log(2)).astype(np.int64)
    xm = np.exp(z.real - e * np.log(2)) * np.exp(1j * z.imag)
    te = np.floor(tau / np.log(2)).astype(np.int64)
    tm = np.exp(tau - te * np.log(2))
    o = oracle.Oracle(sysm).evaluate_x(xm, e, tm, te)
    H, e2 = Hl.cpu().numpy(), e2.cpu().numpy().astype(np.int64)
    worst = 0.0
    for q in range(len(z)):
        for k in range(n):
            ls = o["LSH"][q, k]
            ref = o["Hm"][q, k] * np.exp2(float(o["He"][q, k] - ls))
            got = H[q, k] * np.exp2(float(e2[q, k] - ls))
            worst = max(worst, abs(got - ref))
    # a-priori bound (reading R9/A27): ~2.7 u * max|phi| ~ 1e-12 here
    assert worst <= 1e-10, worst


def test_evaluate_vanishing_terms_huge_lifting(P):
    """A term with tau*omega ~ -1e7 (far below the row) must vanish, not wrap the exponent:
    h = x1 - t^(10^7) x2 at tau = -1 equals x1 (regression: 32-bit overflow in the exp reduction)."""
    sysm = W.from_terms("huge", 2, [[((1, 0), 1.0, 0), ((0, 1), -1.0, 10**7)], [((0, 1), 1.0, 0), ((0, 0), -2.0, 0)]],
                        coeffs="native")
    g = P.System.from_workload(sysm)
    z = np.array([[0.3 + 0.2j, 0.1 - 0.4j]] * 4)
    tau = np.array([-1.0, -3.0, -0.5, -2.0])
    H, Jz, Jtau, e2, st = g.evaluate_log(_cuda(z), _cuda(tau))
    H = H.cpu().numpy() * np.exp2(e2.cpu().numpy().astype(float))
    assert np.allclose(H[:, 0], np.exp(z[:, 0]), rtol=1e-14, atol=0)
    o = oracle.Oracle(sysm).evaluate(np.exp(z), np.exp(tau))
    assert np.allclose(H, o["H"], rtol=1e-14, atol=1e-300)


@pytest.mark.parametrize("n,m,p", [(20, 50, 200), (12, 20, 97), (16, 30, 64)])
def test_dense_tensor_core_evaluate(P, n, m, p):
    """Config C4 (random dense Laurent system): the FP64 tensor-core (DMMA) evaluation path
    (pht_dense.cuh) vs the oracle, scaled and unscaled, and against the generic path."""
    sysm = W.random_dense(n, m, seed=n)
    g = P.System.from_workload(sysm)
    assert g.dense
    x, t, _ = W.random_points(p, n, seed=5, rho_max=0.5)
    o = oracle.Oracle(sysm).evaluate(x, t)
    H, Jx, Jt, st = g.evaluate(_cuda(x), _cuda(t))
    assert np.all(st.cpu().numpy() == 0)
    assert eval_err(H.cpu().numpy(), o["H"], o["SH"]) <= 1e-10
    assert eval_err(Jx.cpu().numpy(), o["Jx"], o["SJx"]) <= 1e-10
    assert eval_err(Jt.cpu().numpy(), o["Jt"], o["SJt"]) <= 1e-10
    Hs, Jxs, Jts, e2, _ = g.evaluate(_cuda(x), _cuda(t), scaled=True)
    sc = np.exp2(e2.cpu().numpy().astype(float))
    assert eval_err(Hs.cpu().numpy() * sc, o["H"], o["SH"]) <= 1e-10
    z, tau = np.log(x), np.log(t)
    Hl, Jz, Jtau, e2l, _ = g.evaluate_log(_cuda(z), _cuda(tau))
    scl = np.exp2(e2l.cpu().numpy().astype(float))
    assert eval_err(Jz.cpu().numpy() * scl[:, :, None], o["Jx"] * x[:, None, :], o["SJx"] * np.abs(x)[:, None, :]) <= 1e-10
    # the direction solve for the same system runs on the generic kernel: still consistent
    dE, dN, st2 = g.euler_newton(_cuda(x), _cuda(t))
    be = backward_err(o["Jx"], dN.cpu().numpy(), -o["H"])
    assert be[st2.cpu().numpy() == 0].max() <= 1e-10
