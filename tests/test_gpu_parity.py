"""GPU parity: the CUDA path (through the C ABI) against the oracle on identical seeded inputs.

Tolerances: evaluation <= 1e-10 in the term-sum metric (BASELINE.json north_star
"relative error <= 1e-10 in FP64 for H and J"); directions: backward error <= 1e-10 and forward
error <= 1e-9 where cond(Jx) <= 1e4 (reading R10).
"""
import numpy as np
import pytest

import oracle
import workloads as W
from tests.parity import backward_err, dirs_parity, eval_err, step_parity, xeval_errs

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


FAMILIES_LOG = ["tile", "dense", "specialized", "lane"]   # every kernel that implements pht_evaluate_log


def _log_family(P, sysm, family):
    g = P.System.from_workload(sysm)
    if family == "specialized":
        g.specialize(P._lib.SPEC_EVAL)
    return g.set_kernels(family)


@pytest.mark.parametrize("family", FAMILIES_LOG)
def test_range_stress_noon10_extended_oracle(P, family):
    """SURVEY §8(d) C5 range-stress set: noon-10 with omega ~ U{0..10^4}, Re z ~ U[-100, 100],
    tau ~ U[-5, 0] -- monomials up to e^(+-5e4), far outside double range.  H, Jz = Jx diag(x)
    and Jtau = t Jt against the oracle's extended-range evaluation at the exact points (SURVEY
    O2), each entry <= 1e-10 of its term sum (reading R9, A25 floor).  A-priori bound (A27):
    2.7 u (sum |a_j rho_j| + omega |tau|) <= 2.7 u 5.03e4 = 1.5e-11."""
    sysm = W.noon(10, lift_max=10_000)
    g = _log_family(P, sysm, family)
    xm, xe, tm, te, z, tau = W.random_extended_points(96, 10, seed=8, rho_max=100.0, tau_lo=-5.0)
    Hl, Jz, Jtau, e2, st = g.evaluate_log(_cuda(z), _cuda(tau))
    assert np.all(st.cpu().numpy() == 0)
    o = oracle.Oracle(sysm).evaluate_x(xm, xe, tm, te)
    eH, eJ, eT = xeval_errs(o, xm, xe, tm, te, Hl.cpu().numpy(), Jz.cpu().numpy(), Jtau.cpu().numpy(),
                            e2.cpu().numpy())
    assert max(eH, eJ, eT) <= 1e-10, (eH, eJ, eT)


@pytest.mark.parametrize("family", FAMILIES_LOG)
@pytest.mark.parametrize("name,n", [("cyclic-5", 5), ("noon-5", 5), ("cyclic-10", 10)])
def test_evaluate_log_extreme_rows(P, name, n, family):
    """Rows whose terms span more than e^512 (online rescale mid-row), including the case where
    the second term of a processed pair triggers the rescale: H, Jz, Jtau vs the extended-range
    oracle, <= 1e-10 of the term sums (A27 bound here ~1e-12)."""
    sysm = {"cyclic-5": W.cyclic(5, lift_max=100), "noon-5": W.noon(5, lift_max=1000),
            "cyclic-10": W.cyclic(10, lift_max=100)}[name]
    xm, xe, tm, te, z, tau = W.random_extended_points(200, n, seed=17, rho_max=300.0, tau_lo=-8.0)
    g = _log_family(P, sysm, family)
    Hl, Jz, Jtau, e2, st = g.evaluate_log(_cuda(z), _cuda(tau))
    assert np.all(st.cpu().numpy() == 0)
    o = oracle.Oracle(sysm).evaluate_x(xm, xe, tm, te)
    eH, eJ, eT = xeval_errs(o, xm, xe, tm, te, Hl.cpu().numpy(), Jz.cpu().numpy(), Jtau.cpu().numpy(),
                            e2.cpu().numpy())
    assert max(eH, eJ, eT) <= 1e-10, (eH, eJ, eT)


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
    """Reading R10 / VERDICT r1 1(iv): identical status-0 sets, backward error <= 1e-10 against the
    oracle's J, and EVERY coordinate of every status-0 point within EPS_SOLVE x its componentwise
    forward-error scale (no point dropped for its condition number)."""
    same, be, ratio = dirs_parity(o, x, t, dE, dN, st)
    assert same
    assert (st == 0).sum() >= 0.9 * len(x)
    assert max(be) <= 1e-10, be
    assert max(ratio) <= 1.0, ratio


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
    """The paper's Euler-Newton step vs the oracle's, same seeded inputs: identical
    statuses and tau, every coordinate of every status-0 point within its error bound."""
    sysm = SYSTEMS[name]()
    o = oracle.Oracle(sysm)
    x, _, tau = W.random_points(p, sysm.n, seed=12, tau_lo=-0.05)
    dtau = np.full(p, 0.01)
    g = P.System.from_workload(sysm)
    xg, taug = _cuda(x), _cuda(tau)
    st, dn = g.pc_step(xg, taug, _cuda(dtau), newton_iters=K)
    same, tau_eq, ratio = step_parity(o, x, tau, dtau, K, xg.cpu().numpy(), st.cpu().numpy(), taug.cpu().numpy())
    assert same and tau_eq
    assert (st.cpu().numpy() == 0).sum() >= 0.9 * p
    assert ratio <= 1.0, ratio


@pytest.mark.parametrize("p", [4099, 100_003])
def test_pc_step_host_oracle_parity(P, p):
    """The end-to-end entry point (pht_pc_step_host, the bench's e2e path; 100,003 points = 4
    pipelined chunks with a ragged last one) against oracle.pc_step on the bench's inputs."""
    import bench
    sysm = bench._system()
    x, _, tau = W.random_points(p, sysm.n, seed=14, tau_lo=bench.TAU_LO)
    dtau = np.full(p, bench.DTAU)
    g = P.System.from_workload(sysm)
    xh, th = x.copy(), tau.copy()
    st, _ = g.pc_step_host(xh, th, dtau, 1)
    pick = np.sort(np.random.default_rng(5).choice(p, min(p, 2048), replace=False))
    same, tau_eq, ratio = step_parity(oracle.Oracle(sysm), x[pick], tau[pick], dtau[pick], 1, xh[pick], st[pick],
                                      th[pick])
    assert same and tau_eq
    assert ratio <= 1.0, ratio


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


def test_pc_step_host_async_chain_equals_sync(P):
    """pht_pc_step_host_async: three chained steps (each chunk's copy-in waits only for the
    previous step's copy-out of the same chunk), then one with a different point count (waits for
    the whole chain), then pht_host_wait -- bitwise the results of the synchronous calls, and a
    synchronous call after an async chain orders itself behind it."""
    sysm = W.cyclic(10, lift_max=100)
    g = P.System.from_workload(sysm)
    p = 300_007                                    # 10 chunks of 32,768 (the minimum), the last one ragged
    x, _, tau = W.random_points(p, 10, seed=17)
    dtau = np.full(p, 0.01)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    xs, ts = x.copy(), tau.copy()
    for _ in range(3):
        g.pc_step_host(xs, ts, dtau)
    xa, ta, da = pin(x), pin(tau), pin(dtau)
    sa, na = pin(np.zeros(p, np.uint8)), pin(np.zeros(p))
    for _ in range(3):
        g.pc_step_host(xa, ta, da, 1, sa, na, asynchronous=True)
    q = 70_001
    xq, tq, dq = pin(x[:q]), pin(tau[:q]), pin(dtau[:q])
    sq, nq = pin(np.zeros(q, np.uint8)), pin(np.zeros(q))
    g.pc_step_host(xq, tq, dq, 1, sq, nq, asynchronous=True)
    g.host_wait()
    assert np.array_equal(xa, xs) and np.array_equal(ta, ts)
    x1, t1 = x[:q].copy(), tau[:q].copy()
    g.pc_step_host(x1, t1, dtau[:q])
    assert np.array_equal(xq, x1) and np.array_equal(tq, t1)
    g.pc_step_host(xa, ta, da, 1, sa, na, asynchronous=True)
    xs2, ts2 = xs.copy(), ts.copy()
    g.pc_step_host(xs2, ts2, dtau)                 # a synchronous step right behind an async one
    g.host_wait()
    g.pc_step_host(xs, ts, dtau)
    assert np.array_equal(xa, xs) and np.array_equal(xs2, xs)


def test_destroy_waits_for_async_host_steps(P):
    """pht_system_destroy right after pht_pc_step_host_async (no pht_host_wait): the handle waits
    for the in-flight copies before it releases the workspace, events and streams; the host
    buffers hold the finished step afterwards."""
    sysm = W.cyclic(10, lift_max=100)
    p = 200_000
    x, _, tau = W.random_points(p, 10, seed=19)
    dtau = np.full(p, 0.01)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    xa, ta, da = pin(x), pin(tau), pin(dtau)
    sa, na = pin(np.zeros(p, np.uint8)), pin(np.zeros(p))
    g = P.System.from_workload(sysm)
    g.pc_step_host(xa, ta, da, 1, sa, na, asynchronous=True)
    g.close()
    xs, ts = x.copy(), tau.copy()
    P.System.from_workload(sysm).pc_step_host(xs, ts, dtau)
    assert np.array_equal(xa, xs) and np.array_equal(ta, ts)


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


@pytest.mark.parametrize("counts", [(1, 3, 9, 2, 14, 8), (8, 8, 5, 3, 11, 1, 2, 16, 7, 6),
                                    (2, 2, 2, 2, 2, 2, 2), (13, 50, 4, 27, 3, 9, 8, 1)])
def test_dense_packed_tiles_ragged_equations(P, counts):
    """The DMMA path streams the terms of all equations in n-tiles of 8 slots: a tile may end one
    equation and start the next (build_dense; at most one start inside a tile, a second is moved to
    the next tile behind padding slots).  Ragged term counts exercise every case: equations shorter
    than a tile, ending exactly at a tile end, a second boundary forcing padding, one-term rows.
    Against the oracle at <= 1e-10 (term-sum metric), unscaled, scaled and log variants."""
    n = len(counts)
    rng = np.random.Generator(np.random.PCG64(sum(counts)))
    eqs = []
    for m in counts:
        seen = set()
        while len(seen) < m:
            seen.add(tuple(int(v) for v in rng.integers(-2, 3, size=n)))
        eqs.append([(a, 1.0) for a in sorted(seen)])
    sysm = W.from_terms(f"ragged-{n}", n, eqs, seed=n, lift_max=20)
    g = P.System.from_workload(sysm).set_kernels("dense")
    x, t, _ = W.random_points(93, n, seed=6, rho_max=0.5)
    o = oracle.Oracle(sysm).evaluate(x, t)
    H, Jx, Jt, st = g.evaluate(_cuda(x), _cuda(t))
    assert np.all(st.cpu().numpy() == 0)
    assert eval_err(H.cpu().numpy(), o["H"], o["SH"]) <= 1e-10
    assert eval_err(Jx.cpu().numpy(), o["Jx"], o["SJx"]) <= 1e-10
    assert eval_err(Jt.cpu().numpy(), o["Jt"], o["SJt"]) <= 1e-10
    Hs, Jxs, Jts, e2, _ = g.evaluate(_cuda(x), _cuda(t), scaled=True)
    sc = np.exp2(e2.cpu().numpy().astype(float))
    assert eval_err(Jxs.cpu().numpy() * sc[:, :, None], o["Jx"], o["SJx"]) <= 1e-10
    Hl, Jz, Jtau, e2l, _ = g.evaluate_log(_cuda(np.log(x)), _cuda(np.log(t)))
    scl = np.exp2(e2l.cpu().numpy().astype(float))
    assert eval_err(Hl.cpu().numpy() * scl, o["H"], o["SH"]) <= 1e-10
    assert eval_err(Jz.cpu().numpy() * scl[:, :, None], o["Jx"] * x[:, None, :], o["SJx"] * np.abs(x)[:, None, :]) <= 1e-10


@pytest.mark.parametrize("family", ["tile", "dense", "specialized", "lane"])
def test_row_rescale_keeps_entries_far_below_the_row(P, family):
    """Regression (found by the C5 range-stress test): the online row rescale by 2^d with
    d < -1074 must not flush entries that stay representable.  h_1 = 1 + x1 + x2^2 at
    x1 = x2 = 2^600: the first term sets the row exponent (0), x1 = 2^600 enters without a
    rescale (600 bits < e^512), x2^2 = 2^1200 rescales by 2^-1200; dh_1/dz_1 = x1 = 2^600 is
    2^-600 of the row and must survive (it is the entry's only term)."""
    sysm = W.from_terms("resc", 2, [[((0, 0), 1.0), ((1, 0), 1.0), ((0, 2), 1.0)],
                                    [((1, 0), 1.0), ((0, 1), 1.0)]], coeffs="native")
    g = P.System.from_workload(sysm)
    if family == "specialized":
        g.specialize(P._lib.SPEC_EVAL)
    g.set_kernels(family)
    z = np.full((3, 2), 600 * np.log(2) + 0j)
    tau = np.zeros(3)
    H, Jz, Jtau, e2, st = [a.cpu().numpy() for a in g.evaluate_log(_cuda(z), _cuda(tau))]
    assert np.all(st == 0)
    # tolerance: the A27 bound 2.7 u |phi| with |phi| = 1200 ln 2 is 2.5e-13
    row = lambda a: a * np.exp2(e2[:, 0].astype(float) - 1200)          # in units of 2^1200
    assert np.allclose(row(Jz[:, 0, 0]), 2.0 ** -600, rtol=1e-12, atol=0), row(Jz[:, 0, 0]) * 2.0 ** 600
    assert np.allclose(row(Jz[:, 0, 1]), 2.0, rtol=1e-12, atol=0), row(Jz[:, 0, 1])
    # (pht_evaluate's dh/dx1 = 1 is 2^-1200 of that row: below the row_exp2 representation, A25)


@pytest.mark.parametrize("family", ["warp", "lane", "tile", "dense"])
def test_log_split_round_trip(P, family):
    """Stage 1 (a1) through evaluation and back: h = x (one term, exponent 1) returns
    H = exp(log|x|) cis(arg x) = x and dh/dx = 1 for every octant, both signed zeros of the
    imaginary part, and |x| from 1e-140 to 1e140 (the table-driven log / atan2 of the warp and lane
    kernels, libdevice in the tile kernel).  Bound: ~2u |log|x|| from the log, ~1 ulp of pi from the
    angle and a few ulp from exp*cis."""
    sysm = W.from_terms("id", 1, [[((1,), 1.0, 0)]], coeffs="native")
    g = P.System.from_workload(sysm).set_kernels(family)
    rng = np.random.default_rng(21)
    mag = np.exp(rng.uniform(-322, 322, 4000))
    ang = rng.uniform(-np.pi, np.pi, 4000)
    ang[:16] = np.arange(16) * np.pi / 8 - np.pi                 # octant boundaries
    x = mag * np.exp(1j * ang)
    x[16:20] = [1.0 + 0.0j, -1.0 + 0.0j, complex(-1.0, -0.0), complex(0.0, -3.0)]
    x = x[:, None]
    H, Jx, Jt, st = [a.cpu().numpy() for a in g.evaluate(_cuda(x), _cuda(np.ones(len(x))))]
    assert np.all(st == 0)
    bound = 2.2e-16 * 3 * (np.abs(np.log(np.abs(x[:, 0]))) + 8)
    assert np.all(np.abs(H[:, 0] - x[:, 0]) / np.abs(x[:, 0]) <= bound)
    assert np.all(np.abs(Jx[:, 0, 0] - 1.0) <= bound)


def test_misaligned_complex_pointers_are_refused(P):
    """Complex arrays move as 16-byte vectors: an only 8-byte-aligned complex pointer is refused
    with PHT_EINVAL up front instead of faulting the context (include/pht.h conventions)."""
    import ctypes
    sysm = W.cyclic(10, lift_max=100)
    g = P.System.from_workload(sysm)
    p, n = 100, 10
    x, t, _ = W.random_points(p, n, seed=44)
    xd, td = _cuda(x), _cuda(t)
    buf = torch.zeros(2 * p * n * n + 1, dtype=torch.float64, device="cuda")
    st = torch.empty(p, dtype=torch.uint8, device="cuda")
    cs = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    X, T, S = ctypes.c_void_p(xd.data_ptr()), ctypes.c_void_p(td.data_ptr()), ctypes.c_void_p(st.data_ptr())
    bad = ctypes.c_void_p(buf.data_ptr() + 8)
    assert g._lib.pht_evaluate(g._h, p, X, T, None, bad, None, None, S, cs) == -1
    assert g._lib.pht_evaluate(g._h, p, ctypes.c_void_p(buf.data_ptr() + 8), T, None, None, None, None, S, cs) == -1
    assert g._lib.pht_euler_newton(g._h, p, X, T, bad, None, S, cs) == -1
    # the handle and the context still work
    H, J, Jt, st2 = g.evaluate(xd, td)
    torch.cuda.synchronize()
    assert bool((st2 == 0).all())


@pytest.mark.parametrize("n,m", [(6, 500), (12, 150), (8, 40)])
def test_lane_evaluation_record_layouts(P, n, m):
    """k_evalw keeps the term records as doubles in shared memory (warp-broadcast loads) and falls
    back to the compact int16 records when those would not fit (n = 6 with 500 terms, n = 12 with
    150 terms per equation); both against the oracle (R9 metric <= 1e-10)."""
    sysm = W.random_dense(n, m, emax=2 if n < 12 else 1, seed=n + m, lift_max=20)
    g = P.System.from_workload(sysm).set_kernels("lane")
    x, t, _ = W.random_points(67, n, seed=2, rho_max=0.3)
    o = oracle.Oracle(sysm).evaluate(x, t)
    H, Jx, Jt, st = g.evaluate(_cuda(x), _cuda(t))
    assert np.all(st.cpu().numpy() == 0)
    assert eval_err(H.cpu().numpy(), o["H"], o["SH"]) <= 1e-10
    assert eval_err(Jx.cpu().numpy(), o["Jx"], o["SJx"]) <= 1e-10
    assert eval_err(Jt.cpu().numpy(), o["Jt"], o["SJt"]) <= 1e-10
