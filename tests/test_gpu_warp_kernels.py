"""The warp-per-group kernels (k_stepw, k_trackw) against the tile kernels
(k_pht, k_track) on identical inputs, and the step against the oracle across the n range the
warp kernels cover.  The row arithmetic and the Gauss-Jordan elimination are the same code in
both layouts, so results agree to rounding; statuses and finite counts are identical.
The kernel family is chosen per handle with pht_system_set_kernels ("warp" / "tile")."""
import numpy as np
import pytest

import oracle
import workloads as W
from tests.parity import rel_err, step_parity
from workloads import startsys as SS

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    import paper_2111_14317_b200 as P
    return P


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


SYS = {"cyclic-5": lambda: W.cyclic(5), "cyclic-7": lambda: W.cyclic(7, lift_max=100),
       "cyclic-10": lambda: W.cyclic(10, lift_max=100), "katsura-10": lambda: W.katsura(10, lift_max=100),
       "noon-10": lambda: W.noon(10, lift_max=100), "chandra-6": lambda: W.chandra(6),
       "random-8x12": lambda: W.random_dense(8, 12), "n1": lambda: W.from_terms("n1", 1, [[((2,), 1.0), ((0,), -3.0)]])}


@pytest.mark.parametrize("name,p,K", [("cyclic-5", 4099, 1), ("cyclic-7", 1001, 2), ("cyclic-10", 3001, 1),
                                      ("katsura-10", 997, 2), ("noon-10", 1003, 1), ("chandra-6", 515, 3),
                                      ("random-8x12", 333, 1), ("n1", 97, 2)])
def test_stepw_equals_tile_kernel(P, name, p, K):
    """Ragged batches (not a multiple of the points per warp or per CTA) and K = 1..3."""
    sysm = SYS[name]()
    g = P.System.from_workload(sysm)
    x, _, tau = W.random_points(p, sysm.n, seed=31, tau_lo=-0.05)
    dtau = _cuda(np.full(p, 0.01))
    out = []
    for fam in ("warp", "tile"):
        g.set_kernels(fam)
        xg, tg = _cuda(x), _cuda(tau)
        st, dn = g.pc_step(xg, tg, dtau, newton_iters=K)
        out.append((xg.cpu().numpy(), tg.cpu().numpy(), st.cpu().numpy(), dn.cpu().numpy()))
    (xw, tw, sw, dw), (xt, tt, stt, dt) = out
    assert np.array_equal(sw, stt) and np.array_equal(tw, tt)
    ok = sw == 0
    assert ok.sum() >= 0.5 * p
    assert rel_err(xw[ok], xt[ok]).max() <= 1e-12
    assert np.allclose(dw[ok], dt[ok], rtol=1e-9, atol=1e-15)


@pytest.mark.parametrize("name,p", [("cyclic-7", 301), ("chandra-6", 200), ("random-8x12", 150)])
def test_stepw_oracle_parity(P, name, p):
    """k_stepw (the default for n <= 12) against the oracle's Euler-Newton step."""
    sysm = SYS[name]()
    o = oracle.Oracle(sysm)
    x, _, tau = W.random_points(p, sysm.n, seed=32, tau_lo=-0.05)
    dtau = np.full(p, 0.01)
    g = P.System.from_workload(sysm)
    xg, tg = _cuda(x), _cuda(tau)
    st, dn = g.pc_step(xg, tg, _cuda(dtau), newton_iters=1)
    same, tau_eq, ratio = step_parity(o, x, tau, dtau, 1, xg.cpu().numpy(), st.cpu().numpy(), tg.cpu().numpy())
    assert same and tau_eq and ratio <= 1.0, (same, tau_eq, ratio)


def test_stepw_status_isolation(P):
    """A zero coordinate, a non-finite x and a non-finite tau flag only their own points."""
    sysm = W.cyclic(10, lift_max=100)
    g = P.System.from_workload(sysm)
    x, _, tau = W.random_points(64, 10, seed=33, tau_lo=-0.05)
    x[5, 3] = 0
    x[17, 0] = np.nan
    tau[40] = np.inf
    xg, tg = _cuda(x), _cuda(tau)
    st, _ = g.pc_step(xg, tg, _cuda(np.full(64, 0.01)), newton_iters=1)
    st = st.cpu().numpy()
    bad = {5, 17, 40}
    assert all(st[i] != 0 for i in bad)
    assert np.sum(st[[i for i in range(64) if i not in bad]] != 0) <= 2


@pytest.mark.parametrize("name,L", [("katsura-10", 10_000), ("cyclic-10", 1_000_000)])
def test_trackw_equals_tile_tracker(P, name, L):
    """Every start path of katsura-10 (990) / cyclic-10 (35,940): identical statuses and finite
    counts, endpoints <= 1e-10 apart (an accept/reject decision may flip at rounding level,
    reading R14 -- the endpoints then still agree to the tracking tolerance)."""
    from workloads.make_starts import CONFIGS
    sysm = CONFIGS[name](L)
    cells = SS.load_cells(name, L)
    z, tau0, ids = SS.start_points_cells(sysm, cells)
    Wc = _cuda(SS.cell_lifts_fast(sysm, cells))
    g = P.System.from_workload(sysm)
    res = []
    for fam in ("warp", "tile"):
        g.set_kernels(fam)
        zd, td = _cuda(z), _cuda(tau0)
        st, stats = g.track_cells(zd, td, Wc, _cuda(ids))
        res.append((zd.cpu().numpy(), st.cpu().numpy()))
    (zw, sw), (zt, stt) = res
    assert np.array_equal(sw, stt) and np.sum(sw == 0) == len(z)
    xw, xt = np.exp(zw), np.exp(zt)
    assert (np.linalg.norm(xw - xt, axis=1) / np.linalg.norm(xt, axis=1)).max() <= 1e-10


@pytest.mark.parametrize("name,p", [("cyclic-5", 2051), ("cyclic-10", 1001), ("katsura-10", 333), ("n1", 65)])
def test_stepw_directions_equal_tile_kernel(P, name, p):
    """pht_euler_newton through k_stepw<N, DIRS> equals the tile kernel k_pht<N, DIRS>."""
    sysm = SYS[name]()
    g = P.System.from_workload(sysm)
    x, t, _ = W.random_points(p, sysm.n, seed=34, tau_lo=-0.05)
    out = []
    for fam in ("warp", "tile"):
        g.set_kernels(fam)
        dE, dN, st = g.euler_newton(_cuda(x), _cuda(t))
        out.append((dE.cpu().numpy(), dN.cpu().numpy(), st.cpu().numpy()))
    (ew, nw, sw), (et, nt, stt) = out
    assert np.array_equal(sw, stt)
    ok = sw == 0
    assert ok.sum() >= 0.5 * p
    assert rel_err(ew[ok], et[ok]).max() <= 1e-12 and rel_err(nw[ok], nt[ok]).max() <= 1e-12


@pytest.mark.parametrize("name,p", [("cyclic-5", 777), ("chandra-6", 517), ("cyclic-7", 1001), ("cyclic-10", 2003), ("noon-10", 301), ("n1", 65)])
def test_evaluate_warp_kernel_equals_tile_kernel(P, name, p):
    """pht_evaluate through k_stepw<N, EVAL_X>, the tile kernel k_phte and the point-per-lane kernel
    k_evalw (TMA stores) agree, unscaled and with row exponents (the same row arithmetic)."""
    sysm = SYS[name]()
    g = P.System.from_workload(sysm)
    x, t, _ = W.random_points(p, sysm.n, seed=35)
    for scaled in (False, True):
        out = []
        for fam in ("warp", "tile", "lane"):
            g.set_kernels(fam)
            r = g.evaluate(_cuda(x), _cuda(t), scaled=scaled)
            out.append([a.cpu().numpy() for a in r])
        for other in out[1:]:
            for a, b in zip(out[0], other):
                if a.dtype == np.complex128:
                    assert np.allclose(a, b, rtol=1e-13, atol=0) or np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)) <= 1e-13
                else:
                    assert np.array_equal(a, b)


@pytest.mark.parametrize("m", [300, 420])
def test_stepw_large_term_tables(P, m):
    """Many terms per equation: the term records no longer fit the warp kernels' shared memory
    (n = 6: 420 terms per equation) and the launch falls back to the tile kernel; just below the
    limit (300 terms) k_stepw runs with one CTA per SM.  Both agree with the tile kernel."""
    sysm = W.random_dense(6, m)
    g = P.System.from_workload(sysm)
    p = 301
    x, t, tau = W.random_points(p, 6, seed=36, tau_lo=-0.05, rho_max=0.3)
    out = []
    for fam in ("warp", "tile"):
        g.set_kernels(fam)
        xg, tg = _cuda(x), _cuda(tau)
        st, _ = g.pc_step(xg, tg, _cuda(np.full(p, 0.01)), newton_iters=1)
        H, Jx, Jt, est = g.evaluate(_cuda(x), _cuda(t))
        out.append((xg.cpu().numpy(), st.cpu().numpy(), Jx.cpu().numpy(), est.cpu().numpy()))
    (xw, sw, jw, ew), (xt, stt, jt, et) = out
    assert np.array_equal(sw, stt) and np.array_equal(ew, et)
    ok = sw == 0
    assert ok.sum() >= 0.5 * p
    assert rel_err(xw[ok], xt[ok]).max() <= 1e-11
    assert np.max(np.abs(jw - jt)) <= 1e-12 * np.max(np.abs(jt))
