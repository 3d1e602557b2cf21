import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2111_14317_b200 as P, workloads as W, oracle
from workloads import startsys as SS
c5 = W.cyclic(5, lift_max=100)
g = P.System.from_workload(c5)
for zmax in (20, None):
    x, tau0, _, z = SS.start_points(c5, zmax=zmax)
    zd, td = torch.from_numpy(z.copy()).cuda(), torch.from_numpy(tau0.copy()).cuda()
    st, stats = g.track(zd, td, log_state=1)
    st = st.cpu().numpy(); stats = stats.cpu().numpy()
    print("zmax", zmax, "log-state status", np.bincount(st, minlength=33)[[0, 2, 4, 8, 16, 32]], "steps", stats[:, 0].min(), stats[:, 0].max(), "rej", stats[:, 1].sum())
    if zmax == 20:
        xd, td = torch.from_numpy(x.copy()).cuda(), torch.from_numpy(tau0.copy()).cuda()
        st2, stats2 = g.track(xd, td)
        print("  x-state status", np.bincount(st2.cpu().numpy(), minlength=33)[[0, 2, 4, 8, 16, 32]], "steps", stats2.cpu().numpy()[:, 0].max())
    # evaluation precision at the start points (log variant vs extended-range oracle)
    Hl, Jz, Jtau, e2, stl = g.evaluate_log(torch.from_numpy(z.copy()).cuda(), torch.from_numpy(tau0.copy()).cuda())
    m, e = oracle.z_to_x(z)
    te = np.floor(tau0 / np.log(2)).astype(np.int64); tm = np.exp(tau0 - te * np.log(2))
    o = oracle.Oracle(c5).evaluate_x(m, e, tm, te)
    H = Hl.cpu().numpy(); e2 = e2.cpu().numpy().astype(np.int64)
    errs = []
    for q in range(len(z)):
        for k in range(5):
            ls = o["LSH"][q, k]
            ref = o["Hm"][q, k] * np.exp2(float(o["He"][q, k] - ls))
            got = H[q, k] * np.exp2(float(e2[q, k] - ls))
            errs.append(abs(got - ref))
    print("  eval H err (term-sum metric) max", max(errs), "median", np.median(errs), "max|Re z|", np.abs(z.real).max())
