import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2111_14317_b200 as P, oracle
from workloads import startsys as SS
from workloads.make_starts import CONFIGS
s = CONFIGS["cyclic-10"](1000000)
cells = SS.load_cells("cyclic-10", 1000000)
Wc = SS.cell_lifts_fast(s, cells)
w0, tau0, cid = SS.start_points_cells(s, cells)
pick = np.sort(np.random.default_rng(3).choice(len(w0), 256, replace=False))
w0, tau0, cid = w0[pick], tau0[pick], cid[pick]
g = P.System.from_workload(s)
for opts in [{}, {"newton_tol": 1e-8}, {"dtau_max": 0.1}, {"dtau_init": 0.01, "dtau_max": 0.1}]:
    wd, td = torch.from_numpy(w0.copy()).cuda(), torch.from_numpy(tau0.copy()).cuda()
    st, stats = g.track_cells(wd, td, torch.from_numpy(Wc).cuda(), torch.from_numpy(cid).cuda(), **opts)
    sg, sts = st.cpu().numpy(), stats.cpu().numpy()
    print(opts, "gpu status", np.bincount(sg, minlength=33)[[0, 2, 4, 8, 16, 32]], flush=True)
    if not opts:
        m, e = oracle.z_to_x(w0)
        xm, xe, to, so, sto = oracle.Oracle(s).track_x(m, e, tau0, cell_lift=Wc, path_cell=cid)
        print("oracle status", np.bincount(so, minlength=33)[[0, 2, 4, 8, 16, 32]])
        bad = np.nonzero(sg != so)[0]
        for b in bad:
            print("path", pick[b], "cell", cid[b], "tau0", tau0[b], "gpu st", sg[b], sts[b], "orc st", so[b], sto[b], "gpu tau_end", td.cpu().numpy()[b], "orc tau_end", to[b])
        z = wd.cpu().numpy(); xg = np.exp(z); xo = xm * np.exp2(xe.astype(float))
        both = (sg == 0) & (so == 0)
        print("max rel endpoint diff", (np.linalg.norm(xg[both]-xo[both],axis=1)/np.linalg.norm(xo[both],axis=1)).max())
