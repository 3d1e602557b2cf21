"""Which cyclic-10 stage-1 paths fail, and why (stats, endpoint size, option sensitivity, oracle)."""
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
g = P.System.from_workload(s)
wcd, cidd = torch.from_numpy(Wc).cuda(), torch.from_numpy(cid).cuda()
wd, td = torch.from_numpy(w0.copy()).cuda(), torch.from_numpy(tau0.copy()).cuda()
st, stats = g.track_cells(wd, td, wcd, cidd)
sg, sts, z = st.cpu().numpy(), stats.cpu().numpy(), wd.cpu().numpy()
bad = np.nonzero(sg != 0)[0]
print("failing", bad.tolist(), "status", sg[bad].tolist())
for b in bad:
    print(" path", b, "cell", cid[b], "tau0", tau0[b], "stats", sts[b].tolist(), "tau_end", td.cpu().numpy()[b],
          "max Re z", z[b].real.max(), "min Re z", z[b].real.min())
sub = lambda a: np.ascontiguousarray(a[bad])
for opts in [{}, {"final_iters": 20}, {"final_tol": 1e-11}, {"dtau_max": 0.1}, {"newton_tol": 1e-12},
             {"dtau_init": 0.01, "dtau_max": 0.05}, {"inf_norm": 1e30}]:
    wb, tb = torch.from_numpy(sub(w0)).cuda(), torch.from_numpy(sub(tau0)).cuda()
    s2, st2 = g.track_cells(wb, tb, wcd, torch.from_numpy(sub(cid)).cuda(), **opts)
    zb = wb.cpu().numpy()
    print(opts, "status", s2.cpu().numpy().tolist(), "steps", st2.cpu().numpy()[:, 0].tolist(), "fin", st2.cpu().numpy()[:, 3].tolist(),
          "maxRe", np.round(zb.real.max(1), 2).tolist())
m, e = oracle.z_to_x(sub(w0))
xm, xe, to, so, sto = oracle.Oracle(s).track_x(m, e, sub(tau0), cell_lift=Wc, path_cell=sub(cid))
print("oracle status", so.tolist(), "stats", sto.tolist(), "log10|x|max", np.round((np.log2(np.abs(xm).max(1)) + xe.max(1)) * 0.30103, 2).tolist())
# do the failing paths converge to an endpoint another path also reaches (path jumping)?
xg = np.exp(z[sg == 0])
for b in bad:
    xb = np.exp(z[b])
    d = np.linalg.norm(xg - xb, axis=1) / np.linalg.norm(xb)
    print(" path", b, "nearest finite endpoint rel dist", d.min())
