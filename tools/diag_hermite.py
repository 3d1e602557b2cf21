import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2111_14317_b200 as P, oracle, workloads as W
from workloads import startsys as SS
s = W.katsura(6, lift_max=10 ** 4)
cells = SS.mixed_cells_fast(s); Wc = SS.cell_lifts(s, cells); w0, tau0, cid = SS.start_points_cells(s, cells)
g = P.System.from_workload(s)
m, e = oracle.z_to_x(w0)
for pr in (0, 1):
    wd, td = torch.from_numpy(w0.copy()).cuda(), torch.from_numpy(tau0.copy()).cuda()
    st, stats = g.track_cells(wd, td, torch.from_numpy(Wc).cuda(), torch.from_numpy(cid).cuda(), predictor=pr)
    sg, sts = st.cpu().numpy(), stats.cpu().numpy()
    xm, xe, _, so, sto = oracle.Oracle(s).track_x(m, e, tau0, cell_lift=Wc, path_cell=cid, predictor=pr)
    same = np.all(sts == sto, axis=1)
    print("pred", pr, "gpu finite", (sg == 0).sum(), "orc finite", (so == 0).sum(), "identical stats", same.sum(), "/", len(sg))
    for i in range(6):
        print("   path", i, "gpu", sg[i], sts[i].tolist(), "orc", so[i], sto[i].tolist())
