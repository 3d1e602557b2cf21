"""Tracking of small systems (all start paths, cell coordinates): generic vs specialised kernels."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_14317_b200 as P  # noqa: E402
import workloads as W  # noqa: E402
from workloads import startsys as SS  # noqa: E402

for name, s in [("cyclic-5", W.cyclic(5, lift_max=100)), ("noon-5", W.noon(5, lift_max=1000)),
                ("cyclic-7", W.cyclic(7, lift_max=10 ** 4)), ("noon-7", W.noon(7, lift_max=10 ** 4))]:
    cells = SS.mixed_cells_fast(s)
    Wc = torch.from_numpy(SS.cell_lifts_fast(s, cells)).cuda()
    w0, tau0, cid = SS.start_points_cells(s, cells)
    cidd = torch.from_numpy(cid).cuda()
    out = {"paths": len(w0)}
    for spec in (False, True):
        g = P.System.from_workload(s)
        if spec:
            g.specialize()
        best = 1e30
        for rep in range(3):
            wd, td = torch.from_numpy(w0.copy()).cuda(), torch.from_numpy(tau0.copy()).cuda()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            st, stats = g.track_cells(wd, td, Wc, cidd)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out["spec" if spec else "generic"] = {"ms": best, "finite": int((st == 0).sum())}
    print(json.dumps({name: out}), flush=True)
