"""Tracking time vs the number of paths (the start set repeated r times): time(r P) - r time(P)
exposes the queue tail (the last paths after the queue drains)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_14317_b200 as P  # noqa: E402
from workloads import startsys as SS  # noqa: E402
from workloads.make_starts import CONFIGS  # noqa: E402

name, L = (sys.argv[1] if len(sys.argv) > 1 else "cyclic-10:1000000").split(":")
L = int(L)
s = CONFIGS[name](L)
cells = SS.load_cells(name, L)
w0, tau0, cid = SS.start_points_cells(s, cells)
g = P.System.from_workload(s)
wc = torch.from_numpy(SS.cell_lifts_fast(s, cells)).cuda()
res = {}
for r in (1, 2, 4):
    W0, T0, C0 = np.tile(w0, (r, 1)), np.tile(tau0, r), np.tile(cid, r)
    best = 1e9
    for _ in range(3):
        wd, td, cd = torch.from_numpy(W0).cuda(), torch.from_numpy(T0).cuda(), torch.from_numpy(C0).cuda()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st, stats = g.track_cells(wd, td, wc, cd)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[r] = round(best, 2)
print(json.dumps({name: res, "tail_estimate_ms": round(2 * res[1] - res[2], 2)}))
