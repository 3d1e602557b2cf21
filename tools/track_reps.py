"""Repeated full tracking runs of one system (run-to-run spread of the tracker), ms per run."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_14317_b200 as P  # noqa: E402
from workloads import startsys as SS  # noqa: E402
from workloads.make_starts import CONFIGS  # noqa: E402

name, L = (sys.argv[1] if len(sys.argv) > 1 else "noon-10:10000").split(":")
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
sysm = CONFIGS[name](int(L))
cells = SS.load_cells(name, int(L))
z, tau0, ids = SS.start_points_cells(sysm, cells)
wc = torch.from_numpy(SS.cell_lifts_fast(sysm, cells)).cuda()
cid = torch.from_numpy(ids).cuda()
g = P.System.from_workload(sysm)
out = []
for r in range(reps):
    zd, td = torch.from_numpy(z.copy()).cuda(), torch.from_numpy(tau0.copy()).cuda()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st, stats = g.track_cells(zd, td, wc, cid)
    e1.record()
    torch.cuda.synchronize()
    out.append(round(e0.elapsed_time(e1), 2))
print(json.dumps({name: out}))
