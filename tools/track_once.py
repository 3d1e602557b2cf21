"""One pht_track_cells launch of all start paths of a stored system (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_14317_b200 as P  # noqa: E402
from workloads import startsys as SS  # noqa: E402
from workloads.make_starts import CONFIGS  # noqa: E402

name, L = (sys.argv[1] if len(sys.argv) > 1 else "katsura-10:10000").split(":")
L = int(L)
s = CONFIGS[name](L)
cells = SS.load_cells(name, L)
w0, tau0, cid = SS.start_points_cells(s, cells)
g = P.System.from_workload(s)
wc, cd = torch.from_numpy(SS.cell_lifts_fast(s, cells)).cuda(), torch.from_numpy(cid).cuda()
for _ in range(2):
    wd, td = torch.from_numpy(w0.copy()).cuda(), torch.from_numpy(tau0.copy()).cuda()
    st, _ = g.track_cells(wd, td, wc, cd)
torch.cuda.synchronize()
print("ok", int((st == 0).sum()))
