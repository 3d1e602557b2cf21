"""Run-to-run determinism of the device tracker: track every start path of a config R times and
compare statuses and endpoints bitwise between runs (tools/track_determinism.py cyclic-10:1000000 8)."""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_14317_b200 as P  # noqa: E402
from workloads import startsys as SS  # noqa: E402
from workloads.make_starts import CONFIGS  # noqa: E402

item, reps = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 8
name, L = item.split(":")
sysm = CONFIGS[name](int(L))
cells = SS.load_cells(name, int(L))
z, tau0, ids = SS.start_points_cells(sysm, cells)
wc = torch.from_numpy(SS.cell_lifts_fast(sysm, cells)).cuda()
cid = torch.from_numpy(ids).cuda()
g = P.System.from_workload(sysm)
ref = None
out = []
for r in range(reps):
    zd, td = torch.from_numpy(z.copy()).cuda(), torch.from_numpy(tau0.copy()).cuda()
    st, stats = g.track_cells(zd, td, wc, cid)
    torch.cuda.synchronize()
    zs, ss = zd.cpu().numpy(), st.cpu().numpy()
    h = hashlib.sha1(zs.tobytes() + ss.tobytes()).hexdigest()[:12]
    if ref is None:
        ref = (zs, ss)
    diff_st = int((ss != ref[1]).sum())
    diff_z = int(np.any(zs != ref[0], axis=1).sum())
    out.append({"run": r, "finite": int((ss == 0).sum()), "hash": h, "status_diff": diff_st, "endpoint_diff_paths": diff_z})
print(json.dumps({item: out}))
