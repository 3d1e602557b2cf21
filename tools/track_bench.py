"""Full path tracking of the benchmark systems on one GPU (log-coordinate state), timed with CUDA
events; prints one JSON object.  Start systems from workloads/data (workloads.make_starts)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_14317_b200 as P  # noqa: E402
import workloads as W  # noqa: E402
from workloads import startsys as SS  # noqa: E402
from workloads.make_starts import CONFIGS  # noqa: E402

res = {}
OPTS = json.loads(os.environ.get("TB_OPTS", "{}"))
which = sys.argv[1:] or ["katsura-10:10000", "noon-10:10000", "cyclic-10:1000000"]
for item in which:
    name, L = item.split(":")
    L = int(L)
    sysm = CONFIGS[name](L)
    t0 = time.time()
    cells = SS.load_cells(name, L)
    CELLS = os.environ.get("TB_CELLS", "1") == "1"
    if CELLS:
        z, tau0, ids = SS.start_points_cells(sysm, cells)
        wc = torch.from_numpy(SS.cell_lifts_fast(sysm, cells)).cuda()
        cid = torch.from_numpy(ids).cuda()
    else:
        z, tau0, ids = SS.start_points_from_cells(sysm, cells)
    prep = time.time() - t0
    g = P.System.from_workload(sysm)
    if os.environ.get("PHT_SPEC") == "1" and sysm.offsets[-1] <= 256:
        t1 = time.time(); g.specialize(); print(json.dumps({"specialize_s": time.time() - t1}), file=sys.stderr)
    out = {}
    for rep in range(2):
        zd, td = torch.from_numpy(z.copy()).cuda(), torch.from_numpy(tau0.copy()).cuda()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if CELLS:
            st, stats = g.track_cells(zd, td, wc, cid, **OPTS)
        else:
            st, stats = g.track(zd, td, log_state=1, **OPTS)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    st = st.cpu().numpy()
    stats = stats.cpu().numpy()
    out.update(paths=len(z), ms=ms, paths_per_s=len(z) / ms * 1e3, status=np.bincount(st, minlength=33)[[0, 2, 4, 8, 16, 32]].tolist(),
               steps_mean=float(stats[:, 0].mean()), steps_max=int(stats[:, 0].max()), evals_total=int(stats[:, 2].sum()),
               rejects_mean=float(stats[:, 1].mean()), final_mean=float(stats[:, 3].mean()),
               evals_per_s=float(stats[:, 2].sum() / ms * 1e3), start_prep_s=prep,
               max_abs_re_z0=float(np.abs(z.real).max()), tau0_min=float(tau0.min()))
    out["opts"] = OPTS
    res[f"{name}:L{L}"] = out
    print(json.dumps({f"{name}:L{L}": out}), flush=True)
