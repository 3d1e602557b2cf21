"""Tail effect of the persistent tracker: time with the stored path order vs the same paths in
descending-evaluations order (longest first, LPT), and how much of the per-path evaluation count
the path's mixed cell explains.  Prints one JSON line per system."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_14317_b200 as P  # noqa: E402
from workloads import startsys as SS  # noqa: E402
from workloads.make_starts import CONFIGS  # noqa: E402

for item in sys.argv[1:] or ["noon-10:10000", "cyclic-10:1000000"]:
    name, L = item.split(":")
    L = int(L)
    sysm = CONFIGS[name](L)
    cells = SS.load_cells(name, L)
    z, tau0, ids = SS.start_points_cells(sysm, cells)
    wc = torch.from_numpy(SS.cell_lifts_fast(sysm, cells)).cuda()
    g = P.System.from_workload(sysm)

    def run(order):
        zd = torch.from_numpy(z[order].copy()).cuda()
        td = torch.from_numpy(tau0[order].copy()).cuda()
        cid = torch.from_numpy(ids[order].copy()).cuda()
        best = None
        for _ in range(2):
            zz, tt = zd.clone(), td.clone()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            st, stats = g.track_cells(zz, tt, wc, cid)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        return best, stats.cpu().numpy()

    base = np.arange(len(z))
    ms0, stats = run(base)
    ev = stats[:, 2].astype(np.float64)
    lpt = np.argsort(-ev, kind="stable")
    ms1, _ = run(lpt)
    # share of the evaluation-count variance explained by the cell (between-cell variance)
    cm = np.bincount(ids, weights=ev) / np.maximum(np.bincount(ids), 1)
    r2 = float(np.var(cm[ids]) / max(np.var(ev), 1e-30))
    if os.environ.get("TT_DUMP"):
        np.save(f"gpurun_out/tail_{name}_evals.npy", stats)
    print(json.dumps({name: {"paths": len(z), "ms_stored_order": ms0, "ms_longest_first": ms1,
                             "evals_mean": float(ev.mean()), "evals_max": float(ev.max()),
                             "evals_p99": float(np.percentile(ev, 99)), "cells": int(ids.max() + 1),
                             "cell_r2": r2}}), flush=True)
