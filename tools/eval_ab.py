"""pht_evaluate / pht_evaluate_log throughput per kernel family: (G points/s evaluate, G points/s
evaluate_log (includes its allocations), max deviation of Jx from the first family), one GPU."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_14317_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

fams = sys.argv[1].split(",") if len(sys.argv) > 1 else ["lane", "warp", "dense", "tile"]
res = {}
for name, sysm, p in [("cyclic-5", W.cyclic(5, lift_max=100), 1 << 22), ("chandra-6", W.chandra(6), 1 << 22),
                      ("cyclic-7", W.cyclic(7, lift_max=100), 1 << 22), ("cyclic-10", W.cyclic(10, lift_max=100), 1 << 21),
                      ("noon-10", W.noon(10, lift_max=100), 1 << 21), ("katsura-10", W.katsura(10, lift_max=100), 1 << 21)]:
    g = P.System.from_workload(sysm)
    x, t, _ = W.random_points(p, sysm.n, seed=5)
    xd, td = torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda()
    n = sysm.n
    out = (torch.empty((p, n), dtype=torch.complex128, device="cuda"), torch.empty((p, n, n), dtype=torch.complex128, device="cuda"),
           torch.empty((p, n), dtype=torch.complex128, device="cuda"), torch.empty(p, dtype=torch.uint8, device="cuda"))
    r = {}
    ref = None
    for fam in fams:
        try:
            g.set_kernels(fam)
        except Exception as e:
            r[fam] = str(e)[:40]
            continue
        for _ in range(2):
            g.evaluate(xd, td, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            g.evaluate(xd, td, out=out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        zd, taud = torch.log(xd), torch.log(td)
        g.evaluate_log(zd, taud)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(3):
            g.evaluate_log(zd, taud)
        e1.record()
        torch.cuda.synchronize()
        msz = e0.elapsed_time(e1) / 3
        J = out[1][:4096].cpu().numpy()
        if ref is None:
            ref = J
            dev = 0.0
        else:
            dev = float(np.max(np.abs(J - ref)) / np.max(np.abs(ref)))
        r[fam] = (round(p / ms / 1e6, 3), round(p / msz / 1e6, 3), dev)
    res[name] = r
print(json.dumps(res))
