"""Standalone pht_evaluate throughput on several configs (device-resident, CUDA events)."""
import json
import time
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_14317_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

res = {}
for name, sysm, p in [("cyclic-5", W.cyclic(5), 1 << 22), ("cyclic-10", W.cyclic(10, lift_max=100), 1 << 21),
                      ("katsura-10", W.katsura(10, lift_max=100), 1 << 21), ("noon-10", W.noon(10, lift_max=100), 1 << 21),
                      ("random-20x50", W.random_dense(20, 50), 1 << 18)]:
    g = P.System.from_workload(sysm)
    if os.environ.get("PHT_SPEC") == "1" and sysm.offsets[-1] <= 256:
        t1 = time.time(); g.specialize(); print(json.dumps({"specialize_s": time.time() - t1}), file=sys.stderr)
    x, t, _ = W.random_points(p, sysm.n, seed=1, rho_max=0.5 if sysm.n > 12 else 1.0)
    xd, td = torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda()
    for _ in range(3):
        out = g.evaluate(xd, td)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    reps = 5
    for _ in range(reps):
        out = g.evaluate(xd, td)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    n = sysm.n
    byts = p * (16 * (n + 2 * n + n * n) + 8 + 1)
    res[name] = {"points": p, "ms": ms, "Gevals_per_s": p / ms / 1e6, "GB_per_s": byts / ms / 1e6}
    del out, xd, td, g
print(json.dumps(res))
