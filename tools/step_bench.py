"""pc_step throughput (K=1, M evals/s = 2 x points x steps / s) on several systems, one GPU."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_14317_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

res = {}
for name, sysm, p in [("cyclic-5", W.cyclic(5, lift_max=100), 1 << 22), ("cyclic-10", W.cyclic(10, lift_max=100), 1 << 22),
                      ("katsura-10", W.katsura(10, lift_max=100), 1 << 21), ("noon-10", W.noon(10, lift_max=100), 1 << 22),
                      ("cyclic-14", W.cyclic(14, lift_max=100), 1 << 20)]:
    g = P.System.from_workload(sysm)
    x, t, _ = W.random_points(p, sysm.n, seed=5, tau_lo=-0.05)
    x0 = torch.from_numpy(x).cuda()
    tau0 = torch.log(torch.from_numpy(t)).cuda()
    dt = torch.full((p,), 1e-3, dtype=torch.float64, device="cuda")
    xd, tau = x0.clone(), tau0.clone()
    for _ in range(2):
        g.pc_step(xd, tau, dt, 1)
    reps = 5
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.pc_step(xd, tau, dt, 1)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    res[name] = round(2 * p / ms / 1e3, 1)
print(json.dumps(res))
