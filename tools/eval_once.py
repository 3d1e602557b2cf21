"""One pht_evaluate launch (for ncu captures): argv[1] = system, PHT_SPEC=1 specialises."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_14317_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cyclic-10"
sysm = {"cyclic-10": lambda: W.cyclic(10, lift_max=100), "random-20x50": lambda: W.random_dense(20, 50),
        "cyclic-5": lambda: W.cyclic(5)}[name]()
g = P.System.from_workload(sysm)
if os.environ.get("PHT_SPEC") == "1":
    g.specialize()
p = 1 << 21 if sysm.n <= 10 else 1 << 20   # the bench.py evaluation sizes
x, t, _ = W.random_points(p, sysm.n, seed=1, rho_max=0.5 if sysm.n > 12 else 1.0)
xd, td = torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda()
for _ in range(2):
    g.evaluate(xd, td)
torch.cuda.synchronize()
print("ok")
