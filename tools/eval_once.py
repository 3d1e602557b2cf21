"""One pht_evaluate launch on cyclic-10 (for ncu captures of the standalone evaluation kernel)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_14317_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
sysm = W.cyclic(10, lift_max=100)
g = P.System.from_workload(sysm)
x, t, _ = W.random_points(p, 10, seed=1)
out = g.evaluate(torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda())
torch.cuda.synchronize()
print("ok", p)
