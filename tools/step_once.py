"""One pc_step launch on cyclic-10 (for ncu captures); PHT_SPEC=1 uses the specialised kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_14317_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cyclic-10"
sysm = {"cyclic-10": lambda: W.cyclic(10, lift_max=100), "katsura-10": lambda: W.katsura(10, lift_max=100),
        "noon-10": lambda: W.noon(10, lift_max=100), "cyclic-5": lambda: W.cyclic(5, lift_max=100)}[name]()
g = P.System.from_workload(sysm)
if os.environ.get("PHT_SPEC") == "1":
    g.specialize()
p = 1 << 20
x, t, _ = W.random_points(p, sysm.n, seed=5, tau_lo=-0.05)
xd = torch.from_numpy(x).cuda()
tau = torch.log(torch.from_numpy(t)).cuda()
dt = torch.full((p,), 1e-3, dtype=torch.float64, device="cuda")
for _ in range(2):
    g.pc_step(xd, tau, dt, 1)
torch.cuda.synchronize()
print("ok")
