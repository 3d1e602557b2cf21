"""C4 (random dense n = 20, 50 terms per equation) pht_evaluate throughput on the DMMA path,
2^20 device-resident points, CUDA events (A/B of k_dense variants: PHT_LIB=...)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_14317_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

p = int(os.environ.get("PHT_DENSE_P", 1 << 20))
reps = int(os.environ.get("PHT_REPS", 5))
sysm = W.random_dense(20, 50)
g = P.System.from_workload(sysm)
x, t, _ = W.random_points(p, sysm.n, seed=1, rho_max=0.5)
xd, td = torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda()
n = sysm.n
H = torch.empty((p, n), dtype=torch.complex128, device="cuda")
Jx = torch.empty((p, n, n), dtype=torch.complex128, device="cuda")
Jt = torch.empty((p, n), dtype=torch.complex128, device="cuda")
st = torch.empty((p,), dtype=torch.uint8, device="cuda")
for _ in range(2):
    g.evaluate(xd, td, out=(H, Jx, Jt, st))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    g.evaluate(xd, td, out=(H, Jx, Jt, st))
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(json.dumps({"points": p, "ms": ms, "Mpoints_per_s": p / ms / 1e3, "kernels": g.kernels}))
