"""Small launches of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck):
k_stepw (step, directions, evaluation), k_evalw (TMA stores, ragged), k_dense, tile kernels
(k_phte, k_pht, k_track), k_trackw (LPR 1 and 2), the compensated final refinement, the
specialised (NVRTC) kernels, projective and QR paths."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_14317_b200 as P  # noqa: E402
import workloads as W  # noqa: E402
from workloads import startsys as SS  # noqa: E402

c = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
for name, sysm in (("cyclic-5", W.cyclic(5, lift_max=100)), ("cyclic-10", W.cyclic(10, lift_max=100)),
                   ("katsura-10", W.katsura(10, lift_max=100)), ("random-12x20", W.random_dense(12, 20))):
    n = sysm.n
    x, t, tau = W.random_points(333, n, seed=1, tau_lo=-0.05, rho_max=0.5)
    for fam in ("auto", "warp", "tile", "lane", "dense"):
        g = P.System.from_workload(sysm).set_kernels(fam)
        g.evaluate(c(x), c(t))
        g.evaluate(c(x), c(t), scaled=True)
        g.evaluate_log(c(np.log(x)), c(tau))
        g.euler_newton(c(x), c(t))
        xd, td = c(x), c(tau)
        g.pc_step(xd, td, c(np.full(333, 0.01)), 2)
    torch.cuda.synchronize()
    print(name, "evaluate/directions/step ok", flush=True)
for name, L in (("cyclic-5", 100), ("noon-5", 1000)):
    s = W.cyclic(5, lift_max=L) if name == "cyclic-5" else W.noon(5, lift_max=L)
    cells = SS.mixed_cells_fast(s)
    Wc = SS.cell_lifts(s, cells)
    w0, tau0, cid = SS.start_points_cells(s, cells)
    for fam in ("auto", "tile"):
        g = P.System.from_workload(s).set_kernels(fam)
        st, _ = g.track_cells(c(w0), c(tau0), c(Wc), c(cid))
        print(name, fam, "track_cells finite", int((st == 0).sum()), "of", len(w0), flush=True)
    g = P.System.from_workload(s).specialize().set_kernels("specialized")
    st, _ = g.track_cells(c(w0), c(tau0), c(Wc), c(cid))
    g.evaluate(c(np.exp(w0[:, :])), c(np.ones(len(w0))))
    print(name, "specialised ok", int((st == 0).sum()), flush=True)
s = W.cyclic(5, lift_max=100)
gq = P.System.from_workload(s).set_solver("qr")
x, t, tau = W.random_points(100, 5, seed=2, tau_lo=-0.05)
gq.euler_newton(c(x), c(t))
gp = P.System.from_workload(s, projective=True)
y = gp.homogenize(c(x))
gp.euler_newton(y, c(t))
torch.cuda.synchronize()
print("qr / projective ok")
