"""Generic vs system-specialised kernels (pht_system_specialize): output agreement on seeded
points and pc_step throughput; prints one JSON object per system."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_14317_b200 as P  # noqa: E402
import workloads as W  # noqa: E402


def rel(a, b):
    a, b = a.reshape(a.shape[0], -1), b.reshape(b.shape[0], -1)
    return float(((a - b).abs().amax(1) / b.abs().amax(1).clamp_min(1e-300)).max())


def step_rate(g, x, tau, dt, reps=10):
    xs, ts = x.clone(), tau.clone()
    g.pc_step(xs, ts, dt, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        xs.copy_(x); ts.copy_(tau)
        g.pc_step(xs, ts, dt, 1)
    e1.record()
    torch.cuda.synchronize()
    return x.shape[0] * 2 / (e0.elapsed_time(e1) / reps) / 1e6  # evals (2 per step) per us = G/s ... M/ms


which = sys.argv[1:] or ["cyclic-5", "cyclic-10", "katsura-10", "noon-10"]
mk = {"cyclic-5": lambda: W.cyclic(5, lift_max=100), "cyclic-10": lambda: W.cyclic(10, lift_max=100),
      "katsura-10": lambda: W.katsura(10, lift_max=100), "noon-10": lambda: W.noon(10, lift_max=100),
      "chandra-6": lambda: W.chandra(6, lift_max=100)}
for name in which:
    sysm = mk[name]()
    out = {}
    g0 = P.System.from_workload(sysm)
    g1 = P.System.from_workload(sysm)
    t0 = time.time()
    g1.specialize()
    out["specialize_s"] = time.time() - t0
    n, p = sysm.n, 1 << 16
    x, t, _ = W.random_points(p, n, seed=3)
    xd, td = torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda()
    a, b = g0.evaluate(xd, td), g1.evaluate(xd, td)
    out["eval_rel"] = [rel(a[i], b[i]) for i in range(3)]
    out["eval_status_eq"] = bool((a[3] == b[3]).all())
    xs, ts, _ = W.random_points(p, n, seed=4, tau_lo=-0.05)
    xd, td = torch.from_numpy(xs).cuda(), torch.from_numpy(ts).cuda()
    a, b = g0.euler_newton(xd, td), g1.euler_newton(xd, td)
    ok = (a[2] == 0) & (b[2] == 0)
    out["dirs_rel"] = [rel(a[i][ok], b[i][ok]) for i in range(2)]
    out["dirs_status_eq"] = float((a[2] == b[2]).float().mean())
    P_ = 1 << 22
    x, t, _ = W.random_points(P_, n, seed=5, tau_lo=-0.05)
    xd = torch.from_numpy(x).cuda()
    tau = torch.log(torch.from_numpy(t)).cuda()
    dt = torch.full((P_,), 1e-3, dtype=torch.float64, device="cuda")
    x0, t0_ = xd.clone(), tau.clone()
    x1, t1_ = xd.clone(), tau.clone()
    s0, _ = g0.pc_step(x0, t0_, dt, 1)
    s1, _ = g1.pc_step(x1, t1_, dt, 1)
    ok = (s0 == 0) & (s1 == 0)
    out["step_rel"] = rel(x1[ok], x0[ok])
    out["step_Mevals_per_s"] = {"generic": step_rate(g0, xd, tau, dt) * 1e3, "specialized": step_rate(g1, xd, tau, dt) * 1e3}
    print(json.dumps({name: out}), flush=True)
    del g0, g1
