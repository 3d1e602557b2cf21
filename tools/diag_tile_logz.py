"""Where does the tile kernel's pht_evaluate_log Jz differ from the oracle (term-sum metric)?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2111_14317_b200 as P, workloads as W, oracle
np.seterr(all="ignore")
for name, sysm, rho, tl in [("cyclic-5", W.cyclic(5, lift_max=100), 300.0, -8.0), ("noon-10", W.noon(10, lift_max=10000), 100.0, -5.0)]:
    n = sysm.n
    xm, xe, tm, te, z, tau = W.random_extended_points(64, n, seed=17, rho_max=rho, tau_lo=tl)
    o = oracle.Oracle(sysm).evaluate_x(xm, xe, tm, te)
    lx = np.log2(np.abs(xm)) + xe
    for fam in ("tile", "dense"):
        g = P.System.from_workload(sysm).set_kernels(fam)
        H, J, T, e2, st = [a.cpu().numpy() for a in g.evaluate_log(torch.from_numpy(z).cuda(), torch.from_numpy(tau).cuda())]
        ls = o["LSJx"] + lx[:, None, :]
        lsh = o["LSH"][:, :, None]
        ls_eff = np.maximum(ls, lsh - 960)
        got = J * np.exp2(e2[:, :, None] - ls_eff)
        ref = o["Jxm"] * xm[:, None, :] * np.exp2(o["Jxe"] + xe[:, None, :] - ls_eff)
        err = np.where(np.isneginf(ls), 0, np.abs(got - ref))
        idx = np.argwhere(err > 1e-10)
        print(name, fam, "bad", len(idx))
        for q, k, j in idx[:6]:
            print("  q k j", q, k, j, "gpu", J[q, k, j], "e2", e2[q, k], "ref m", o["Jxm"][q, k, j] * xm[q, j], "ref e", o["Jxe"][q, k, j] + xe[q, j],
                  "ls", ls[q, k, j], "lsh", o["LSH"][q, k], "H gpu", H[q, k], "Hm", o["Hm"][q, k], "He", o["He"][q, k])
