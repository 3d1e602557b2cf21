"""Compute and store the mixed cells of a benchmark system (workload preparation).

    python -m workloads.make_starts katsura-10|cyclic-10|noon-10|cyclic-5 [lift_max]

Writes workloads/data/<name>_L<lift_max>.npz with the cells (term-id pairs, alpha, gap,
volume).  The system itself is regenerated deterministically from (name, lift_max, seed);
start points are derived from the cells at load time (workloads.startsys.load_start_points).
"""
import sys
import time

import numpy as np

from . import systems as S
from . import startsys as SS

CONFIGS = {
    "cyclic-5": lambda L: S.cyclic(5, lift_max=L),
    "cyclic-10": lambda L: S.cyclic(10, lift_max=L),
    "katsura-10": lambda L: S.katsura(10, lift_max=L),
    "noon-10": lambda L: S.noon(10, lift_max=L),
}


def main():
    name = sys.argv[1]
    L = int(sys.argv[2]) if len(sys.argv) > 2 else 10_000
    sysm = CONFIGS[name](L)
    t0 = time.time()
    cells = SS.mixed_cells_fast(sysm)
    dt = time.time() - t0
    n = sysm.n
    pairs = np.array([c["pairs"] for c in cells], np.int32).reshape(len(cells), n, 2)
    alpha_num = np.array([[a.numerator for a in c["alpha"]] for c in cells], dtype=object)
    alpha_den = np.array([[a.denominator for a in c["alpha"]] for c in cells], dtype=object)
    gap = np.array([float(c["gap"]) for c in cells])
    vol = np.array([c["volume"] for c in cells], np.int64)
    out = f"{SS.DATA_DIR}/{name}_L{L}.npz"
    np.savez_compressed(out, pairs=pairs, alpha=np.array([[float(a) for a in c["alpha"]] for c in cells]),
                        alpha_num=alpha_num.astype(str), alpha_den=alpha_den.astype(str), gap=gap, volume=vol,
                        lift_max=L, seconds=dt, stats=SS.mixed_cells_fast.last_stats)
    print(f"{name} L={L}: {len(cells)} cells, mixed volume {int(vol.sum())}, {dt:.1f} s -> {out}", flush=True)


if __name__ == "__main__":
    main()
