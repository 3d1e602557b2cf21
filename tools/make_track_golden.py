"""Oracle-tracked golden endpoints of EVERY start path (VERDICT r1 "next" 1(iii)).

    python tools/make_track_golden.py [katsura-10 cyclic-10 noon-10]

For each benchmark system this runs the CPU oracle's extended-range tracker (oracle.c
orc_track_x, cell coordinates, the pht_track_opts defaults) on all start paths and stores, under
tests/golden/track_<name>.npz:
  status   uint8 [P]       the oracle's per-path status (0 = finite, ledger A24)
  xm, xe   [P, n]          endpoint x = xm * 2**xe (complex128 mantissa, int exponent)
  stats    int32 [P, 4]    accepted steps, rejected steps, evaluations, final iterations
and a small JSON summary (counts, threads, seconds).  Inputs come from workloads/ (the stored
mixed cells); nothing here touches the CUDA path (task rule 3: every expected value is written
by a committed script that calls only oracle/).  Takes ~12 minutes on 8 cores.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from workloads import startsys as SS  # noqa: E402
from workloads.make_starts import CONFIGS  # noqa: E402

LIFT = {"katsura-10": 10_000, "noon-10": 10_000, "cyclic-10": 1_000_000}
GOLDEN = os.path.join(ROOT, "tests", "golden")


def main(names):
    nt = oracle.set_threads(0)
    for name in names:
        L = LIFT[name]
        s = CONFIGS[name](L)
        cells = SS.load_cells(name, L)
        Wc = SS.cell_lifts_fast(s, cells)
        w0, tau0, cid = SS.start_points_cells(s, cells)
        m, e = oracle.z_to_x(w0)   # test plumbing: the oracle takes x = m 2^e, never log/exp of points
        t0 = time.time()
        xm, xe, tau, st, stats = oracle.Oracle(s).track_x(m, e, tau0, cell_lift=Wc, path_cell=cid)
        sec = time.time() - t0
        out = os.path.join(GOLDEN, f"track_{name}.npz")
        np.savez_compressed(out, status=st.astype(np.uint8), xm=xm, xe=xe.astype(np.int32),
                            stats=stats.astype(np.int32), lift_max=L)
        summ = dict(system=name, lift_max=L, paths=int(len(st)), finite=int((st == 0).sum()),
                    status_counts={int(k): int(v) for k, v in zip(*np.unique(st, return_counts=True))},
                    evals=int(stats[:, 2].sum()), threads=nt, seconds=round(sec, 1),
                    script="tools/make_track_golden.py (oracle.c orc_track_x, default options)")
        with open(os.path.join(GOLDEN, f"track_{name}.json"), "w") as f:
            json.dump(summ, f, indent=1)
        print(json.dumps(summ), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["katsura-10", "cyclic-10", "noon-10"])
