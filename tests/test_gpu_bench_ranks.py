"""The multi-rank bench flow on real hardware: `bench.py --gpus 2`
spawns two ranks, each steps its own shard of points and tracks its shard of the katsura-10 start
paths, the per-rank kernel times are maxed, and the ONE packed gather brings every endpoint and
status to rank 0, which prints one line.  The GPU boxes of this build have one B200, so both ranks
run on cuda:0 with gloo carrying the collectives (bench.py's test-only --dist-backend gloo
--all-on-device0): the ranks' kernels are independent and never wait on each other, so this
exercises the N > 1 code path, not a scaling number."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_shard_and_gather():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "1",
                        "--points", "65536", "--e2e-steps", "1", "--tracking", "katsura-10", "--no-evaluation",
                        "--no-paper-protocol", "--no-cpu-baseline", "--dist-backend", "gloo", "--all-on-device0"],
                       capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak"
    assert d["value"] > 0 and d["gpu_launches"] > 0
    k = d["tracking"]["katsura-10"]
    # every one of the 990 paths gathered on rank 0 with the oracle's status (all finite)
    assert k["paths"] == 990 and k["finite"] == 990, k
    assert len(k["per_rank_kernel_ms"]) == 2 and k["imbalance"] >= 1.0
