"""Multi-GPU host logic on CPU: path sharding index math and the end-of-run gather (world size 2,
gloo backend, 127.0.0.1 rendezvous)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2111_14317_b200.shard import block_size, gather_to_rank0, shard_indices


@pytest.mark.parametrize("n,world", [(1, 1), (7, 2), (70, 3), (35940, 8), (5, 8)])
def test_shards_partition_the_paths(n, world):
    parts = [shard_indices(n, r, world, seed=3) for r in range(world)]
    allidx = np.concatenate(parts)
    assert sorted(allidx.tolist()) == list(range(n))
    sizes = [len(p) for p in parts]
    assert max(sizes) - min(sizes) <= 1 and max(sizes) <= block_size(n, world)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    idx = shard_indices(n, rank, world, seed=5)
    # fake per-path results that encode the path index
    x = torch.tensor([[complex(i, -i), complex(2 * i, 1)] for i in idx], dtype=torch.complex128).reshape(-1, 2)
    st = torch.tensor([i % 7 for i in idx], dtype=torch.uint8)
    stats = torch.tensor([[i, 2 * i, 3 * i, 4] for i in idx], dtype=torch.int64).reshape(-1, 4)
    calls = []
    orig = dist.all_gather_into_tensor
    dist.all_gather_into_tensor = lambda *a, **k: (calls.append(1), orig(*a, **k))[1]
    try:
        out = gather_to_rank0({"x": x, "status": st, "stats": stats}, idx, n)
    finally:
        dist.all_gather_into_tensor = orig
    assert len(calls) == 1          # exactly one collective
    if rank == 0:
        ok = (torch.equal(out["x"][:, 0].real, torch.arange(n, dtype=torch.float64))
              and torch.equal(out["status"], torch.tensor([i % 7 for i in range(n)], dtype=torch.uint8))
              and torch.equal(out["stats"][:, 1], 2 * torch.arange(n))
              and out["x"].dtype == torch.complex128 and out["status"].dtype == torch.uint8
              and torch.equal(out["x"][:, 1].imag, torch.ones(n, dtype=torch.float64)))
        q.put(bool(ok))
    else:
        assert out is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [11, 1000])
def test_gather_world2_gloo(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=10) is True


def test_bench_spawns_ranks_for_gpus_n():
    """`bench.py --gpus 2` without a torchrun environment starts 2 ranks itself (the driver's
    command line works unchanged for N = 1..8); rank 0 alone prints ONE JSON line.  Driven through
    the reference arm, which runs on CPU (the oracle), so the bootstrap is exercised here."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0", "--ref-points", "64"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2


def test_bench_refuses_world_size_mismatch():
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0", "--ref-points", "64"],
                       capture_output=True, text=True, timeout=120, env=env)
    assert r.returncode == 2 and "WORLD_SIZE" in r.stdout
