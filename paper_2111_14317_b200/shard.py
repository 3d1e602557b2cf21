"""Multi-GPU path sharding (reading R20).

Paths are independent ("pleasantly parallel"), and the paper's constraint (c) is to
"minimize communication between devices".  So each rank (one process per GPU) tracks its
own shard of the start points with no communication, and ONE gather at the end collects the
endpoints, statuses and statistics on rank 0.

* `shard_indices`: a seeded permutation of the path indices (so paths of the same mixed cell,
  which have similar lengths, spread over the ranks), cut into `world` contiguous blocks whose
  sizes differ by at most one.
* `gather_to_rank0`: packs every per-path result of this rank (path index, endpoint re/im,
  status, statistics) into ONE float64 row per path, pads the block to the common size and runs
  exactly ONE `all_gather_into_tensor` (NCCL over NVLink on GPUs, gloo on CPU); rank 0 unpacks
  and restores the original path order.  Integers travel as float64 (exact below 2^53).
  Works with CPU tensors (gloo) and CUDA tensors (nccl) alike.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def shard_indices(n_paths: int, rank: int, world: int, seed: int = 0) -> np.ndarray:
    """Path indices owned by `rank` (a permutation block; blocks partition range(n_paths))."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    perm = np.random.Generator(np.random.PCG64(seed)).permutation(n_paths)
    base, extra = divmod(n_paths, world)
    start = rank * base + min(rank, extra)
    size = base + (1 if rank < extra else 0)
    return perm[start:start + size]


def block_size(n_paths: int, world: int) -> int:
    return -(-n_paths // world)


def _columns(t: torch.Tensor) -> int:
    """float64 columns one path's entry of t occupies in the packed row."""
    per = 1
    for d in t.shape[1:]:
        per *= int(d)
    return per * (2 if t.is_complex() else 1)


def gather_to_rank0(local: dict, indices: np.ndarray, n_paths: int, group=None) -> dict | None:
    """Gather per-path result tensors (first dim = this rank's paths, in `indices` order) to rank 0
    with ONE collective (minimise communication between devices).

    Row layout (float64): [path index | each tensor's entries, complex as (re, im) pairs, integers
    converted exactly].  Returns on rank 0 a dict of tensors with first dim n_paths in the
    original path order and the original dtypes; None elsewhere.  Padding rows carry index -1.
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    B = block_size(n_paths, world)
    any_t = next(iter(local.values()))
    dev = any_t.device
    names = list(local)
    cols = [_columns(local[k]) for k in names]
    width = 1 + sum(cols)
    row = torch.zeros((B, width), dtype=torch.float64, device=dev)
    row[:, 0] = -1.0
    m = len(indices)
    row[:m, 0] = torch.as_tensor(indices, dtype=torch.float64, device=dev)
    c = 1
    for k, w in zip(names, cols):
        t = local[k]
        if t.shape[0] != m:
            raise ValueError(f"{k}: first dim {t.shape[0]} != {m} local paths")
        # (integer results -- statuses, step counts -- are far below 2^53; not checked on the device,
        # which would synchronise inside the caller's timed region)
        v = torch.view_as_real(t.contiguous()) if t.is_complex() else t
        row[:m, c:c + w] = v.reshape(m, w).to(torch.float64)
        c += w
    buf = torch.empty((world * B, width), dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(buf, row, group=group)          # the one collective
    if rank != 0:
        return None
    keep = buf[:, 0] >= 0
    order = buf[keep, 0].to(torch.int64)
    data = buf[keep]
    res = {}
    c = 1
    for k, w in zip(names, cols):
        t = local[k]
        part = data[:, c:c + w]
        c += w
        full = torch.empty((n_paths, w), dtype=torch.float64, device=dev)
        full[order] = part
        if t.is_complex():
            out = torch.view_as_complex(full.reshape((n_paths,) + tuple(t.shape[1:]) + (2,)).contiguous())
            res[k] = out.to(t.dtype)
        else:
            res[k] = full.reshape((n_paths,) + tuple(t.shape[1:])).to(t.dtype)
    return res
