"""Multi-GPU path sharding (reading R20).

Paths are independent ("pleasantly parallel"), and the paper's constraint (c) is to
"minimize communication between devices".  So each rank (one process per GPU) tracks its
own shard of the start points with no communication, and ONE gather at the end collects the
endpoints, statuses and statistics on rank 0.

* `shard_indices`: a seeded permutation of the path indices (so paths of the same mixed cell,
  which have similar lengths, spread over the ranks), cut into `world` contiguous blocks whose
  sizes differ by at most one.
* `gather_to_rank0`: pads each rank's block to the common size, one `all_gather_into_tensor` per
  result tensor (NCCL over NVLink on GPUs, gloo on CPU), and rank 0 restores the original path
  order.  Works with CPU tensors (gloo) and CUDA tensors (nccl) alike.
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


def gather_to_rank0(local: dict, indices: np.ndarray, n_paths: int, group=None) -> dict | None:
    """Gather per-path result tensors (first dim = this rank's paths, in `indices` order) to rank 0.

    Returns on rank 0 a dict of tensors with first dim n_paths in the original path order,
    None elsewhere.  One all_gather per tensor; the padding rows carry index -1.
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    B = block_size(n_paths, world)
    any_t = next(iter(local.values()))
    dev = any_t.device
    idx = torch.full((B,), -1, dtype=torch.int64, device=dev)
    idx[:len(indices)] = torch.as_tensor(indices, dtype=torch.int64, device=dev)
    all_idx = torch.empty((world * B,), dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(all_idx, idx, group=group)
    out = {}
    for name, t in local.items():
        if t.shape[0] != len(indices):
            raise ValueError(f"{name}: first dim {t.shape[0]} != {len(indices)} local paths")
        pad = torch.zeros((B,) + tuple(t.shape[1:]), dtype=t.dtype, device=dev)
        pad[:t.shape[0]] = t
        if t.is_complex():  # gloo/nccl all_gather on complex: go through a real view
            pad_r = torch.view_as_real(pad).contiguous()
            buf = torch.empty((world * B,) + tuple(pad_r.shape[1:]), dtype=pad_r.dtype, device=dev)
            dist.all_gather_into_tensor(buf, pad_r, group=group)
            buf = torch.view_as_complex(buf)
        else:
            buf = torch.empty((world * B,) + tuple(t.shape[1:]), dtype=t.dtype, device=dev)
            dist.all_gather_into_tensor(buf, pad.contiguous(), group=group)
        out[name] = buf
    if rank != 0:
        return None
    keep = all_idx >= 0
    order = all_idx[keep]
    res = {}
    for name, buf in out.items():
        full = torch.empty((n_paths,) + tuple(buf.shape[1:]), dtype=buf.dtype, device=dev)
        full[order] = buf[keep]
        res[name] = full
    return res
