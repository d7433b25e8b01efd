"""Multi-GPU sharding of independent ciphertexts.

The encrypted KAN path has no exchange inside an inference: one sample is one
ciphertext through the whole pipeline. A job of B samples is split
round-robin over the ranks (one process per GPU, torch.distributed over NCCL
on NVLink / gloo on CPU for tests); evaluation keys are generated per rank
from the same seed (identical material, no broadcast needed), and the only
collective is one gather of the level-0 output ciphertexts to rank 0.
"""

from __future__ import annotations

import numpy as np


def shard_indices(n: int, rank: int, world: int) -> np.ndarray:
    """Round-robin sample indices owned by `rank` (SURVEY §8e partitioning)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    return np.arange(rank, n, world)


def shard_rows(x: np.ndarray, rank: int, world: int) -> np.ndarray:
    return np.asarray(x)[shard_indices(len(x), rank, world)]


def unshard_rows(parts, n: int) -> np.ndarray:
    """Inverse of shard_rows: parts[r] holds rows rank r owns."""
    world = len(parts)
    first = np.asarray(parts[0])
    out = np.empty((n,) + first.shape[1:], dtype=first.dtype)
    for r, part in enumerate(parts):
        out[shard_indices(n, r, world)] = part
    return out


def gather_to_root(tensor, world: int, rank: int, group=None):
    """Gather equally shaped per-rank tensors to rank 0 (NCCL: NVLink peer
    transfers of the output ciphertext limbs). Returns the list on rank 0."""
    import torch.distributed as dist

    if world == 1:
        return [tensor]
    bufs = [tensor.new_empty(tensor.shape) for _ in range(world)] if rank == 0 else None
    dist.gather(tensor, gather_list=bufs, dst=0, group=group)
    return bufs
