"""Multi-GPU sharding of independent ciphertexts.

The encrypted KAN path has no exchange inside an inference: one sample is one
ciphertext through the whole pipeline (reference: a sequential per-input loop,
/root/reference/pkg/src/hekan/inference.py:336-351; concurrency across inputs
is allowed). A global batch of n samples is split into contiguous
blocks, one per rank (one process per GPU; torch.distributed over NCCL on
NVLink, gloo for the CPU tests):

* every rank builds its backend from ONE shared seed (`shared_seed`: drawn
  from the OS CSPRNG on rank 0 and broadcast), so evaluation keys are
  identical everywhere and rank 0 can decrypt every rank's output;
* each rank encrypts its block with `sample_offset` = its first global sample
  index: encryption randomness is indexed by global sample, so no (a, e) pair
  repeats across ranks and the shards are bit-identical to the same samples
  encrypted by one process;
* the only collective is `gather_ciphertexts`: one gather of the level-0
  output ciphertexts (2 limbs per sample) to rank 0, reassembled in global
  sample order.
"""

from __future__ import annotations

import numpy as np


def block_range(n: int, rank: int, world: int) -> tuple:
    """[start, stop) of the samples `rank` owns; n must divide evenly."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    if n % world:
        raise ValueError(f"global batch {n} does not split evenly over {world} ranks")
    per = n // world
    return rank * per, (rank + 1) * per


def shard_rows(x: np.ndarray, rank: int, world: int) -> np.ndarray:
    lo, hi = block_range(len(x), rank, world)
    return np.asarray(x)[lo:hi]


def shared_seed(world: int, rank: int, device=None) -> int:
    """A 63-bit key seed from rank 0's CSPRNG, broadcast to every rank."""
    import secrets

    seed = secrets.randbits(63)
    if world == 1:
        return seed
    import torch
    import torch.distributed as dist

    t = torch.tensor([seed if rank == 0 else 0], dtype=torch.int64, device=device)
    dist.broadcast(t, src=0)
    return int(t.item())


def _as_tensor(buf):
    import torch

    return buf if torch.is_tensor(buf) else torch.from_numpy(np.asarray(buf).view(np.int64))


def gather_ciphertexts(be, ct, world: int, rank: int, group=None):
    """Gather every rank's ciphertext block (same level and batch on every
    rank) to rank 0 as ONE batched ciphertext of rank 0's backend, samples in
    global order. NCCL moves device buffers over NVLink; gloo moves host
    buffers (the oracle engine). Returns None on ranks != 0."""
    if world == 1:
        return ct
    import torch
    import torch.distributed as dist

    shape = (2, ct.level + 1, ct.batch, be.n)
    mine = _as_tensor(ct.data).reshape(shape).contiguous()
    bufs = [torch.empty_like(mine) for _ in range(world)] if rank == 0 else None
    dist.gather(mine, gather_list=bufs, dst=0, group=group)
    if rank != 0:
        return None
    full = torch.cat(bufs, dim=2).reshape(-1)
    data = full if torch.is_tensor(ct.data) else full.numpy().view(np.uint64)
    return be.adopt(data, ct.level, world * ct.batch)
