"""Multi-GPU plumbing: one process per GPU, chains sharded by
global chain id, reductions as ordered sums over global ids.

Chains are independent, so the data path has no collective: every rank runs
its contiguous global-id range [begin, end) (the Philox counters are keyed by
global chain id, so a chain's trajectory does not depend on the GPU count).
The estimators' exchange steps (per-phase counts, pilot quantiles, warm-start
resampling, moment and f-value sums) go through ONE primitive: an allgather
of equal host shards in rank order, installed into the library with
``spec_set_comm`` and implemented here over ``torch.distributed`` (NCCL on
GPU boxes, gloo for the CPU tests).  The library takes every sum in global
order (csrc/specwalk.cu: walk_entry, volume, expectation), so results are
bit-identical for 1, 2, 4 or 8 GPUs.  This module holds no arithmetic of the
method: only shard ranges and the transport.
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple

import numpy as np


def shard_range(total: int, rank: int, world: int, align: int = 1) -> Tuple[int, int]:
    """Contiguous global-id range of `rank` (equal shards; total % (world*align) == 0)."""
    if total % (world * align):
        raise ValueError(f"{total} chains do not split into {world} shards of multiples of {align}")
    per = total // world
    return rank * per, (rank + 1) * per


def make_allgather(group=None, device: Optional[str] = None) -> Callable[[np.ndarray], np.ndarray]:
    """allgather(local) -> concatenation of every rank's equal-length shard, rank order."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    if device is None and dist.get_backend(group) == "nccl":
        device = f"cuda:{torch.cuda.current_device()}"  # NCCL moves CUDA tensors only

    def allgather(local: np.ndarray) -> np.ndarray:
        t = torch.from_numpy(np.ascontiguousarray(local, dtype=np.float64))
        if device is not None:
            t = t.to(device)
        out = torch.empty(world * t.numel(), dtype=torch.float64, device=t.device)
        dist.all_gather_into_tensor(out, t, group=group)
        return out.cpu().numpy()

    return allgather


def attach(spectrahedron, group=None, device: Optional[str] = None) -> None:
    """Install the torch.distributed allgather into a Spectrahedron context."""
    import torch.distributed as dist

    spectrahedron.set_comm(make_allgather(group, device), dist.get_rank(group), dist.get_world_size(group))


def distributed_walk_sample(spectrahedron, chains: int, steps: int, L: float, rho: int, seed: int, kind: int = 0,
                            T: float = 1.0, group=None) -> dict:
    """Sharded walk_sample: this rank runs its contiguous global-id range (no collective in
    the data path); the library reduces the end-point moments over ranks through the
    allgather installed by attach() (sums in global chunk order, identical on every rank).
    Shards must be multiples of 1024 chains (the library's moment chunk)."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    begin, end = shard_range(chains, rank, world, 1024)
    return spectrahedron.walk_sample(end - begin, steps, L, rho, seed, kind=kind, chain_begin=begin, T=T)
