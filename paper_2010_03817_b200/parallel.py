"""Multi-GPU plumbing: one process per GPU, chains sharded by
global chain id, reductions as ordered sums over global ids.

Chains are independent, so the data path has no collective: every rank runs
its contiguous global-id range [begin, end) (the Philox counters are keyed by
global chain id, so a chain's trajectory does not depend on the GPU count).
The estimators' exchange steps (per-phase counts, pilot quantiles, warm-start
resampling, moment and f-value sums) go through ONE primitive: an allgather
of equal host shards in rank order, installed into the library with
``spec_set_comm`` and implemented here over ``torch.distributed`` (NCCL on
GPU boxes, gloo for the CPU tests).  Sums are then taken in global order, so
results are bit-identical for 1, 2, 4 or 8 GPUs.
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


def ordered_sum(parts: np.ndarray, nshards: int) -> np.ndarray:
    """Sum equal shards of `parts` (rank order) sequentially: (((p0 + p1) + p2) + ...)."""
    parts = np.asarray(parts).reshape(nshards, -1)
    acc = parts[0].copy()
    for k in range(1, nshards):
        acc = acc + parts[k]
    return acc


def chunk_moments(X: np.ndarray, chunk: int) -> np.ndarray:
    """Per-chunk end-point moments (sum x, packed lower sum x x^T), chunks of `chunk`
    consecutive global chain ids -- the layout of the library's moments_chunk_kernel."""
    n = X.shape[1]
    il = np.tril_indices(n)
    out = []
    for k in range(0, X.shape[0], chunk):
        Y = X[k:k + chunk]
        s = np.zeros(n)
        ss = np.zeros(len(il[0]))
        for row in Y:  # chain order
            s = s + row
            ss = ss + np.outer(row, row)[il]
        out.append(np.concatenate([s, ss]))
    return np.concatenate(out)


def reduce_chunked_moments(local_chunks: np.ndarray, n: int, allgather) -> Tuple[np.ndarray, np.ndarray]:
    """Gather every rank's chunk partials and add them in global chunk order."""
    stride = n + n * (n + 1) // 2
    allc = np.asarray(allgather(local_chunks)).reshape(-1, stride)
    acc = allc[0].copy()
    for k in range(1, allc.shape[0]):
        acc = acc + allc[k]
    return acc[:n], acc[n:]


def attach(spectrahedron, group=None, device: Optional[str] = None) -> None:
    """Install the torch.distributed allgather into a Spectrahedron context."""
    import torch.distributed as dist

    spectrahedron.set_comm(make_allgather(group, device), dist.get_rank(group), dist.get_world_size(group))


def distributed_walk_moments(spectrahedron, chains: int, steps: int, L: float, rho: int, seed: int,
                             kind: int = 0, T: float = 1.0, chunk: int = 1024, group=None):
    """Sharded walk (no collective in the data path) + deterministic moments of the
    end points: each rank walks its global-id range, computes chunk partials in
    chain order, and the partials are summed in global chunk order on every rank."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    begin, end = shard_range(chains, rank, world, chunk)
    out = spectrahedron.walk_sample(end - begin, steps, L, rho, seed, kind=kind, chain_begin=begin, T=T)
    parts = chunk_moments(out["final_x"], chunk)
    sx, sxx = reduce_chunked_moments(parts, spectrahedron.n, make_allgather(group))
    return sx, sxx, out["stats"]
