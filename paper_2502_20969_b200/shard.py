"""Multi-GPU plumbing of the retrieval path.

One process per GPU. Queries shard independently — each GPU serves its own
micro-batches against its own cluster cache — so there is
no collective on the data path. torch.distributed is used only to agree on
the routing input (every rank's resident set, one byte per cluster) and to
take the max of the ranks' timings.

Routing follows assign_cache_aware (sched.cpp:87-144): overlap[b][w] =
|probe union of batch b ∩ resident set of worker w|, then the greedy with a
cap of ceil(nb / nw) per worker (`laiv.greedy_assign`, the library's C++
greedy). Every rank builds the same matrix from the same all-gathered inputs,
so every rank computes the same assignment without a broadcast.
"""
from __future__ import annotations

import numpy as np

from . import laiv


def shard_indices(n: int, rank: int, world: int) -> np.ndarray:
    """Query indices rank `rank` serves under weak scaling (round-robin)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    return np.arange(rank, n, world)


def probe_union_masks(probes: np.ndarray, batches: list[laiv.MicroBatch], nc: int) -> np.ndarray:
    """[nb, nc] byte masks of each batch's distinct probed clusters
    (batch_probe_union, sched.cpp:15-26). probes: [nq, L] cluster ids."""
    out = np.zeros((len(batches), nc), np.uint8)
    for b, mb in enumerate(batches):
        if mb.queries:
            out[b, np.asarray(probes)[mb.queries].reshape(-1)] = 1
    return out


def overlap_matrix(unions: np.ndarray, resident: np.ndarray) -> np.ndarray:
    """overlap[b][w] = |unions[b] ∩ resident[w]| (sched.cpp:103-108)."""
    u = np.asarray(unions, np.uint64)
    r = np.asarray(resident, np.uint64)
    return u @ r.T


def route(batches: list[laiv.MicroBatch], probes: np.ndarray, resident: np.ndarray) -> list[int]:
    """Batch -> worker by the cache-aware greedy over all workers' resident
    masks ([nw, nc])."""
    nc = resident.shape[1]
    return laiv.greedy_assign(overlap_matrix(probe_union_masks(probes, batches, nc), resident))


def gather_resident(mask: np.ndarray, device=None) -> np.ndarray:
    """All-gather one byte per cluster from every rank -> [world, nc]."""
    import torch
    import torch.distributed as dist

    t = torch.as_tensor(np.ascontiguousarray(mask, np.uint8))
    if device is not None:
        t = t.to(device)
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t)
    return np.stack([p.cpu().numpy() for p in parts])


def max_over_ranks(values, device=None) -> list[float]:
    """Element-wise max over ranks (timings: the slowest rank defines the job)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.cpu().tolist()]
