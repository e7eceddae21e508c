"""Multi-GPU plumbing for the sharded path.

The hot path shards naturally:
  * build   -- independent images (or independent layout indices) per rank: no collective;
  * query   -- a dictionary range-partitioned in Morton order: every rank computes an exact local
               top-k on its shard (sm_100a kernels), then the k packed (dist<<32 | key) values of
               every rank are all-gathered and merged.  Packed values are unique and their integer
               order is the reference's (distance, key) order (proj/include/zinpaint/types.hpp:26-31),
               so the merged top-k equals knn_search over the whole dictionary;
  * brute force -- each rank scans its shard; the winners are min-reduced as packed u64
               (cost<<32 | key), exact for the same reason (proj/src/engine.cpp:226-234).
The collectives run through torch.distributed (NCCL on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np


def shard_ranges(n: int, world: int) -> list[tuple[int, int]]:
    """Contiguous [begin, end) ranges of a Morton-ordered index, one per rank (sizes differ by <= 1)."""
    base, extra = divmod(n, world)
    out, b = [], 0
    for r in range(world):
        e = b + base + (1 if r < extra else 0)
        out.append((b, e))
        b = e
    return out


def merge_topk(lists, k: int) -> np.ndarray:
    """Exact global top-k of per-shard ascending packed lists (knn_list::sorted order)."""
    k = max(int(k), 1)
    allv = np.concatenate([np.asarray(l, dtype=np.uint64) for l in lists]) if lists else np.zeros(0, np.uint64)
    allv = allv[allv != np.uint64(0xFFFFFFFFFFFFFFFF)]
    return np.sort(allv)[:k]


def _torch():
    import torch
    import torch.distributed as dist
    return torch, dist


def allgather_topk(local: np.ndarray, k: int, group=None, device=None) -> np.ndarray:
    """All-gather every rank's k packed candidates (padded with UINT64_MAX) and merge them."""
    torch, dist = _torch()
    k = max(int(k), 1)
    pad = np.full(k, np.iinfo(np.int64).max, dtype=np.int64)
    loc = np.asarray(local, dtype=np.uint64)[:k].astype(np.int64)  # packed < 2^63 (dist < 2^31)
    pad[:loc.size] = loc
    t = torch.from_numpy(pad)
    if device is not None:
        t = t.to(device)
    world = dist.get_world_size(group)
    bufs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(bufs, t, group=group)
    merged = np.sort(np.concatenate([b.cpu().numpy() for b in bufs]))
    merged = merged[merged != np.iinfo(np.int64).max][:k]
    return merged.astype(np.uint64)


def allreduce_min_packed(value: int, group=None, device=None) -> int:
    """Min-reduce one packed (cost<<32 | key) winner over all ranks (exact tie order)."""
    torch, dist = _torch()
    t = torch.tensor([min(int(value), np.iinfo(np.int64).max)], dtype=torch.int64)
    if device is not None:
        t = t.to(device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return int(t.item())
