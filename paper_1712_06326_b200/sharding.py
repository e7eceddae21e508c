"""Multi-GPU plumbing for the sharded path.

The hot path shards naturally:
  * build   -- the dictionary is range-partitioned by Morton key: rank r ends up holding exactly
               positions shard_ranges(n, G)[r] of every layout index that multi_index::build
               (proj/src/builder.cpp:202-224) produces on one host, so every shard's windows are
               the reference's global windows.  The stages run on the device (zi_shard_*, C ABI;
               shard.cu); between them this module runs the collectives:
                 moments       all-reduce SUM  (exact int64: bit-identical for any G)
                 lo / hi       all-reduce MIN / MAX (order-preserving int64 of the fp64 ranges):
                               approximate ranges of the tensor-core projection's min / max
                               pass, then the exact ranges over every rank's candidates
                 samples       all-gather, splitters on the host (zi_shard_splitters)
                 records       all-to-all (sample sort), then an all-to-all that rebalances the
                               received Morton ranges to the exact shard ranges
               Independent images still run as plain replicas (bench.py, weak scaling).
  * query   -- every rank computes an exact local top-k on its shard (sm_100a kernels), the k
               packed (dist<<32 | key) values of every rank are all-gathered and merged.  Packed
               values are unique and their integer order is the reference's (distance, key) order
               (proj/include/zinpaint/types.hpp:26-31), so the merged top-k equals knn_search
               over the whole dictionary; the merged list is refined once (zi_refine_best);
  * brute force -- each rank scans its dictionary slice; the winners are min-reduced as packed
               u64 (cost<<32 | key), exact for the same reason (proj/src/engine.cpp:226-234).
The collectives run through torch.distributed (NCCL on the GPU box, gloo in the CPU tests), or
in-process (LoopbackComm: G shards driven by one process, for single-GPU tests of the stages).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from ._lib import check, i64p, lib, ptr, u8p, u32p, u64p

I64_MAX = np.iinfo(np.int64).max
SENTINEL = 0xFFFFFFFF


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
    """All-gather every rank's k packed candidates (padded with INT64_MAX) and merge them."""
    torch, dist = _torch()
    k = max(int(k), 1)
    pad = np.full(k, I64_MAX, dtype=np.int64)
    loc = np.asarray(local, dtype=np.uint64)[:k].astype(np.int64)  # packed < 2^63 (dist < 2^31)
    pad[:loc.size] = loc
    t = torch.from_numpy(pad)
    if device is not None:
        t = t.to(device)
    world = dist.get_world_size(group)
    bufs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(bufs, t, group=group)
    merged = np.sort(np.concatenate([b.cpu().numpy() for b in bufs]))
    merged = merged[merged != I64_MAX][:k]
    return merged.astype(np.uint64)


def allreduce_min_packed(value: int, group=None, device=None) -> int:
    """Min-reduce one packed (cost<<32 | key) winner over all ranks (exact tie order)."""
    torch, dist = _torch()
    t = torch.tensor([min(int(value), I64_MAX)], dtype=torch.int64)
    if device is not None:
        t = t.to(device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return int(t.item())


# ------------------------------------------------------------------ order-preserving fp64 <-> int64
def double_to_ordered_i64(x) -> np.ndarray:
    """double_to_ordered (csrc/common.cuh) ^ 2^63: an int64 whose signed order is the fp64 order
    (-0.0 < +0.0), so MIN/MAX all-reduces of quantiser ranges are exact and sign-of-zero exact."""
    b = np.ascontiguousarray(x, dtype=np.float64).view(np.uint64)
    top = np.uint64(1 << 63)
    u = np.where(b & top, ~b, b | top)
    return (u ^ top).view(np.int64)


def ordered_i64_to_double(v) -> np.ndarray:
    top = np.uint64(1 << 63)
    u = np.ascontiguousarray(v, dtype=np.int64).view(np.uint64) ^ top
    b = np.where(u & top, u & ~top, ~u)
    return b.view(np.float64)


# ------------------------------------------------------------------ communicators
class Comm:
    """Collectives over the shards this process drives (lists, one entry per local shard)."""
    world: int
    ranks: list

    def allreduce(self, arrs, op: str):  # op in {"sum", "min", "max"}; int64 arrays
        raise NotImplementedError

    def allgather(self, arrs):  # equal-shape arrays -> per local shard, a list over all ranks
        raise NotImplementedError

    def alltoallv(self, sends, send_counts, recv_counts):  # [N, W1] int32 tensors, counts in records
        raise NotImplementedError

    def barrier(self):
        pass


class LoopbackComm(Comm):
    """G shards in one process (single-GPU tests of the sharded stages; no waiting kernels:
    every stage finishes on every shard before the next exchange)."""

    def __init__(self, world: int):
        self.world = world
        self.ranks = list(range(world))

    def allreduce(self, arrs, op):
        a = np.stack([np.asarray(x, dtype=np.int64) for x in arrs])
        r = {"sum": a.sum(0), "min": a.min(0), "max": a.max(0)}[op]
        return [r.copy() for _ in arrs]

    def allgather(self, arrs):
        full = [np.asarray(x) for x in arrs]
        return [list(full) for _ in arrs]

    def alltoallv(self, sends, send_counts, recv_counts):
        torch, _ = _torch()
        offs = [np.concatenate([[0], np.cumsum(np.asarray(c, dtype=np.int64))]) for c in send_counts]
        out = []
        for d in range(self.world):
            parts = [sends[s][int(offs[s][d]):int(offs[s][d + 1])] for s in range(self.world)]
            out.append(torch.cat(parts, 0) if parts else sends[d][:0])
        if out and out[0].is_cuda:
            torch.cuda.synchronize()  # the shards' stages run on their own (non-blocking) streams
        return out


class TorchComm(Comm):
    """One shard per process over torch.distributed (NCCL with device tensors, gloo on CPU)."""

    def __init__(self, group=None, device=None):
        torch, dist = _torch()
        self.group = group
        self.device = device
        self.world = dist.get_world_size(group)
        self.ranks = [dist.get_rank(group)]

    def _t(self, a):
        torch, _ = _torch()
        t = torch.from_numpy(np.ascontiguousarray(a))
        return t.to(self.device) if self.device is not None else t

    def allreduce(self, arrs, op):
        torch, dist = _torch()
        (a,) = arrs
        t = self._t(np.asarray(a, dtype=np.int64))
        dist.all_reduce(t, op={"sum": dist.ReduceOp.SUM, "min": dist.ReduceOp.MIN, "max": dist.ReduceOp.MAX}[op],
                        group=self.group)
        return [t.cpu().numpy()]

    def allgather(self, arrs):
        torch, dist = _torch()
        (a,) = arrs
        a = np.ascontiguousarray(a)
        is_u32 = a.dtype == np.uint32
        t = self._t(a.view(np.int32) if is_u32 else a.astype(np.int64) if a.dtype == np.uint64 else a)
        bufs = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(bufs, t, group=self.group)
        out = [b.cpu().numpy() for b in bufs]
        if is_u32:
            out = [o.view(np.uint32) for o in out]
        elif a.dtype == np.uint64:
            out = [o.astype(np.uint64) for o in out]
        return [out]

    def alltoallv(self, sends, send_counts, recv_counts):
        torch, dist = _torch()
        (s,) = sends
        sc = [int(v) for v in send_counts[0]]
        rc = [int(v) for v in recv_counts[0]]
        dev = s.device
        if s.is_cuda and dist.get_backend(self.group) != "nccl":
            torch.cuda.synchronize(dev)  # host staging for backends without device buffers (gloo)
            s = s.cpu()
        recv = torch.empty((sum(rc), s.shape[1]), dtype=s.dtype, device=s.device)
        dist.all_to_all_single(recv, s, rc, sc, group=self.group)
        if recv.device != dev:
            recv = recv.to(dev)
        if recv.is_cuda:
            torch.cuda.synchronize(recv.device)
        return [recv]

    def barrier(self):
        _, dist = _torch()
        dist.barrier(group=self.group)


# ------------------------------------------------------------------ device shard (C ABI)
class _DeviceRecords:
    """A shard-owned device buffer of n records (W1 u32 words each) seen by torch, zero copy."""

    def __init__(self, ptr: int, n: int, w1: int):
        self.__cuda_array_interface__ = {"shape": (n, w1), "typestr": "<i4", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


class DeviceShard:
    """One rank's zi_shard (include/zinpaint_b200.h): the device side of a sharded build."""

    def __init__(self, image, known, cfg, rank: int, world: int, ctx=None):
        from . import Context, _u8
        self.ctx = ctx or Context.default()
        self.cfg = cfg
        img = _u8(image)
        self.height, self.width = img.shape[:2]
        self.channels = 1 if img.ndim == 2 else img.shape[2]
        kn = _u8(known)
        self._img, self._known = img, kn
        h = C.c_void_p()
        check(lib().zi_shard_create(self.ctx.h, ptr(img, u8p), ptr(kn, u8p), self.width, self.height, self.channels,
                                    C.byref(cfg), rank, world, C.byref(h)))
        self.h = h
        self.rank, self.world = rank, world
        self._mi = None
        self._info()

    def _info(self):
        v = np.zeros(10, dtype=np.uint64)
        check(lib().zi_shard_info(self.h, ptr(v, u64p)))
        (self.n_total, self.row_begin, self.row_end, self.F, self.dims, self.words, _, _, self.stage,
         self.held) = (int(x) for x in v)
        return v

    # -- stages
    def moments(self) -> np.ndarray:
        out = np.zeros(self.F + self.F * self.F, dtype=np.int64)
        check(lib().zi_shard_moments(self.h, ptr(out, i64p)))
        return out

    def fit_project(self, moments):
        m = np.ascontiguousarray(moments, dtype=np.int64)
        lo = np.zeros(8 * self.dims, dtype=np.int64)
        hi = np.zeros(8 * self.dims, dtype=np.int64)
        check(lib().zi_shard_fit_project(self.h, ptr(m, i64p), ptr(lo, i64p), ptr(hi, i64p)))
        return lo, hi

    def refine_ranges(self, lo, hi):
        """Global (approximate, on the tensor-core path) ranges -> this rank's exact partial ranges."""
        lo = np.ascontiguousarray(lo, dtype=np.int64)
        hi = np.ascontiguousarray(hi, dtype=np.int64)
        lo2 = np.zeros_like(lo)
        hi2 = np.zeros_like(hi)
        check(lib().zi_shard_refine_ranges(self.h, ptr(lo, i64p), ptr(hi, i64p), ptr(lo2, i64p), ptr(hi2, i64p)))
        return lo2, hi2

    def quantize_sort(self, lo, hi, samples: int) -> np.ndarray:
        lo = np.ascontiguousarray(lo, dtype=np.int64)
        hi = np.ascontiguousarray(hi, dtype=np.int64)
        out = np.zeros((8 * samples, self.words + 1), dtype=np.uint32)
        check(lib().zi_shard_quantize_sort(self.h, ptr(lo, i64p), ptr(hi, i64p), samples, ptr(out, u32p)))
        return out

    def partition(self, splitters):
        sp = np.ascontiguousarray(splitters, dtype=np.uint32)
        counts = np.zeros((self.world, 8), dtype=np.uint64)
        d = C.c_void_p()
        check(lib().zi_shard_partition(self.h, ptr(sp, u32p) if sp.size else None, ptr(counts, u64p), C.byref(d)))
        return counts, self._as_tensor(d.value, int(counts.sum()))

    def receive(self, recv, all_counts):
        ac = np.ascontiguousarray(all_counts, dtype=np.uint64)
        counts2 = np.zeros((self.world, 8), dtype=np.uint64)
        d = C.c_void_p()
        check(lib().zi_shard_receive(self.h, C.c_void_p(recv.data_ptr()) if recv.numel() else None,
                                     ptr(ac, u64p), ptr(counts2, u64p), C.byref(d)))
        return counts2, self._as_tensor(d.value, int(counts2.sum()))

    def rebuild(self):
        """Restart the stages for another build (same device-resident image; buffers kept)."""
        check(lib().zi_shard_rebuild(self.h))
        self._info()

    def finish_local(self):
        """One rank: finalise the locally sorted layouts (no exchange)."""
        check(lib().zi_shard_finish_local(self.h))
        self._info()

    def finish(self, recv2, all_counts2):
        ac = np.ascontiguousarray(all_counts2, dtype=np.uint64)
        check(lib().zi_shard_finish(self.h, C.c_void_p(recv2.data_ptr()) if recv2.numel() else None, ptr(ac, u64p)))
        self._info()

    def _as_tensor(self, p, n):
        torch, _ = _torch()
        dev = torch.device("cuda", self.ctx.device)  # the shard ctx's GPU, not torch's current one
        if n == 0 or not p:
            return torch.zeros((0, self.words + 1), dtype=torch.int32, device=dev)
        return torch.as_tensor(_DeviceRecords(p, n, self.words + 1), device=dev)

    # -- the built shard
    @property
    def multi_index(self):
        """Borrowed MultiIndex view of this rank's slice (8 index shards + dictionary slice)."""
        if self._mi is None:
            from . import MultiIndex
            h = C.c_void_p()
            check(lib().zi_shard_multi_index(self.h, C.byref(h)))
            mi = MultiIndex.__new__(MultiIndex)
            mi._borrowed = True  # the shard owns the handle
            mi.ctx = self.ctx
            mi.cfg = self.cfg
            mi.height, mi.width, mi.channels = self.height, self.width, self.channels
            mi._img, mi._known = self._img, self._known
            mi.h = h
            mi._refresh_info()
            self._mi = mi
        return self._mi

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            if self._mi is not None:
                self._mi.h = None
            lib().zi_shard_destroy(h)
            self.h = None


# ------------------------------------------------------------------ the stage driver
def splitters_from_samples(samples: Sequence[np.ndarray], words: int, world: int) -> np.ndarray:
    """zi_shard_splitters over the all-gathered sample rows (host; order = layout, Morton, row)."""
    allrows = np.ascontiguousarray(np.concatenate([np.asarray(s, dtype=np.uint32).reshape(-1, words + 1)
                                                   for s in samples]))
    out = np.zeros((8 * max(world - 1, 0), words + 1), dtype=np.uint32)
    check(lib().zi_shard_splitters(ptr(allrows, u32p), allrows.shape[0], words, world,
                                   ptr(out, u32p) if out.size else None))
    return out


def rebalance_plan(all_counts: np.ndarray, world: int, n_total: int, me: int):
    """zi_shard_rebalance_plan: (records to each destination [G][8], start positions [G][8])."""
    ac = np.ascontiguousarray(all_counts, dtype=np.uint64)
    cnt = np.zeros((world, 8), dtype=np.uint64)
    st = np.zeros((world, 8), dtype=np.uint64)
    check(lib().zi_shard_rebalance_plan(ptr(ac, u64p), world, n_total, me, ptr(cnt, u64p), ptr(st, u64p)))
    return cnt, st


def build_sharded(shards: list, comm: Comm, samples: int = 256) -> dict:
    """Run the sharded build over the local shards (one per rank this process drives).

    Works for any object with the DeviceShard stage methods (the CPU tests drive a numpy
    stand-in through the same sequence).  Returns per-stage exchange sizes for reporting."""
    world = comm.world
    mom = comm.allreduce([sh.moments() for sh in shards], "sum")
    lohi = [sh.fit_project(m) for sh, m in zip(shards, mom)]
    lo = comm.allreduce([x[0] for x in lohi], "min")
    hi = comm.allreduce([x[1] for x in lohi], "max")
    lohi = [sh.refine_ranges(a, b) for sh, a, b in zip(shards, lo, hi)]  # exact ranges (tensor-core path)
    lo = comm.allreduce([x[0] for x in lohi], "min")
    hi = comm.allreduce([x[1] for x in lohi], "max")
    samp = [sh.quantize_sort(a, b, samples if world > 1 else 0) for sh, a, b in zip(shards, lo, hi)]
    words = shards[0].words
    if world == 1 and all(hasattr(sh, "finish_local") for sh in shards):
        for sh in shards:  # one rank: the sorted layouts are the index, no exchange
            sh.finish_local()
        return {"records_exchanged": 0, "records_rebalanced": 0, "words_per_record": words + 1}
    if world > 1:
        gathered = comm.allgather(samp)
        spl = [splitters_from_samples(g, words, world) for g in gathered]
    else:
        spl = [np.zeros((0, words + 1), dtype=np.uint32) for _ in shards]
    parts = [sh.partition(s) for sh, s in zip(shards, spl)]
    all_counts = [np.stack(g) for g in comm.allgather([c for c, _ in parts])]  # [src][dst][8]
    me = comm.ranks
    recv = comm.alltoallv([t for _, t in parts], [c.sum(1) for c, _ in parts],
                          [ac[:, r, :].sum(1) for ac, r in zip(all_counts, me)])
    parts2 = [sh.receive(rv, ac) for sh, rv, ac in zip(shards, recv, all_counts)]
    all_counts2 = [np.stack(g) for g in comm.allgather([c for c, _ in parts2])]
    recv2 = comm.alltoallv([t for _, t in parts2], [c.sum(1) for c, _ in parts2],
                           [ac[:, r, :].sum(1) for ac, r in zip(all_counts2, me)])
    for sh, rv, ac in zip(shards, recv2, all_counts2):
        sh.finish(rv, ac)
    a1, a2 = all_counts[0], all_counts2[0]
    moved1 = int(a1.sum() - sum(a1[r, r].sum() for r in range(world)))
    moved2 = int(a2.sum() - sum(a2[r, r].sum() for r in range(world)))
    return {"records_exchanged": moved1, "records_rebalanced": moved2, "words_per_record": words + 1}


def sharded_query(shards: list, comm: Comm, target_values, target_known, k: int, norm: int = 0):
    """query_best_patch (proj/src/engine.cpp:178-213) over range-partitioned shards: local exact
    top-k per shard, all-gather + merge of the packed lists, one refine of the global top-k.
    Returns, per local shard, (key, cost, error, layout_id, candidates) -- identical on all."""
    from . import BestPatch, _u8
    k = max(int(k), 1)
    tv, tk = _u8(target_values), _u8(target_known)
    lists, lids = [], []
    for sh in shards:
        (_, _, _, lid, _), cand = sh.multi_index.query_best_patch(tv, tk, k, norm, return_candidates=True)
        pad = np.full(k, I64_MAX, dtype=np.int64)
        pad[:cand.size] = cand.astype(np.int64)
        lists.append(pad)
        lids.append(lid)
    gathered = comm.allgather(lists)
    out = []
    for sh, g, lid in zip(shards, gathered, lids):
        merged = np.sort(np.concatenate(g))
        merged = np.ascontiguousarray(merged[merged != I64_MAX][:k].astype(np.uint64))
        bp = BestPatch()
        check(lib().zi_refine_best(sh.multi_index.h, ptr(tv, u8p), ptr(tk, u8p),
                                   ptr(merged, u64p) if merged.size else None, merged.size, norm, C.byref(bp)))
        out.append((bp.key, bp.cost, bp.error, lid, merged.size))
    return out


def sharded_brute_force(shards: list, comm: Comm, target_values, target_known, norm: int = 0):
    """brute_force_best (proj/src/engine.cpp:220-236) over the dictionary slices: packed MIN."""
    vals = []
    for sh in shards:
        key, cost, _ = sh.multi_index.brute_force_best(target_values, target_known, norm)
        vals.append(np.array([(int(cost) << 32) | int(key) if sh.multi_index.n else I64_MAX], dtype=np.int64))
    red = comm.allreduce(vals, "min")
    return [(int(r[0]) & 0xFFFFFFFF, int(r[0]) >> 32) for r in red]


class ShardedMultiIndex:
    """This rank's part of a multi_index range-partitioned over a torch.distributed group (one
    GPU per rank).  Query results equal MultiIndex's on the whole image, bit for bit."""

    def __init__(self, image, known, cfg=None, group=None, samples: int = 256, ctx=None, **kw):
        import torch

        from . import index_config
        _, dist = _torch()
        self.cfg = cfg if cfg is not None else index_config(**kw)
        dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else None
        self.comm = TorchComm(group, device=dev if dist.get_backend(group) == "nccl" else None)
        self.shard = DeviceShard(image, known, self.cfg, self.comm.ranks[0], self.comm.world, ctx=ctx)
        self.exchange = build_sharded([self.shard], self.comm, samples)

    @property
    def multi_index(self):
        return self.shard.multi_index

    def index_arrays(self, l: int):
        return self.multi_index.index_arrays(l)

    def query_best_patch(self, target_values, target_known, k: Optional[int] = None, norm=None):
        k = self.cfg.knn if k is None else k
        nrm = self.cfg.norm if norm is None else norm
        return sharded_query([self.shard], self.comm, target_values, target_known, k, nrm)[0]

    def brute_force_best(self, target_values, target_known, norm=None):
        nrm = self.cfg.norm if norm is None else norm
        return sharded_brute_force([self.shard], self.comm, target_values, target_known, nrm)[0]
