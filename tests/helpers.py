"""Shared numpy helpers for the parity tests (test code, not product)."""
from __future__ import annotations

import numpy as np


def morton_words(coords: np.ndarray) -> list[np.ndarray]:
    """Interleaved Morton address (level 7 first, dim 0 first) as uint64 words, MSW first.

    Restates the explicit interleave oracle of proj/tests/support/oracles.hpp:33-39.
    """
    coords = np.asarray(coords, dtype=np.uint8)
    n, D = coords.shape
    bits = []
    for level in range(7, -1, -1):
        for d in range(D):
            bits.append((coords[:, d] >> level) & 1)
    nb = len(bits)
    words = []
    for start in range(0, nb, 64):
        w = np.zeros(n, dtype=np.uint64)
        chunk = bits[start:start + 64]
        for b in chunk:
            w = (w << np.uint64(1)) | b.astype(np.uint64)
        words.append(w)
    return words


def is_morton_sorted(coords: np.ndarray, keys: np.ndarray) -> bool:
    """Adjacent pairs ordered by (Morton address, packed key) -- zcurve.cpp:116-125."""
    if len(keys) < 2:
        return True
    words = morton_words(coords)
    less = np.zeros(len(keys) - 1, dtype=bool)
    equal = np.ones(len(keys) - 1, dtype=bool)
    for w in words:
        a, b = w[:-1], w[1:]
        less |= equal & (a < b)
        equal &= a == b
    less |= equal & (keys[:-1] < keys[1:])
    return bool(less.all())


def fillfront(known: np.ndarray) -> list[tuple[int, int]]:
    """KNOWN pixels with an UNKNOWN 4-neighbour, row-major (proj/src/image.cpp:49-61)."""
    k = known != 0
    h, w = k.shape
    unk = ~k
    nb = np.zeros_like(k)
    nb[:, 1:] |= unk[:, :-1]
    nb[:, :-1] |= unk[:, 1:]
    nb[1:, :] |= unk[:-1, :]
    nb[:-1, :] |= unk[1:, :]
    ys, xs = np.nonzero(k & nb)
    return list(zip(xs.tolist(), ys.tolist()))


def pca_of(mi, layouts=range(8)):
    pm = np.stack([mi.layout(l)["mean"] for l in layouts])
    pc = np.stack([mi.layout(l)["components"] for l in layouts])
    return pm, pc


class OracleShard:
    """CPU stand-in for sharding.DeviceShard (test infrastructure): the same stage methods and
    record format (Morton words + (layout << 29 | global row) payload), computed with the oracle
    restatement and numpy, so the multi-process orchestration (sharding.build_sharded over gloo)
    is exercised end to end on CPU.  D <= 8 (the Morton key fits a uint64 here)."""

    def __init__(self, img, known, K, coverage, dims, rank, world):
        import oracle
        from paper_1712_06326_b200 import sharding
        self.o, self.sh = oracle, sharding
        self.img, self.K, self.rank, self.world = img, K, rank, world
        self.ch = 1 if img.ndim == 2 else img.shape[2]
        self.dict = oracle.collect_dictionary(known, K)
        self.n_total = int(self.dict.size)
        self.row_begin, self.row_end = sharding.shard_ranges(self.n_total, world)[rank]
        self.rc = oracle.subset_layouts(K, coverage)
        self.m = self.rc.shape[1]
        self.mc = self.m * self.ch
        self.dims = min(dims, self.mc, self.n_total)
        assert self.dims <= 8
        self.words = (self.dims + 3) // 4
        self.F = K * K * self.ch
        self.out = {}

    @property
    def _rows(self):
        return self.dict[self.row_begin:self.row_end]

    def moments(self):
        s, S = self.o.patch_moments(self.img, self.K, self._rows)
        return np.concatenate([s, S.ravel()])

    def fit_project(self, mom):
        F, D = self.F, self.dims
        s, S = mom[:F], mom[F:].reshape(F, F)
        self.models, self.y = [], []
        lo, hi = np.full((8, D), np.inf), np.full((8, D), -np.inf)
        for l in range(8):
            cols = self.o.layout_columns(self.rc[l], self.K, self.ch)
            mean, cov = self.o.layout_covariance(s, S, self.n_total, cols)
            comp, eig = self.o.pca_from_cov(cov, D)
            self.models.append((mean, comp))
            if self._rows.size:
                a, b, _, y = self.o.project_build(self.img, self._rows, self.rc[l], mean, comp)
                lo[l], hi[l] = a, b
            else:
                y = np.zeros((0, D))
            self.y.append(y)
        olo = self.sh.double_to_ordered_i64(lo.ravel())
        ohi = self.sh.double_to_ordered_i64(hi.ravel())
        if not self._rows.size:  # identities of MIN / MAX, as the device shard reports them
            olo[:], ohi[:] = np.iinfo(np.int64).max, np.iinfo(np.int64).min
        return olo, ohi

    def refine_ranges(self, lo, hi):  # the oracle's ranges are exact already
        return np.array(lo, dtype=np.int64), np.array(hi, dtype=np.int64)

    def _key(self, coords):
        D = self.dims
        key = np.zeros(coords.shape[0], dtype=np.uint64)
        for d in range(D):
            for L in range(8):
                bit = (coords[:, d].astype(np.uint64) >> np.uint64(L)) & np.uint64(1)
                key |= bit << np.uint64(L * D + D - 1 - d)
        return key

    def _coords(self, key):
        D = self.dims
        c = np.zeros((key.size, D), dtype=np.uint8)
        for d in range(D):
            for L in range(8):
                c[:, d] |= (((key >> np.uint64(L * D + D - 1 - d)) & np.uint64(1)) << np.uint64(L)).astype(np.uint8)
        return c

    def _records(self, key, payload):
        r = np.zeros((key.size, self.words + 1), dtype=np.uint32)
        for k in range(self.words):
            r[:, k] = ((key >> np.uint64(32 * k)) & np.uint64(0xFFFFFFFF)).astype(np.uint32)
        r[:, self.words] = payload
        return r

    def _unpack(self, recs):
        key = np.zeros(recs.shape[0], dtype=np.uint64)
        for k in range(self.words):
            key |= recs[:, k].astype(np.uint64) << np.uint64(32 * k)
        return key, recs[:, self.words].astype(np.uint64)

    def _sort(self, recs):
        key, pay = self._unpack(recs)
        return recs[np.lexsort((pay, key, pay >> np.uint64(29)))]

    def quantize_sort(self, lo, hi, samples):
        lo = self.sh.ordered_i64_to_double(lo).reshape(8, self.dims)
        hi = self.sh.ordered_i64_to_double(hi).reshape(8, self.dims)
        q = np.vectorize(self.o.quantize, otypes=[np.uint8])
        n = self.row_end - self.row_begin
        rows = np.arange(self.row_begin, self.row_end, dtype=np.uint64)
        parts = []
        for l in range(8):
            coords = np.stack([q(lo[l, d], hi[l, d], self.y[l][:, d]) for d in range(self.dims)], 1) \
                if n else np.zeros((0, self.dims), np.uint8)
            parts.append(self._records(self._key(coords), (np.uint64(l) << np.uint64(29)) | rows))
        self.recs = self._sort(np.concatenate(parts))
        out = np.full((8 * samples, self.words + 1), 0xFFFFFFFF, dtype=np.uint32)
        if n:
            for l in range(8):
                for j in range(samples):
                    out[l * samples + j] = self.recs[l * n + (2 * j + 1) * n // (2 * samples)]
        return out

    def _composite(self, rec):
        key, pay = self._unpack(rec.reshape(1, -1))
        return (int(key[0]) << 32) | int(pay[0])

    def partition(self, splitters):
        import bisect
        import torch
        n, G = self.row_end - self.row_begin, self.world
        counts = np.zeros((G, 8), dtype=np.uint64)
        segs = []
        for l in range(8):
            seg = [self._composite(r) for r in self.recs[l * n:(l + 1) * n]]
            b = [0] + [bisect.bisect_left(seg, self._composite(splitters[l * (G - 1) + j])) for j in range(G - 1)] + [n]
            b = np.maximum.accumulate(b)
            segs.append(b)
        send = []
        for g in range(G):
            for l in range(8):
                counts[g, l] = segs[l][g + 1] - segs[l][g]
                send.append(self.recs[l * n + segs[l][g]:l * n + segs[l][g + 1]])
        return counts, torch.from_numpy(np.concatenate(send).view(np.int32))

    def receive(self, recv, all_counts):
        import torch
        recs = self._sort(recv.numpy().view(np.uint32))
        G, me = self.world, self.rank
        held = all_counts[:, me, :].sum(0).astype(np.int64)
        base = np.concatenate([[0], np.cumsum(held)])
        cnt, st = self.sh.rebalance_plan(all_counts, G, self.n_total, me)
        send = [recs[base[l] + int(st[g, l]):base[l] + int(st[g, l]) + int(cnt[g, l])]
                for g in range(G) for l in range(8)]
        return cnt, torch.from_numpy(np.concatenate(send).view(np.int32))

    def finish(self, recv2, all_counts2):
        recs = recv2.numpy().view(np.uint32)
        G, me = self.world, self.rank
        off, by = 0, {l: [] for l in range(8)}
        for s in range(G):
            for l in range(8):
                c = int(all_counts2[s, me, l])
                by[l].append(recs[off:off + c])
                off += c
        for l in range(8):
            r = np.concatenate(by[l])
            key, pay = self._unpack(r)
            self.out[l] = (self._coords(key), self.dict[(pay & np.uint64((1 << 29) - 1)).astype(np.int64)])

    def index_arrays(self, l):
        return self.out[l]
