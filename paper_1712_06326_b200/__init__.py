"""B200-native SFC multi-index (arXiv 1712.06326) -- drop-in for the reference's hot path.

The module-level functions mirror the reference's Python binding ``zinpaint``
(proj/python/bindings.cpp:169-194) -- same names, arguments, defaults and result layout:
``inpaint``, ``knn_search``, ``subset_layouts``, ``morton_less``, ``less_most_significant_bit``.
The classes expose the C++ surface the reference's tests use (``zcurve_index``,
``multi_index``, ``query_best_patch``, ``brute_force_best``).  Everything goes through the C ABI
of ``libzinpaint_b200.so`` (include/zinpaint_b200.h); the compute runs in hand-written sm_100a
kernels.  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import math
from typing import Optional

import numpy as np

from . import _lib
from ._lib import (BestPatch, EmptyDictionaryError, IndexConfig, InpaintConfig, IterationRecord, MultiIndexInfo,
                   RunStats, ZIError, check, lib, ptr, u8p, u32p, u64p, i32p, i64p, f64p, f32p)

__all__ = ["inpaint", "knn_search", "subset_layouts", "morton_less", "less_most_significant_bit", "Context",
           "ZCurveIndex", "MultiIndex", "VectorIndex", "EmptyDictionaryError", "ZIError", "index_config", "NORMS"]

NORMS = {"l2": 0, "l1": 1}


def _norm(norm) -> int:
    if isinstance(norm, str):
        if norm not in NORMS:
            raise ValueError("norm must be 'l2' or 'l1'")
        return NORMS[norm]
    return int(norm)


def _u8(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint8)


# ------------------------------------------------------------------ host utilities
def less_most_significant_bit(a: int, b: int) -> bool:
    """proj/include/zinpaint/morton.hpp:10-12"""
    return bool(lib().zi_less_most_significant_bit(int(a), int(b)))


def morton_less(a, b) -> bool:
    """proj/include/zinpaint/morton.hpp:18-29 (bindings.cpp:158-165)"""
    a, b = _u8(a), _u8(b)
    if a.ndim != 1 or b.ndim != 1 or a.shape != b.shape:
        raise ValueError("morton_less expects two equal-length byte vectors")
    return bool(lib().zi_morton_less(ptr(a, u8p), ptr(b, u8p), a.size))


def subset_layouts(patch_size: int, coverage: float):
    """build_subset_layouts (proj/src/layouts.cpp:13-60), in the binding's dict form."""
    m = lib().zi_subset_pixel_count(patch_size, coverage)
    rc = np.zeros(max(8 * max(m, 1) * 2, 2), dtype=np.int32)
    mm = C.c_int32()
    check(lib().zi_subset_layouts(patch_size, coverage, ptr(rc, i32p), C.byref(mm)))
    m = mm.value
    rc = rc[:8 * m * 2].reshape(8, m, 2)
    mid = (patch_size - 1) // 2
    k = patch_size
    anchors = [(0, mid), (mid, k - 1), (k - 1, mid), (mid, 0), (0, 0), (0, k - 1), (k - 1, 0), (k - 1, k - 1)]
    return [{"id": l, "anchor": anchors[l], "pixels": [tuple(int(v) for v in p) for p in rc[l]]} for l in range(8)]


def index_config(patch_size=9, coverage=0.6, dims=10, knn=80, mu=256, nu=2048, norm="l2") -> IndexConfig:
    """index_config (proj/include/zinpaint/builder.hpp:24-34) with the reference defaults."""
    return IndexConfig(patch_size, coverage, dims, knn, mu, nu, _norm(norm))


# ------------------------------------------------------------------ device context
class Context:
    """One device + one CUDA stream (the zi_ctx handle)."""

    _default: Optional["Context"] = None

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib().zi_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device

    @classmethod
    def default(cls) -> "Context":
        if cls._default is None:
            cls._default = Context(0)
        return cls._default

    def synchronize(self):
        check(lib().zi_ctx_synchronize(self.h))

    def timer_start(self):
        check(lib().zi_timer_start(self.h))

    def timer_stop(self) -> float:
        ms = C.c_double()
        check(lib().zi_timer_stop(self.h, C.byref(ms)))
        return ms.value

    def flush_l2(self):
        check(lib().zi_ctx_flush_l2(self.h))

    @property
    def kernel_launches(self) -> int:
        return int(lib().zi_ctx_kernel_launches(self.h))

    def set_profiling(self, on: bool):
        check(lib().zi_ctx_set_profiling(self.h, int(on)))

    def set_sort_policy(self, dims: int, policy: int):
        """8-layout build sort for `dims`: 0 learn, -1 LSD passes (fused finalize), k > 0 MSD bytes."""
        check(lib().zi_ctx_set_sort_policy(self.h, int(dims), int(policy)))

    def set_profile_filter(self, names=None):
        """Time only these kernels while profiling (None: every kernel)."""
        check(lib().zi_ctx_set_profile_filter(self.h, ",".join(names).encode() if names else None))

    def profile(self) -> dict:
        """{kernel name: (total device ms, launches)} since set_profiling(True)."""
        out = {}
        i = 0
        while True:
            ms = C.c_double()
            n = C.c_uint64()
            name = C.c_char_p()
            if lib().zi_ctx_profile(self.h, i, C.byref(ms), C.byref(n), C.byref(name)) != 0:
                break
            out[name.value.decode()] = (ms.value, n.value)
            i += 1
        return out

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            lib().zi_ctx_destroy(h)
            self.h = None


# ------------------------------------------------------------------ z-curve index
class ZCurveIndex:
    """zcurve_index (proj/include/zinpaint/zcurve.hpp:117-145), device resident."""

    def __init__(self, handle, owner=None, ctx: Optional[Context] = None):
        self.h = handle
        self._owner = owner  # keeps a borrowing MultiIndex alive
        self._ctx = ctx
        n = C.c_uint64()
        d = C.c_uint32()
        check(lib().zi_index_size(self.h, C.byref(n), C.byref(d)))
        self.n, self.dims = n.value, d.value

    @classmethod
    def from_descriptors(cls, coords, keys, dims: Optional[int] = None, layout_id: int = 0,
                         ctx: Optional[Context] = None) -> "ZCurveIndex":
        """zcurve_index::from_descriptors (proj/src/zcurve.cpp:108-138)."""
        ctx = ctx or Context.default()
        coords = _u8(coords)
        keys = np.ascontiguousarray(keys, dtype=np.uint32)
        if dims is None:
            dims = coords.shape[1] if coords.ndim == 2 else 0
        n = keys.size
        if coords.size != n * dims:
            raise ValueError("zcurve_index: coords/keys size mismatch")
        h = C.c_void_p()
        check(lib().zi_index_from_descriptors(ctx.h, ptr(coords, u8p), ptr(keys, u32p), n, dims, layout_id,
                                              C.byref(h)))
        return cls(h, ctx=ctx)

    def __len__(self):
        return self.n

    def export(self):
        coords = np.zeros((self.n, self.dims), dtype=np.uint8)
        keys = np.zeros(self.n, dtype=np.uint32)
        check(lib().zi_index_export(self.h, ptr(coords, u8p), ptr(keys, u32p)))
        return coords, keys

    def knn(self, query, k: int, mu: int = 256, norm="l2") -> np.ndarray:
        """knn_search (proj/src/zcurve.cpp:429-452): packed (dist<<32|key) ascending."""
        q = _u8(query)
        if q.size != self.dims:
            raise ValueError("query must have dims bytes")
        out = np.zeros(max(1, min(max(k, 1), max(self.n, 1))), dtype=np.uint64)
        cnt = C.c_uint32()
        check(lib().zi_knn_search(self.h, ptr(q, u8p), k, mu, _norm(norm), ptr(out, u64p), C.byref(cnt)))
        return out[:cnt.value].copy()

    def knn_batch(self, queries, k: int, norm="l2"):
        q = _u8(queries)
        nq = q.shape[0]
        kk = max(k, 1)
        out = np.zeros((nq, kk), dtype=np.uint64)
        cnt = np.zeros(nq, dtype=np.uint32)
        check(lib().zi_knn_search_batch(self.h, ptr(q, u8p), nq, k, _norm(norm), ptr(out, u64p), ptr(cnt, u32p)))
        return out, cnt

    def knn_batch_bench(self, queries, k: int, norm="l2", reps: int = 5, return_results: bool = False):
        """Device-resident batched k-NN timed with CUDA events -> (ms per batch, stats[3], results)."""
        q = _u8(queries)
        nq = q.shape[0]
        ms = C.c_double()
        stats = np.zeros(3, dtype=np.uint64)
        out = np.zeros((nq, k), dtype=np.uint64) if return_results else None
        cnt = np.zeros(nq, dtype=np.uint32) if return_results else None
        check(lib().zi_knn_batch_bench(self.h, ptr(q, u8p), nq, k, _norm(norm), reps, C.byref(ms), ptr(stats, u64p),
                                       ptr(out, u64p) if out is not None else None,
                                       ptr(cnt, u32p) if cnt is not None else None))
        return ms.value, stats, (out, cnt)

    def __del__(self):
        h = getattr(self, "h", None)
        if h and self._owner is None:
            lib().zi_index_destroy(h)
        self.h = None


class PatchIndex:
    """build_index (proj/include/zinpaint/builder.hpp:77-81, proj/src/builder.cpp:129-195): ONE
    layout index over a caller-given dictionary, fitted, projected and sorted on the device."""

    def __init__(self, image, keys, layout_rc, cfg: Optional[IndexConfig] = None, ctx: Optional[Context] = None,
                 **kw):
        self.ctx = ctx or Context.default()
        self.cfg = cfg if cfg is not None else index_config(**kw)
        img = _u8(image)
        self.height, self.width = img.shape[:2]
        self.channels = 1 if img.ndim == 2 else img.shape[2]
        keys = np.ascontiguousarray(keys, dtype=np.uint32)
        rc = np.ascontiguousarray(layout_rc, dtype=np.int32).reshape(-1, 2)
        self.m = rc.shape[0]
        h = C.c_void_p()
        check(lib().zi_index_build(self.ctx.h, ptr(img, u8p), self.width, self.height, self.channels,
                                   ptr(keys, u32p), keys.size, ptr(rc, i32p), self.m, C.byref(self.cfg), C.byref(h)))
        self.h = h
        d, mc = C.c_int32(), C.c_int32()
        check(lib().zi_patch_index_model(self.h, C.byref(d), C.byref(mc), None, None, None, None, None, None, None))
        self.dims, self.mc, self.n = d.value, mc.value, keys.size

    def model(self) -> dict:
        D, mc = self.dims, self.mc
        mean, comp, eig, lo, hi = np.zeros(mc), np.zeros((D, mc)), np.zeros(D), np.zeros(D), np.zeros(D)
        bs, ss = C.c_double(), C.c_double()
        check(lib().zi_patch_index_model(self.h, None, None, ptr(mean, f64p), ptr(comp, f64p), ptr(eig, f64p),
                                         ptr(lo, f64p), ptr(hi, f64p), C.byref(bs), C.byref(ss)))
        return {"mean": mean, "components": comp, "eigenvalues": eig, "lo": lo, "hi": hi,
                "build_seconds": bs.value, "sort_seconds": ss.value}

    def index(self) -> "ZCurveIndex":
        h = C.c_void_p()
        check(lib().zi_patch_index_get_index(self.h, C.byref(h)))
        return ZCurveIndex(h, owner=self)

    def make_query(self, target_values, target_known) -> np.ndarray:
        """patch_index::make_query (proj/src/builder.cpp:110-127), on the device."""
        tv, tk = _u8(target_values), _u8(target_known)
        out = np.zeros(self.dims, dtype=np.uint8)
        check(lib().zi_make_query(self.h, ptr(tv, u8p), ptr(tk, u8p), ptr(out, u8p)))
        return out

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            lib().zi_patch_index_destroy(h)
            self.h = None


def brute_force_scan(image, keys, target_values, target_known, patch_size: int, norm="l2",
                     ctx: Optional[Context] = None):
    """brute_force_best(image, target, dictionary, norm) (proj/src/engine.cpp:220-236) over a caller
    dictionary -> (key, cost, error)."""
    ctx = ctx or Context.default()
    img = _u8(image)
    h, w = img.shape[:2]
    ch = 1 if img.ndim == 2 else img.shape[2]
    keys = np.ascontiguousarray(keys, dtype=np.uint32)
    tv, tk = _u8(target_values), _u8(target_known)
    bp = BestPatch()
    check(lib().zi_brute_force_scan(ctx.h, ptr(img, u8p), w, h, ch, ptr(keys, u32p), keys.size, ptr(tv, u8p),
                                    ptr(tk, u8p), patch_size, _norm(norm), C.byref(bp)))
    return bp.key, bp.cost, bp.error


# ------------------------------------------------------------------ cfg5 vector index
class VectorIndex:
    """Index over fp32 feature vectors (BASELINE configs[4]): PCA fit, projection, quantiser and
    Morton sort on the device; rows are the keys (proj/python/bindings.cpp:109-125)."""

    def __init__(self, X, dims: int, ctx: Optional[Context] = None):
        """X: (n, dim) float32 -- a numpy array, or a CUDA tensor (built from device memory)."""
        self.ctx = ctx or Context.default()
        h = C.c_void_p()
        if hasattr(X, "is_cuda") and X.is_cuda:
            if X.dtype.__str__() != "torch.float32" or X.dim() != 2 or not X.is_contiguous():
                raise ValueError("X must be a contiguous (n, dim) float32 tensor")
            self.n, self.dim = int(X.shape[0]), int(X.shape[1])
            check(lib().zi_vector_index_build_device(self.ctx.h, C.c_void_p(X.data_ptr()), self.n, self.dim, dims,
                                                     C.byref(h)))
        else:
            X = np.ascontiguousarray(X, dtype=np.float32)
            if X.ndim != 2:
                raise ValueError("X must be (n, dim) float32")
            self.n, self.dim = X.shape
            check(lib().zi_vector_index_build(self.ctx.h, ptr(X, f32p), self.n, self.dim, dims, C.byref(h)))
        self.h = h
        d = C.c_int32()
        bms = C.c_double()
        check(lib().zi_vector_index_model(self.h, C.byref(d), None, None, None, None, None, C.byref(bms)))
        self.dims, self.build_ms = d.value, bms.value

    def model(self) -> dict:
        D, dim = self.dims, self.dim
        mean, comp, eig, lo, hi = np.zeros(dim), np.zeros((D, dim)), np.zeros(D), np.zeros(D), np.zeros(D)
        check(lib().zi_vector_index_model(self.h, None, ptr(mean, f64p), ptr(comp, f64p), ptr(eig, f64p),
                                          ptr(lo, f64p), ptr(hi, f64p), None))
        return {"mean": mean, "components": comp, "eigenvalues": eig, "lo": lo, "hi": hi}

    def index(self) -> "ZCurveIndex":
        h = C.c_void_p()
        check(lib().zi_vector_index_get_index(self.h, C.byref(h)))
        return ZCurveIndex(h, owner=self, ctx=self.ctx)

    def make_queries(self, Q, known) -> np.ndarray:
        Q = np.ascontiguousarray(Q, dtype=np.float32)
        kn = _u8(known)
        out = np.zeros((Q.shape[0], self.dims), dtype=np.uint8)
        check(lib().zi_vector_make_queries(self.h, ptr(Q, f32p), ptr(kn, u8p), Q.shape[0], ptr(out, u8p)))
        return out

    def knn(self, Q, known, k: int = 80, norm="l2"):
        Q = np.ascontiguousarray(Q, dtype=np.float32)
        kn = _u8(known)
        nq = Q.shape[0]
        out = np.zeros((nq, max(k, 1)), dtype=np.uint64)
        cnt = np.zeros(nq, dtype=np.uint32)
        check(lib().zi_vector_knn_batch(self.h, ptr(Q, f32p), ptr(kn, u8p), nq, k, _norm(norm), ptr(out, u64p),
                                        ptr(cnt, u32p)))
        return out, cnt

    def __del__(self):
        h = getattr(self, "h", None)
        try:
            if h:
                lib().zi_vector_index_destroy(h)
        except TypeError:  # interpreter shutdown
            pass
        self.h = None


# ------------------------------------------------------------------ multi-index
class MultiIndex:
    """multi_index::build (proj/src/builder.cpp:202-224): 8 layout indices, device resident."""

    def __init__(self, image, known, cfg: Optional[IndexConfig] = None, ctx: Optional[Context] = None, **kw):
        self.ctx = ctx or Context.default()
        self.cfg = cfg if cfg is not None else index_config(**kw)
        img = _u8(image)
        if img.ndim not in (2, 3):
            raise ValueError("image must be (H, W) or (H, W, 3) uint8")
        self.height, self.width = img.shape[:2]
        self.channels = 1 if img.ndim == 2 else img.shape[2]
        kn = _u8(known)
        if kn.shape != (self.height, self.width):
            raise ValueError("image/mask dimensions differ")
        self._img, self._known = img, kn
        h = C.c_void_p()
        check(lib().zi_multi_index_build(self.ctx.h, ptr(img, u8p), ptr(kn, u8p), self.width, self.height,
                                         self.channels, C.byref(self.cfg), C.byref(h)))
        self.h = h
        self._refresh_info()

    def save(self, path) -> None:
        """save_multi_index (proj/src/io_index.cpp:133-137): ZIDX1, eight blocks, layout 0 first."""
        check(lib().zi_multi_index_save(self.h, str(path).encode()))

    @classmethod
    def load(cls, path, image, known=None, ctx: Optional[Context] = None) -> "MultiIndex":
        """load_multi_index (proj/src/io_index.cpp:139-154) plus the image queries are refined
        against; `known` (optional) is kept as the default mask for inpaint()."""
        self = cls.__new__(cls)
        self.ctx = ctx or Context.default()
        img = _u8(image)
        if img.ndim not in (2, 3):
            raise ValueError("image must be (H, W) or (H, W, 3) uint8")
        self.height, self.width = img.shape[:2]
        self.channels = 1 if img.ndim == 2 else img.shape[2]
        self._img = img
        self._known = _u8(known) if known is not None else np.ones((self.height, self.width), np.uint8)
        h = C.c_void_p()
        check(lib().zi_multi_index_load(self.ctx.h, str(path).encode(), ptr(img, u8p), self.width, self.height,
                                        self.channels, C.byref(h)))
        self.h = h
        self._refresh_info()
        self.cfg = index_config(patch_size=self.info.patch_size, coverage=self.info.coverage, dims=self.dims)
        return self

    def _refresh_info(self):
        info = MultiIndexInfo()
        check(lib().zi_multi_index_get_info(self.h, C.byref(info)))
        self.info = info
        self.n, self.dims, self.m = info.n, info.dims, info.m

    def rebuild(self):
        check(lib().zi_multi_index_rebuild(self.h))
        self._refresh_info()

    @property
    def dictionary(self) -> np.ndarray:
        out = np.zeros(self.n, dtype=np.uint32)
        check(lib().zi_multi_index_dictionary(self.h, ptr(out, u32p)))
        return out

    def layout(self, l: int) -> dict:
        mc = self.m * self.channels
        rc = np.zeros((self.m, 2), dtype=np.int32)
        mean = np.zeros(mc)
        comp = np.zeros((self.dims, mc))
        eig = np.zeros(self.dims)
        lo = np.zeros(self.dims)
        hi = np.zeros(self.dims)
        check(lib().zi_multi_index_layout(self.h, l, ptr(rc, i32p), ptr(mean, f64p), ptr(comp, f64p),
                                          ptr(eig, f64p), ptr(lo, f64p), ptr(hi, f64p)))
        return {"id": l, "pixels": rc, "mean": mean, "components": comp, "eigenvalues": eig, "lo": lo, "hi": hi}

    def index_arrays(self, l: int):
        coords = np.zeros((self.n, self.dims), dtype=np.uint8)
        keys = np.zeros(self.n, dtype=np.uint32)
        check(lib().zi_multi_index_layout_index(self.h, l, ptr(coords, u8p), ptr(keys, u32p)))
        return coords, keys

    def index(self, l: int) -> ZCurveIndex:
        h = C.c_void_p()
        check(lib().zi_multi_index_get_index(self.h, l, C.byref(h)))
        return ZCurveIndex(h, owner=self)

    def moments(self):
        F = self.cfg.patch_size ** 2 * self.channels
        s = np.zeros(F, dtype=np.int64)
        S = np.zeros((F, F), dtype=np.int64)
        check(lib().zi_multi_index_moments(self.h, ptr(s, i64p), ptr(S, i64p)))
        return s, S

    def query_best_patch(self, target_values, target_known, k: Optional[int] = None, norm=None,
                         return_candidates: bool = False):
        """query_best_patch (proj/src/engine.cpp:178-213) -> (key, cost, error, layout_id, candidates)."""
        tv, tk = _u8(target_values), _u8(target_known)
        k = self.cfg.knn if k is None else k
        nrm = self.cfg.norm if norm is None else _norm(norm)
        bp = BestPatch()
        knn = np.zeros(max(1, min(max(k, 1), self.n)), dtype=np.uint64) if return_candidates else None
        check(lib().zi_query_best_patch(self.h, ptr(tv, u8p), ptr(tk, u8p), k, nrm, C.byref(bp),
                                        ptr(knn, u64p) if knn is not None else None))
        res = (bp.key, bp.cost, bp.error, bp.layout_id, bp.candidates)
        if return_candidates:
            return res, knn[:bp.candidates].copy()
        return res

    def make_query(self, layout: int, target_values, target_known) -> np.ndarray:
        """indices[layout].make_query (proj/src/builder.cpp:110-127), on the device."""
        tv, tk = _u8(target_values), _u8(target_known)
        out = np.zeros(self.dims, dtype=np.uint8)
        check(lib().zi_multi_index_make_query(self.h, layout, ptr(tv, u8p), ptr(tk, u8p), ptr(out, u8p)))
        return out

    def brute_force_best(self, target_values, target_known, norm=None):
        """brute_force_best (proj/src/engine.cpp:220-236) -> (key, cost, error)."""
        tv, tk = _u8(target_values), _u8(target_known)
        nrm = self.cfg.norm if norm is None else _norm(norm)
        bp = BestPatch()
        check(lib().zi_brute_force_best(self.h, ptr(tv, u8p), ptr(tk, u8p), nrm, C.byref(bp)))
        return bp.key, bp.cost, bp.error

    def inpaint(self, image=None, known=None, knn=None, norm=None, oracle=False, oracle_stride=1,
                brute_force=False):
        """inpaint with prebuilt indices (proj/include/zinpaint/engine.hpp:115-118)."""
        img = self._img if image is None else _u8(image)
        kn = self._known if known is None else _u8(known)
        cfg = IndexConfig(self.cfg.patch_size, self.cfg.coverage, self.cfg.dims,
                          self.cfg.knn if knn is None else knn, self.cfg.mu, self.cfg.nu,
                          self.cfg.norm if norm is None else _norm(norm))
        icfg = InpaintConfig(1, int(oracle), oracle_stride, int(brute_force))
        out = np.zeros_like(img)
        cap = int((kn == 0).sum()) + 1
        recs = (IterationRecord * cap)()
        nrec = C.c_uint64()
        stats = RunStats()
        check(lib().zi_inpaint_with_index(self.h, ptr(img, u8p), ptr(kn, u8p), C.byref(cfg), C.byref(icfg),
                                          ptr(out, u8p), recs, cap, C.byref(nrec), C.byref(stats)))
        return out, np.ctypeslib.as_array(recs)[:nrec.value].copy(), stats

    def __del__(self):
        h = getattr(self, "h", None)
        if h and not getattr(self, "_borrowed", False):
            lib().zi_multi_index_destroy(h)
        self.h = None


# ------------------------------------------------------------------ reference binding mirror
def _records_to_dicts(recs):
    out = []
    for r in recs:
        bf = float(r["bf_error"])
        out.append({"iteration": int(r["iteration"]), "target": (int(r["target_x"]), int(r["target_y"])),
                    "layout": int(r["layout_id"]),
                    "source": (int(r["source_key"]) & 0xFFFF, int(r["source_key"]) >> 16),
                    "z_error": float(r["z_error"]), "bf_error": None if math.isnan(bf) else bf,
                    "candidates": int(r["candidates"])})
    return out


def inpaint_raw(image, known, cfg: IndexConfig, brute_force=False, oracle=False, oracle_stride=1,
                ctx: Optional[Context] = None):
    """inpaint (proj/src/engine.cpp:442-480) on a 0/1 known mask; returns (image, records, stats)."""
    ctx = ctx or Context.default()
    img = _u8(image)
    if img.ndim not in (2, 3):
        raise ValueError("image must be (H, W) or (H, W, 3) uint8")
    h, w = img.shape[:2]
    ch = 1 if img.ndim == 2 else img.shape[2]
    kn = _u8(known)
    if kn.shape != (h, w):
        raise ValueError("inpaint: image/mask dimensions differ")
    icfg = InpaintConfig(1, int(oracle), oracle_stride, int(brute_force))
    out = np.zeros_like(img)
    cap = int((kn == 0).sum()) + 1
    recs = (IterationRecord * cap)()
    nrec = C.c_uint64()
    stats = RunStats()
    check(lib().zi_inpaint(ctx.h, ptr(img, u8p), ptr(kn, u8p), w, h, ch, C.byref(cfg), C.byref(icfg), ptr(out, u8p),
                           recs, cap, C.byref(nrec), C.byref(stats)))
    return out, np.ctypeslib.as_array(recs)[:nrec.value].copy(), stats


def inpaint(image, mask, patch_size=9, coverage=0.6, dims=10, knn=80, mu=256, nu=2048, norm="l2", workers=0,
            oracle=False):
    """Fill the unknown pixels of `image` (mask < 128) from its known parts.

    Mirrors ``zinpaint.inpaint`` (proj/python/bindings.cpp:55-98, :172-176).
    """
    img = _u8(image)
    if img.ndim not in (2, 3):
        raise ValueError("image must be (H, W) or (H, W, 3) uint8")
    if img.ndim == 3 and img.shape[2] not in (1, 3):
        raise ValueError("image must have 1 or 3 channels")
    if img.ndim == 3 and img.shape[2] == 1:
        img = img[:, :, 0]
    m = np.asarray(mask)
    if m.ndim != 2:
        raise ValueError("mask must be (H, W) uint8")
    known = (m >= 128).astype(np.uint8)  # bindings.cpp:38-40
    cfg = index_config(patch_size, coverage, dims, knn, mu, nu, norm)
    out, recs, stats = inpaint_raw(img, known, cfg, oracle=oracle)
    mean_ae = None if math.isnan(stats.mean_ae) else stats.mean_ae
    return {"image": out, "records": _records_to_dicts(recs),
            "stats": {"dictionary_size": int(stats.dictionary_size), "iterations": int(stats.iterations),
                      "build_wall_seconds": stats.build_wall_seconds, "inpaint_seconds": stats.inpaint_seconds,
                      "mean_ae": mean_ae}}


def knn_search(points, query, k, mu=256, norm="l2", workers=1):
    """Exact knn over byte points via the z-curve index; returns (distances, row indices).

    Mirrors ``zinpaint.knn_search`` (proj/python/bindings.cpp:100-142): row i is keyed as
    packed (x = i & 0xffff, y = i >> 16), so the packed key equals i.
    """
    pts = _u8(points)
    if pts.ndim != 2:
        raise ValueError("points must be (n, D) uint8")
    n, dims = pts.shape
    q = _u8(query)
    if q.ndim != 1 or q.shape[0] != dims:
        raise ValueError("query must be a (D,) uint8 vector")
    if n > 0xFFFFFFFF:
        raise ValueError("too many points")
    keys = np.arange(n, dtype=np.uint32)
    idx = ZCurveIndex.from_descriptors(pts, keys, dims)
    packed = idx.knn(q, k, mu, norm) if n else np.zeros(0, dtype=np.uint64)
    return (packed >> np.uint64(32)).astype(np.uint32), (packed & np.uint64(0xFFFFFFFF)).astype(np.uint64)
