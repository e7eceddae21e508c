"""CPU oracle for the SFC multi-index hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference`` arm) may import this package, and only as the checker or the timed CPU
baseline.  The product (``paper_1712_06326_b200``) never imports it.

Two libraries back it:

* ``libzoracle.so`` (``zoracle.cpp``): a restatement of the reference's Eigen-dependent code
  (``proj/src/builder.cpp``, ``pca.cpp``, ``engine.cpp``) with a pinned canonical fp64 order.
* ``_ref/libzref.so`` (``ref_shim.cpp`` + the reference's own unmodified
  ``proj/src/{zcurve,pool,layouts,image}.cpp``): the reference itself, for the parts that
  compile without Eigen.  Built by ``make -C oracle ref`` while ``/root/reference`` exists;
  the built ``.so`` travels to the GPU box.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_u8p = C.POINTER(C.c_uint8)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)

L2, L1 = 0, 1


def _p(a, t):
    return a.ctypes.data_as(t)


class Record(C.Structure):
    _fields_ = [("tx", C.c_int32), ("ty", C.c_int32), ("layout_id", C.c_int32), ("sx", C.c_int32),
                ("sy", C.c_int32), ("cost", C.c_uint32), ("z_error", C.c_double),
                ("bf_error", C.c_double), ("candidates", C.c_int64)]


_lib = None
_ref = None


def build(ref: bool = True) -> None:
    """Compile the oracle (and the reference shim when /root/reference exists)."""
    import subprocess
    subprocess.run(["make", "-s", "-C", _HERE, "all"], check=True)
    if ref and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", _HERE, "ref"], check=True)


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "libzoracle.so")
        if not os.path.exists(path):
            build(ref=False)
        L = C.CDLL(path)
        L.zo_subset_pixel_count.restype = C.c_int
        L.zo_subset_pixel_count.argtypes = [C.c_int, C.c_double]
        L.zo_build_subset_layouts.restype = C.c_int
        L.zo_build_subset_layouts.argtypes = [C.c_int, C.c_double, _ip]
        L.zo_less_msb.restype = C.c_int
        L.zo_morton_less.restype = C.c_int
        L.zo_morton_less.argtypes = [_u8p, _u8p, C.c_int]
        L.zo_collect_dictionary.restype = C.c_int64
        L.zo_collect_dictionary.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, _u32p]
        L.zo_patch_moments.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, _u32p, C.c_int64, _i64p, _i64p]
        L.zo_layout_covariance.argtypes = [_i64p, _i64p, C.c_int, C.c_int64, _ip, C.c_int, _f64p, _f64p]
        L.zo_pca_from_cov.restype = C.c_int
        L.zo_pca_from_cov.argtypes = [_f64p, C.c_int, C.c_int, _f64p, _f64p]
        _f32p = C.POINTER(C.c_float)
        L.zo_vec_mean_cov.argtypes = [_f32p, C.c_int64, C.c_int, C.c_int64, _f64p, _f64p]
        L.zo_vec_project.argtypes = [_f32p, C.c_int64, C.c_int, _f64p, _f64p, C.c_int, _f64p, _f64p, _u8p]
        L.zo_vec_make_query.argtypes = [_f32p, _u8p, C.c_int, _f64p, _f64p, _f64p, _f64p, C.c_int, _u8p]
        L.zo_quantize.restype = C.c_uint8
        L.zo_quantize.argtypes = [C.c_double, C.c_double, C.c_double]
        L.zo_project_build.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, _u32p, C.c_int64, _ip, C.c_int,
                                       _f64p, _f64p, C.c_int, _f64p, _f64p, _u8p, _f64p]
        L.zo_from_descriptors.restype = C.c_int
        L.zo_from_descriptors.argtypes = [_u8p, _u32p, C.c_int64, C.c_int, _u8p, _u32p]
        L.zo_knn_linear.restype = C.c_int64
        L.zo_knn_linear.argtypes = [_u8p, _u32p, C.c_int64, C.c_int, _u8p, C.c_int64, C.c_int, _u64p]
        L.zo_select_index.restype = C.c_int
        L.zo_select_index.argtypes = [_u8p, C.c_int, _ip, C.c_int]
        L.zo_make_query.argtypes = [_u8p, _u8p, C.c_int, C.c_int, _ip, C.c_int, _f64p, _f64p, _f64p, _f64p,
                                    C.c_int, _u8p]
        L.zo_masked_cost_at.restype = C.c_uint32
        L.zo_masked_cost_at.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, _u8p, _u8p, C.c_int, C.c_uint32, C.c_int]
        L.zo_brute_force_best.restype = C.c_uint64
        L.zo_brute_force_best.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, _u8p, _u8p, C.c_int, _u32p,
                                          C.c_int64, C.c_int]
        L.zo_extract_patch_clamped.argtypes = [_u8p, _u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                               C.c_int, _u8p, _u8p]
        L.zo_confidence_term.restype = C.c_double
        L.zo_confidence_term.argtypes = [_u8p, C.c_int, C.c_int, _f64p, C.c_int, C.c_int, C.c_int]
        L.zo_compute_priority.restype = C.c_double
        L.zo_compute_priority.argtypes = [_u8p, _u8p, C.c_int, C.c_int, C.c_int, _f64p, C.c_int, C.c_int,
                                          C.c_int]
        L.zo_mi_build.restype = C.c_void_p
        L.zo_mi_build.argtypes = [_u8p, _u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                  _f64p, _f64p, C.c_int, C.c_int]
        L.zo_mi_free.argtypes = [C.c_void_p]
        L.zo_mi_set_knn.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.zo_mi_set_layout.argtypes = [C.c_void_p, C.c_int, _f64p, _f64p, _f64p, _f64p, _u8p, _u32p]
        for fn in ("zo_mi_size",):
            getattr(L, fn).restype = C.c_int64
            getattr(L, fn).argtypes = [C.c_void_p]
        for fn in ("zo_mi_dims", "zo_mi_mc", "zo_mi_m"):
            getattr(L, fn).restype = C.c_int
            getattr(L, fn).argtypes = [C.c_void_p]
        L.zo_mi_dictionary.argtypes = [C.c_void_p, _u32p]
        L.zo_mi_layout.argtypes = [C.c_void_p, C.c_int, _ip]
        L.zo_mi_pca.argtypes = [C.c_void_p, C.c_int, _f64p, _f64p, _f64p, _f64p, _f64p]
        L.zo_mi_index.argtypes = [C.c_void_p, C.c_int, _u8p, _u32p]
        L.zo_mi_query_best_patch.restype = C.c_uint64
        L.zo_mi_query_best_patch.argtypes = [C.c_void_p, _u8p, _u8p, _u8p, C.c_int64, C.c_int, _ip, _i64p, _u64p]
        L.zo_inpaint.restype = C.c_int64
        L.zo_inpaint.argtypes = [C.c_void_p, _u8p, _u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64,
                                 C.c_int, C.c_int, C.c_int, C.c_int64, _u8p, C.POINTER(Record), C.c_int64,
                                 C.c_int64]
        L.zo_error.restype = C.c_char_p
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(os.path.join(_HERE, "_ref", "libzref.so"))


def ref():
    """The reference's own compiled zcurve/layouts/image code (oracle/_ref/libzref.so)."""
    global _ref
    if _ref is None:
        path = os.path.join(_HERE, "_ref", "libzref.so")
        if not os.path.exists(path):
            build(ref=True)
        R = C.CDLL(path)
        R.zr_less_msb.restype = C.c_int
        R.zr_morton_less.restype = C.c_int
        R.zr_morton_less.argtypes = [_u8p, _u8p, C.c_int]
        R.zr_layouts.restype = C.c_int
        R.zr_layouts.argtypes = [C.c_int, C.c_double, _ip]
        R.zr_index_create.restype = C.c_void_p
        R.zr_index_create.argtypes = [_u8p, _u32p, C.c_int64, C.c_int]
        R.zr_index_free.argtypes = [C.c_void_p]
        R.zr_index_export.argtypes = [C.c_void_p, _u8p, _u32p]
        R.zr_index_knn.restype = C.c_int64
        R.zr_index_knn.argtypes = [C.c_void_p, _u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _u64p]
        R.zr_index_knn_batch.restype = C.c_int64
        R.zr_index_knn_batch.argtypes = [C.c_void_p, _u8p, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.c_int, _u64p]
        R.zr_index_knn_batch_mt.restype = C.c_int64
        R.zr_index_knn_batch_mt.argtypes = [C.c_void_p, _u8p, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int,
                                            C.c_int, _u64p, _u32p]
        R.zr_hook_create.restype = C.c_void_p
        R.zr_hook_create.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int]
        R.zr_hook_free.argtypes = [C.c_void_p]
        R.zr_extract_patch_clamped.argtypes = [_u8p, _u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                               C.c_int, _u8p, _u8p]
        R.zr_fillfront.restype = C.c_int64
        R.zr_fillfront.argtypes = [_u8p, C.c_int, C.c_int, _ip]
        _ref = R
    return _ref


class RefIndex:
    """The reference's own ``zcurve_index`` (proj/src/zcurve.cpp, compiled unmodified into
    oracle/_ref/libzref.so): ``from_descriptors`` at construction, ``knn_search`` per query."""

    def __init__(self, coords, keys):
        coords = np.ascontiguousarray(coords, dtype=np.uint8)
        keys = np.ascontiguousarray(keys, dtype=np.uint32)
        self.n, self.dims = coords.shape
        self.h_ = ref().zr_index_create(_p(coords, _u8p), _p(keys, _u32p), self.n, self.dims)
        if not self.h_:
            raise ValueError("zcurve_index::from_descriptors rejected the input")

    def __del__(self):
        h = getattr(self, "h_", None)
        if h:
            ref().zr_index_free(h)
            self.h_ = None

    def export(self):
        c = np.zeros((self.n, self.dims), dtype=np.uint8)
        k = np.zeros(self.n, dtype=np.uint32)
        ref().zr_index_export(self.h_, _p(c, _u8p), _p(k, _u32p))
        return c, k

    def knn(self, query, k, norm=L2, mu=256, nu=2048, workers=1):
        q = np.ascontiguousarray(query, dtype=np.uint8)
        out = np.zeros(max(1, k), dtype=np.uint64)
        cnt = ref().zr_index_knn(self.h_, _p(q, _u8p), k, mu, nu, norm, workers, _p(out, _u64p))
        return out[:cnt].copy()

    def knn_batch(self, queries, k, norm=L2, mu=256, nu=2048, threads=None):
        """(packed nq x k, counts nq); queries split over host threads, sequential traversal each."""
        q = np.ascontiguousarray(queries, dtype=np.uint8)
        nq = q.shape[0]
        out = np.zeros((nq, max(1, k)), dtype=np.uint64)
        cnt = np.zeros(nq, dtype=np.uint32)
        threads = threads or (os.cpu_count() or 1)
        ref().zr_index_knn_batch_mt(self.h_, _p(q, _u8p), nq, k, mu, nu, norm, threads, _p(out, _u64p),
                                    _p(cnt, _u32p))
        return out, cnt


def ref_from_descriptors(coords, keys):
    """Sorted (coords, keys) from the reference's compiled ``from_descriptors``."""
    return RefIndex(coords, keys).export()


# ------------------------------------------------------------------ numpy-level helpers
def _u8(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


def subset_layouts(K: int, coverage: float) -> np.ndarray:
    """(8, m, 2) int32 (row, col) offsets -- restates proj/src/layouts.cpp:13-60."""
    m = lib().zo_subset_pixel_count(K, coverage)
    out = np.zeros((8, max(m, 1), 2), dtype=np.int32)
    got = lib().zo_build_subset_layouts(K, coverage, _p(out, _ip))
    if got < 0:
        raise ValueError(lib().zo_error().decode())
    return out


def morton_less(a, b) -> bool:
    a, b = _u8(a), _u8(b)
    return bool(lib().zo_morton_less(_p(a, _u8p), _p(b, _u8p), a.size))


def collect_dictionary(known: np.ndarray, K: int) -> np.ndarray:
    known = _u8(known)
    h, w = known.shape
    out = np.zeros(max(w * h, 1), dtype=np.uint32)
    n = lib().zo_collect_dictionary(_p(known, _u8p), w, h, K, _p(out, _u32p))
    return out[:n].copy()


def _img_dims(img):
    img = _u8(img)
    h, w = img.shape[:2]
    ch = 1 if img.ndim == 2 else img.shape[2]
    return img, w, h, ch


def patch_moments(img, K, keys):
    img, w, h, ch = _img_dims(img)
    keys = np.ascontiguousarray(keys, dtype=np.uint32)
    F = K * K * ch
    s = np.zeros(F, dtype=np.int64)
    S = np.zeros((F, F), dtype=np.int64)
    lib().zo_patch_moments(_p(img, _u8p), w, h, ch, K, _p(keys, _u32p), keys.size, _p(s, _i64p), _p(S, _i64p))
    return s, S


def layout_columns(rc: np.ndarray, K: int, ch: int) -> np.ndarray:
    return np.array([(r * K + c) * ch + k for r, c in rc for k in range(ch)], dtype=np.int32)


def layout_covariance(s, S, n, cols):
    cols = np.ascontiguousarray(cols, dtype=np.int32)
    mc = cols.size
    mean = np.zeros(mc)
    cov = np.zeros((mc, mc))
    s = np.ascontiguousarray(s, dtype=np.int64)
    S = np.ascontiguousarray(S, dtype=np.int64)
    lib().zo_layout_covariance(_p(s, _i64p), _p(S, _i64p), s.size, n, _p(cols, _ip), mc, _p(mean, _f64p),
                               _p(cov, _f64p))
    return mean, cov


def pca_from_cov(cov, D):
    cov = np.ascontiguousarray(cov, dtype=np.float64)
    mc = cov.shape[0]
    comp = np.zeros((D, mc))
    eig = np.zeros(D)
    if lib().zo_pca_from_cov(_p(cov, _f64p), mc, D, _p(comp, _f64p), _p(eig, _f64p)) != 0:
        raise ValueError(lib().zo_error().decode())
    return comp, eig


def quantize(lo, hi, y) -> int:
    return int(lib().zo_quantize(lo, hi, y))


def project_build(img, keys, rc, mean, comp):
    img, w, h, ch = _img_dims(img)
    keys = np.ascontiguousarray(keys, dtype=np.uint32)
    rc = np.ascontiguousarray(rc, dtype=np.int32)
    mean = np.ascontiguousarray(mean, dtype=np.float64)
    comp = np.ascontiguousarray(comp, dtype=np.float64)
    D = comp.shape[0]
    n = keys.size
    lo = np.zeros(D)
    hi = np.zeros(D)
    coords = np.zeros((n, D), dtype=np.uint8)
    y = np.zeros((n, D))
    lib().zo_project_build(_p(img, _u8p), w, h, ch, _p(keys, _u32p), n, _p(rc, _ip), rc.shape[0],
                           _p(mean, _f64p), _p(comp, _f64p), D, _p(lo, _f64p), _p(hi, _f64p),
                           _p(coords, _u8p), _p(y, _f64p))
    return lo, hi, coords, y


def from_descriptors(coords, keys):
    coords = _u8(coords)
    keys = np.ascontiguousarray(keys, dtype=np.uint32)
    n, D = coords.shape
    co = np.zeros_like(coords)
    ko = np.zeros_like(keys)
    if lib().zo_from_descriptors(_p(coords, _u8p), _p(keys, _u32p), n, D, _p(co, _u8p), _p(ko, _u32p)) != 0:
        raise ValueError(lib().zo_error().decode())
    return co, ko


def knn_linear(coords, keys, query, k, norm=L2):
    coords = _u8(coords)
    keys = np.ascontiguousarray(keys, dtype=np.uint32)
    query = _u8(query)
    n, D = coords.shape
    out = np.zeros(max(1, min(max(k, 1), n)), dtype=np.uint64)
    cnt = lib().zo_knn_linear(_p(coords, _u8p), _p(keys, _u32p), n, D, _p(query, _u8p), k, norm, _p(out, _u64p))
    return out[:cnt].copy()


def make_query(tv, tk, K, C, rc, mean, comp, lo, hi):
    """patch_index::make_query (proj/src/builder.cpp:110-127): D quantised bytes."""
    tv, tk = _u8(tv), _u8(tk)
    rc = np.ascontiguousarray(rc, dtype=np.int32)
    comp = np.ascontiguousarray(comp, dtype=np.float64)
    D = comp.shape[0]
    out = np.zeros(D, dtype=np.uint8)
    lib().zo_make_query(_p(tv, _u8p), _p(tk, _u8p), K, C, _p(rc, _ip), rc.shape[0],
                        _p(np.ascontiguousarray(mean, dtype=np.float64), _f64p), _p(comp, _f64p),
                        _p(np.ascontiguousarray(lo, dtype=np.float64), _f64p),
                        _p(np.ascontiguousarray(hi, dtype=np.float64), _f64p), D, _p(out, _u8p))
    return out


def masked_cost_at(img, tv, tk, K, key, norm=L2):
    img, w, h, ch = _img_dims(img)
    tv, tk = _u8(tv), _u8(tk)
    return int(lib().zo_masked_cost_at(_p(img, _u8p), w, h, ch, _p(tv, _u8p), _p(tk, _u8p), K, int(key), norm))


def brute_force_best(img, tv, tk, K, keys, norm=L2) -> int:
    img, w, h, ch = _img_dims(img)
    tv, tk = _u8(tv), _u8(tk)
    keys = np.ascontiguousarray(keys, dtype=np.uint32)
    return int(lib().zo_brute_force_best(_p(img, _u8p), w, h, ch, _p(tv, _u8p), _p(tk, _u8p), K,
                                         _p(keys, _u32p), keys.size, norm))


def extract_patch_clamped(img, known, cx, cy, K):
    img, w, h, ch = _img_dims(img)
    known = _u8(known)
    tv = np.zeros(K * K * ch, dtype=np.uint8)
    tk = np.zeros(K * K, dtype=np.uint8)
    lib().zo_extract_patch_clamped(_p(img, _u8p), _p(known, _u8p), w, h, ch, cx, cy, K, _p(tv, _u8p), _p(tk, _u8p))
    return tv, tk


def compute_priority(img, known, conf, cx, cy, K):
    img, w, h, ch = _img_dims(img)
    known = _u8(known)
    conf = np.ascontiguousarray(conf, dtype=np.float64)
    return lib().zo_compute_priority(_p(img, _u8p), _p(known, _u8p), w, h, ch, _p(conf, _f64p), cx, cy, K)


def confidence_term(known, conf, cx, cy, K):
    known = _u8(known)
    h, w = known.shape
    conf = np.ascontiguousarray(conf, dtype=np.float64)
    return lib().zo_confidence_term(_p(known, _u8p), w, h, _p(conf, _f64p), cx, cy, K)


@dataclass
class LayoutIndex:
    rc: np.ndarray
    mean: np.ndarray
    comp: np.ndarray
    eig: np.ndarray
    lo: np.ndarray
    hi: np.ndarray
    coords: np.ndarray
    keys: np.ndarray


class MultiIndex:
    """Restated ``multi_index::build`` (proj/src/builder.cpp:202-224)."""

    def __init__(self, img, known, K=9, coverage=0.6, dims=10, pca_mean=None, pca_comp=None, layouts=None,
                 threads=None):
        """layouts: the layout ids to build (default all 8; the others stay empty); threads:
        layouts built concurrently (default: one per host core, at most 8)."""
        self.img, self.w, self.h, self.ch = _img_dims(img)
        self.known = _u8(known)
        self.K = K
        L = lib()
        pm = pc = None
        if pca_mean is not None:
            self._pm = np.ascontiguousarray(pca_mean, dtype=np.float64)
            self._pc = np.ascontiguousarray(pca_comp, dtype=np.float64)
            pm, pc = _p(self._pm, _f64p), _p(self._pc, _f64p)
        mask = 0xFF if layouts is None else sum(1 << int(l) for l in layouts)
        if threads is None:
            threads = min(8, os.cpu_count() or 1)
        self.h_ = L.zo_mi_build(_p(self.img, _u8p), _p(self.known, _u8p), self.w, self.h, self.ch, K, coverage,
                                dims, pm, pc, mask, threads)
        if not self.h_:
            raise ValueError(L.zo_error().decode())
        self.n = L.zo_mi_size(self.h_)
        self.dims = L.zo_mi_dims(self.h_)
        self.mc = L.zo_mi_mc(self.h_)
        self.m = L.zo_mi_m(self.h_)

    def __del__(self):
        h = getattr(self, "h_", None)
        if h:
            lib().zo_mi_free(h)
            self.h_ = None
        hk = getattr(self, "_hook", None)
        if hk:
            ref().zr_hook_free(hk)
            self._hook = None

    def dictionary(self):
        out = np.zeros(self.n, dtype=np.uint32)
        lib().zo_mi_dictionary(self.h_, _p(out, _u32p))
        return out

    def index(self, l) -> LayoutIndex:
        L = lib()
        rc = np.zeros((self.m, 2), dtype=np.int32)
        L.zo_mi_layout(self.h_, l, _p(rc, _ip))
        mean = np.zeros(self.mc)
        comp = np.zeros((self.dims, self.mc))
        eig = np.zeros(self.dims)
        lo = np.zeros(self.dims)
        hi = np.zeros(self.dims)
        L.zo_mi_pca(self.h_, l, _p(mean, _f64p), _p(comp, _f64p), _p(eig, _f64p), _p(lo, _f64p), _p(hi, _f64p))
        coords = np.zeros((self.n, self.dims), dtype=np.uint8)
        keys = np.zeros(self.n, dtype=np.uint32)
        L.zo_mi_index(self.h_, l, _p(coords, _u8p), _p(keys, _u32p))
        return LayoutIndex(rc, mean, comp, eig, lo, hi, coords, keys)

    def set_layout(self, l, mean, comp, lo, hi, coords, keys):
        """Replace layout l's model, quantiser and sorted index (e.g. with a device build's)."""
        self._keep = getattr(self, "_keep", {})
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (mean, comp, lo, hi)]
        coords = np.ascontiguousarray(coords, dtype=np.uint8)
        keys = np.ascontiguousarray(keys, dtype=np.uint32)
        lib().zo_mi_set_layout(self.h_, l, *[_p(a, _f64p) for a in arrs], _p(coords, _u8p), _p(keys, _u32p))

    def use_reference_knn(self, workers=None, mu=256, nu=2048):
        """Answer the fill loop's k-NN queries with the reference's compiled knn_search over its own
        zcurve_index per layout (built by the compiled from_descriptors from this index's arrays),
        on a priority_pool of workers - 1 threads (run_loop's default: workers = host cores)."""
        import threading
        workers = workers or (os.cpu_count() or 1)
        refs = [None] * 8
        def mk(l):
            ix = self.index(l)
            refs[l] = RefIndex(ix.coords, ix.keys)
        th = [threading.Thread(target=mk, args=(l,)) for l in range(8)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        handles = (C.c_void_p * 8)(*[r.h_ for r in refs])
        self._refs = refs
        self._hook = ref().zr_hook_create(handles, workers, mu, nu)
        fn = C.cast(ref().zr_hook_knn, C.c_void_p)
        lib().zo_mi_set_knn(self.h_, fn, self._hook)
        self._hook_fn = fn
        return workers

    def query_best_patch(self, img, tv, tk, k, norm=L2):
        img = _u8(img)
        tv, tk = _u8(tv), _u8(tk)
        lid = C.c_int()
        nc = C.c_int64()
        knn = np.zeros(max(1, min(k, self.n)), dtype=np.uint64)
        best = lib().zo_mi_query_best_patch(self.h_, _p(img, _u8p), _p(tv, _u8p), _p(tk, _u8p), k, norm,
                                            C.byref(lid), C.byref(nc), _p(knn, _u64p))
        return int(best), lid.value, nc.value, knn[:nc.value].copy()


def inpaint(img, known, K=9, coverage=0.6, dims=10, knn=80, norm=L2, brute_force=False, oracle=False,
            oracle_stride=1, mi: MultiIndex | None = None, pca_mean=None, pca_comp=None, max_iter=0):
    """Restated ``inpaint`` / ``run_loop`` (proj/src/engine.cpp:371-506).

    max_iter > 0 stops after that many iterations (the first records of the full run).
    Returns (image_out, records ndarray of Record).
    """
    img, w, h, ch = _img_dims(img)
    known = _u8(known)
    if mi is None and not brute_force and (known == 0).any():
        mi = MultiIndex(img, known, K, coverage, dims, pca_mean, pca_comp)
    out = np.zeros_like(img)
    cap = int((known == 0).sum()) + 1
    if max_iter > 0:
        cap = min(cap, int(max_iter))
    recs = (Record * cap)()
    n = lib().zo_inpaint(mi.h_ if mi is not None else None, _p(img, _u8p), _p(known, _u8p), w, h, ch, K, knn,
                         norm, int(brute_force), int(oracle), oracle_stride, _p(out, _u8p), recs, cap,
                         int(max_iter))
    if n < 0:
        raise RuntimeError(lib().zo_error().decode())
    arr = np.ctypeslib.as_array(recs)[:n].copy()
    return out, arr


# ------------------------------------------------------------------ cfg5 vector index
VEC_STRIPE = 32768  # canonical stripe of paper_1712_06326_b200/csrc/k_vector.cu


def vec_mean_cov(X, stripe=VEC_STRIPE):
    """Mean and covariance of fp32 rows in the device build's canonical fp64 order."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    n, dim = X.shape
    mean = np.zeros(dim)
    cov = np.zeros((dim, dim))
    lib().zo_vec_mean_cov(X.ctypes.data_as(C.POINTER(C.c_float)), n, dim, stripe, _p(mean, _f64p), _p(cov, _f64p))
    return mean, cov


def vec_project(X, mean, comp):
    """(lo, hi, coords n x D) -- projection + quantiser of the vector index (canonical order)."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    n, dim = X.shape
    mean = np.ascontiguousarray(mean, dtype=np.float64)
    comp = np.ascontiguousarray(comp, dtype=np.float64)
    D = comp.shape[0]
    lo, hi = np.zeros(D), np.zeros(D)
    coords = np.zeros((n, D), dtype=np.uint8)
    lib().zo_vec_project(X.ctypes.data_as(C.POINTER(C.c_float)), n, dim, _p(mean, _f64p), _p(comp, _f64p), D,
                         _p(lo, _f64p), _p(hi, _f64p), _p(coords, _u8p))
    return lo, hi, coords


def vec_make_query(x, known, mean, comp, lo, hi):
    x = np.ascontiguousarray(x, dtype=np.float32)
    known = _u8(known)
    D = comp.shape[0]
    out = np.zeros(D, dtype=np.uint8)
    lib().zo_vec_make_query(x.ctypes.data_as(C.POINTER(C.c_float)), _p(known, _u8p), x.shape[0],
                            _p(np.ascontiguousarray(mean, dtype=np.float64), _f64p),
                            _p(np.ascontiguousarray(comp, dtype=np.float64), _f64p),
                            _p(np.ascontiguousarray(lo, dtype=np.float64), _f64p),
                            _p(np.ascontiguousarray(hi, dtype=np.float64), _f64p), D, _p(out, _u8p))
    return out
