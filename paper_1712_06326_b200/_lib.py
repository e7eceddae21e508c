"""ctypes binding of the C ABI in include/zinpaint_b200.h (libzinpaint_b200.so).

The library is built in-tree (``__graft_entry__.build()`` / ``make -C paper_1712_06326_b200/csrc``)
and there is no fallback: if it is missing every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ZI_LIB_PATH") or os.path.join(HERE, "libzinpaint_b200.so")  # ZI_LIB_PATH: dev A/B of a variant build

u8p = C.POINTER(C.c_uint8)
f32p = C.POINTER(C.c_float)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)
vp = C.c_void_p

ZI_OK, ZI_E_INVALID, ZI_E_EMPTY_DICT, ZI_E_RUNTIME, ZI_E_RANGE, ZI_E_CUDA, ZI_E_OOM = range(7)


class IndexConfig(C.Structure):
    """index_config (proj/include/zinpaint/builder.hpp:24-34)."""
    _fields_ = [("patch_size", C.c_int32), ("coverage", C.c_double), ("dims", C.c_int32), ("knn", C.c_int32),
                ("mu", C.c_uint32), ("nu", C.c_uint32), ("norm", C.c_int32)]


class InpaintConfig(C.Structure):
    _fields_ = [("workers", C.c_int32), ("oracle", C.c_int32), ("oracle_stride", C.c_uint64),
                ("brute_force", C.c_int32)]


class BestPatch(C.Structure):
    _fields_ = [("key", C.c_uint32), ("cost", C.c_uint32), ("error", C.c_double), ("layout_id", C.c_uint32),
                ("candidates", C.c_uint64)]


class IterationRecord(C.Structure):
    _fields_ = [("iteration", C.c_uint64), ("target_x", C.c_int32), ("target_y", C.c_int32),
                ("layout_id", C.c_uint32), ("source_key", C.c_uint32), ("cost", C.c_uint32), ("pad_", C.c_uint32),
                ("z_error", C.c_double), ("bf_error", C.c_double), ("candidates", C.c_uint64),
                ("elapsed_seconds", C.c_double)]


class RunStats(C.Structure):
    _fields_ = [("dictionary_size", C.c_uint64), ("sort_seconds", C.c_double), ("build_wall_seconds", C.c_double),
                ("inpaint_seconds", C.c_double), ("iterations", C.c_uint64), ("mean_ae", C.c_double),
                ("ae_excluded", C.c_uint64), ("confidence_low", C.c_double), ("confidence_high", C.c_double)]


class MultiIndexInfo(C.Structure):
    _fields_ = [("n", C.c_uint64), ("dims", C.c_int32), ("m", C.c_int32), ("channels", C.c_int32),
                ("patch_size", C.c_int32), ("width", C.c_int32), ("height", C.c_int32),
                ("build_seconds", C.c_double), ("eigen_seconds", C.c_double),
                ("pca_on_device", C.c_int32), ("coverage", C.c_double), ("loaded", C.c_int32)]


# name -> (restype, argtypes); mirrors include/zinpaint_b200.h one to one
SIGNATURES = {
    "zi_last_error": (C.c_char_p, []),
    "zi_version": (C.c_char_p, []),
    "zi_ctx_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
    "zi_ctx_destroy": (C.c_int, [vp]),
    "zi_ctx_synchronize": (C.c_int, [vp]),
    "zi_timer_start": (C.c_int, [vp]),
    "zi_timer_stop": (C.c_int, [vp, f64p]),
    "zi_ctx_kernel_launches": (C.c_uint64, [vp]),
    "zi_ctx_flush_l2": (C.c_int, [vp]),
    "zi_ctx_set_profiling": (C.c_int, [vp, C.c_int]),
    "zi_ctx_profile": (C.c_int, [vp, C.c_int, f64p, u64p, C.POINTER(C.c_char_p)]),
    "zi_ctx_set_profile_filter": (C.c_int, [vp, C.c_char_p]),
    "zi_ctx_set_sort_policy": (C.c_int, [vp, C.c_int32, C.c_int32]),
    "zi_less_most_significant_bit": (C.c_int, [C.c_int, C.c_int]),
    "zi_morton_less": (C.c_int, [u8p, u8p, C.c_uint32]),
    "zi_subset_pixel_count": (C.c_int, [C.c_int, C.c_double]),
    "zi_subset_layouts": (C.c_int, [C.c_int, C.c_double, i32p, i32p]),
    "zi_subset_layout_anchors": (C.c_int, [C.c_int, i32p]),
    "zi_index_config_validate": (C.c_int, [C.POINTER(IndexConfig), C.c_int]),
    "zi_index_config_default": (None, [C.POINTER(IndexConfig)]),
    "zi_index_from_descriptors": (C.c_int, [vp, u8p, u32p, C.c_uint64, C.c_uint32, C.c_uint32, C.POINTER(vp)]),
    "zi_index_destroy": (C.c_int, [vp]),
    "zi_index_size": (C.c_int, [vp, u64p, C.POINTER(C.c_uint32)]),
    "zi_index_export": (C.c_int, [vp, u8p, u32p]),
    "zi_knn_search": (C.c_int, [vp, u8p, C.c_uint32, C.c_uint32, C.c_int32, u64p, C.POINTER(C.c_uint32)]),
    "zi_knn_search_batch": (C.c_int, [vp, u8p, C.c_uint64, C.c_uint32, C.c_int32, u64p, C.POINTER(C.c_uint32)]),
    "zi_knn_batch_bench": (C.c_int, [vp, u8p, C.c_uint64, C.c_uint32, C.c_int32, C.c_int32, f64p, u64p, u64p,
                                     C.POINTER(C.c_uint32)]),
    "zi_index_build": (C.c_int, [vp, u8p, C.c_int32, C.c_int32, C.c_int32, u32p, C.c_uint64, i32p, C.c_int32,
                                 C.POINTER(IndexConfig), C.POINTER(vp)]),
    "zi_patch_index_destroy": (C.c_int, [vp]),
    "zi_patch_index_model": (C.c_int, [vp, i32p, i32p, f64p, f64p, f64p, f64p, f64p, f64p, f64p]),
    "zi_patch_index_get_index": (C.c_int, [vp, C.POINTER(vp)]),
    "zi_make_query": (C.c_int, [vp, u8p, u8p, u8p]),
    "zi_multi_index_make_query": (C.c_int, [vp, C.c_int32, u8p, u8p, u8p]),
    "zi_brute_force_scan": (C.c_int, [vp, u8p, C.c_int32, C.c_int32, C.c_int32, u32p, C.c_uint64, u8p, u8p,
                                      C.c_int32, C.c_int32, C.POINTER(BestPatch)]),
    "zi_dictionary_collect": (C.c_int, [vp, u8p, C.c_int32, C.c_int32, C.c_int32, u32p, C.c_uint64, u64p]),
    "zi_multi_index_build": (C.c_int, [vp, u8p, u8p, C.c_int32, C.c_int32, C.c_int32, C.POINTER(IndexConfig),
                                       C.POINTER(vp)]),
    "zi_multi_index_build_to": (C.c_int, [vp, u8p, u8p, C.c_int32, C.c_int32, C.c_int32, C.POINTER(IndexConfig),
                                          u32p, C.c_uint64, u64p, C.POINTER(vp)]),
    "zi_multi_index_rebuild": (C.c_int, [vp]),
    "zi_vector_index_build": (C.c_int, [vp, f32p, C.c_uint64, C.c_int32, C.c_int32, C.POINTER(vp)]),
    "zi_vector_index_build_device": (C.c_int, [vp, vp, C.c_uint64, C.c_int32, C.c_int32, C.POINTER(vp)]),
    "zi_vector_index_destroy": (C.c_int, [vp]),
    "zi_vector_index_model": (C.c_int, [vp, i32p, f64p, f64p, f64p, f64p, f64p, f64p]),
    "zi_vector_index_get_index": (C.c_int, [vp, C.POINTER(vp)]),
    "zi_vector_make_queries": (C.c_int, [vp, f32p, u8p, C.c_uint64, u8p]),
    "zi_vector_knn_batch": (C.c_int, [vp, f32p, u8p, C.c_uint64, C.c_uint32, C.c_int32, u64p, u32p]),
    "zi_multi_index_save": (C.c_int, [vp, C.c_char_p]),
    "zi_multi_index_load": (C.c_int, [vp, C.c_char_p, u8p, C.c_int32, C.c_int32, C.c_int32, C.POINTER(vp)]),
    "zi_multi_index_destroy": (C.c_int, [vp]),
    "zi_multi_index_get_info": (C.c_int, [vp, C.POINTER(MultiIndexInfo)]),
    "zi_multi_index_dictionary": (C.c_int, [vp, u32p]),
    "zi_multi_index_layout": (C.c_int, [vp, C.c_int32, i32p, f64p, f64p, f64p, f64p, f64p]),
    "zi_multi_index_layout_index": (C.c_int, [vp, C.c_int32, u8p, u32p]),
    "zi_multi_index_get_index": (C.c_int, [vp, C.c_int32, C.POINTER(vp)]),
    "zi_multi_index_moments": (C.c_int, [vp, i64p, i64p]),
    "zi_query_best_patch": (C.c_int, [vp, u8p, u8p, C.c_uint32, C.c_int32, C.POINTER(BestPatch), u64p]),
    "zi_brute_force_best": (C.c_int, [vp, u8p, u8p, C.c_int32, C.POINTER(BestPatch)]),
    "zi_refine_best": (C.c_int, [vp, u8p, u8p, u64p, C.c_uint32, C.c_int32, C.POINTER(BestPatch)]),
    "zi_shard_create": (C.c_int, [vp, u8p, u8p, C.c_int32, C.c_int32, C.c_int32, C.POINTER(IndexConfig), C.c_int32,
                                  C.c_int32, C.POINTER(vp)]),
    "zi_shard_destroy": (C.c_int, [vp]),
    "zi_shard_rebuild": (C.c_int, [vp]),
    "zi_shard_finish_local": (C.c_int, [vp]),
    "zi_shard_info": (C.c_int, [vp, u64p]),
    "zi_shard_moments": (C.c_int, [vp, i64p]),
    "zi_shard_fit_project": (C.c_int, [vp, i64p, i64p, i64p]),
    "zi_shard_refine_ranges": (C.c_int, [vp, i64p, i64p, i64p, i64p]),
    "zi_shard_quantize_sort": (C.c_int, [vp, i64p, i64p, C.c_uint32, u32p]),
    "zi_shard_splitters": (C.c_int, [u32p, C.c_uint64, C.c_int32, C.c_int32, u32p]),
    "zi_shard_partition": (C.c_int, [vp, u32p, u64p, C.POINTER(vp)]),
    "zi_shard_rebalance_plan": (C.c_int, [u64p, C.c_int32, C.c_uint64, C.c_int32, u64p, u64p]),
    "zi_shard_receive": (C.c_int, [vp, vp, u64p, u64p, C.POINTER(vp)]),
    "zi_shard_finish": (C.c_int, [vp, vp, u64p]),
    "zi_shard_multi_index": (C.c_int, [vp, C.POINTER(vp)]),
    "zi_inpaint": (C.c_int, [vp, u8p, u8p, C.c_int32, C.c_int32, C.c_int32, C.POINTER(IndexConfig),
                             C.POINTER(InpaintConfig), u8p, C.POINTER(IterationRecord), C.c_uint64, u64p,
                             C.POINTER(RunStats)]),
    "zi_inpaint_with_index": (C.c_int, [vp, u8p, u8p, C.POINTER(IndexConfig), C.POINTER(InpaintConfig), u8p,
                                        C.POINTER(IterationRecord), C.c_uint64, u64p, C.POINTER(RunStats)]),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
                               " -- there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class ZIError(RuntimeError):
    pass


class EmptyDictionaryError(RuntimeError):
    """empty_dictionary_error (proj/include/zinpaint/builder.hpp:19-22)."""


def check(status: int) -> None:
    if status == ZI_OK:
        return
    msg = lib().zi_last_error().decode()
    if status == ZI_E_INVALID:
        raise ValueError(msg)
    if status == ZI_E_EMPTY_DICT:
        raise EmptyDictionaryError(msg)
    if status == ZI_E_RANGE:
        raise IndexError(msg)
    if status == ZI_E_OOM:
        raise MemoryError(msg)
    raise ZIError(f"[{status}] {msg}")


def ptr(a, t):
    return a.ctypes.data_as(t)
