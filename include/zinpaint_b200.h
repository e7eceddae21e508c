/*
 * zinpaint_b200.h -- the drop-in C ABI of the B200-native SFC multi-index hot path.
 *
 * The reference (`zinpaint`, /root/reference/proj) has no C ABI: its hot path sits behind
 * C++ free functions and value types (proj/include/zinpaint/{zcurve,builder,engine}.hpp) and
 * a pybind11 module (proj/python/bindings.cpp).  Every entry point below names the reference
 * interface it replaces (file:line).  Plain pointers and sizes only; all buffers are HOST
 * buffers owned by the caller; device memory is owned by the opaque handles.  No exception
 * crosses this boundary: every call returns a zi_status and zi_last_error() explains it.
 * The C++ mirror of the reference API (include/zinpaint_b200.hpp) rethrows the reference's
 * exception types from these codes.
 */
#ifndef ZINPAINT_B200_H
#define ZINPAINT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes; the C++ mirror maps them back to the reference's exceptions ---- */
typedef enum {
    ZI_OK = 0,
    ZI_E_INVALID = 1,    /* std::invalid_argument   (proj/src/builder.cpp:38-53, zcurve.cpp:111-114) */
    ZI_E_EMPTY_DICT = 2, /* empty_dictionary_error  (proj/include/zinpaint/builder.hpp:19-22) */
    ZI_E_RUNTIME = 3,    /* std::runtime_error      (proj/src/engine.cpp:387-388) */
    ZI_E_RANGE = 4,      /* std::out_of_range       (proj/src/image.cpp:12-13) */
    ZI_E_CUDA = 5,       /* CUDA runtime failure (no reference counterpart) */
    ZI_E_OOM = 6         /* device allocation failure */
} zi_status;

typedef enum { ZI_NORM_L2 = 0, ZI_NORM_L1 = 1 } zi_norm; /* norm_kind (types.hpp:7) */

/* index_config (proj/include/zinpaint/builder.hpp:24-34); defaults 9/0.6/10/80/256/2048/L2 */
typedef struct {
    int32_t patch_size;
    double coverage;
    int32_t dims;
    int32_t knn;
    uint32_t mu; /* accepted and validated; the GPU search does not traverse by leaves */
    uint32_t nu; /* accepted and validated; no CPU thread pool on the GPU path */
    int32_t norm;
} zi_index_config;

/* inpaint_config (proj/include/zinpaint/engine.hpp:25-31) minus the index part */
typedef struct {
    int32_t workers; /* accepted; the GPU path has no CPU worker pool */
    int32_t oracle;  /* run the exhaustive scan beside the index every oracle_stride iterations */
    uint64_t oracle_stride;
    int32_t brute_force; /* replace the index query with the exhaustive scan */
} zi_inpaint_config;

/* best_patch (proj/include/zinpaint/engine.hpp:52-58) */
typedef struct {
    uint32_t key; /* packed y<<16 | x (types.hpp:15-17) */
    uint32_t cost;
    double error;
    uint32_t layout_id;
    uint64_t candidates;
} zi_best_patch;

/* iteration_record (proj/include/zinpaint/engine.hpp:14-23); bf_error is NaN when absent */
typedef struct {
    uint64_t iteration;
    int32_t target_x, target_y;
    uint32_t layout_id;
    uint32_t source_key;
    uint32_t cost;
    uint32_t pad_;
    double z_error;
    double bf_error;
    uint64_t candidates;
    double elapsed_seconds;
} zi_iteration_record;

/* run_stats (proj/include/zinpaint/engine.hpp:33-44); mean_ae is NaN when absent */
typedef struct {
    uint64_t dictionary_size;
    double sort_seconds;
    double build_wall_seconds;
    double inpaint_seconds;
    uint64_t iterations;
    double mean_ae;
    uint64_t ae_excluded;
    double confidence_low;
    double confidence_high;
} zi_run_stats;

typedef struct {
    uint64_t n;       /* dictionary size */
    int32_t dims;     /* effective D = min(cfg.dims, m*C, n)  (proj/src/builder.cpp:137) */
    int32_t m;        /* pixels per layout = subset_pixel_count(K, c) */
    int32_t channels;
    int32_t patch_size;
    int32_t width, height;
    double build_seconds;      /* device time of the last build (events) */
    double eigen_seconds;      /* host wall time spent in the eigen-solve step (launch or host solve) */
    int32_t pca_on_device;     /* 1: covariance + eigen-solve ran in k_pca (mc <= 224), 0: host solve */
    double coverage;           /* layout coverage c */
    int32_t loaded;            /* 1: read from a ZIDX1 file */
} zi_multi_index_info;

typedef struct zi_ctx zi_ctx;                 /* one device + one stream + scratch */
typedef struct zi_patch_index zi_patch_index; /* patch_index (proj/include/zinpaint/builder.hpp:60-75) */
typedef struct zi_index zi_index;             /* zcurve_index (proj/include/zinpaint/zcurve.hpp:117-145) */
typedef struct zi_multi_index zi_multi_index; /* multi_index (proj/include/zinpaint/builder.hpp:84-92) */

const char* zi_last_error(void);
const char* zi_version(void);

/* ---- context ---- */
zi_status zi_ctx_create(int device, zi_ctx** out);
zi_status zi_ctx_destroy(zi_ctx* ctx);
zi_status zi_ctx_synchronize(zi_ctx* ctx);
/* device-side timing on the ctx stream (CUDA events), for bench.py */
zi_status zi_timer_start(zi_ctx* ctx);
zi_status zi_timer_stop(zi_ctx* ctx, double* ms);
/* write a 256 MiB scratch buffer on the ctx stream so the next step starts with a cold L2 */
zi_status zi_ctx_flush_l2(zi_ctx* ctx);
/* number of kernels this ctx has launched so far (gpu_launches evidence) */
uint64_t zi_ctx_kernel_launches(const zi_ctx* ctx);
/* per-kernel device time accumulated while profiling is on (name-indexed, see api.cu) */
zi_status zi_ctx_set_profiling(zi_ctx* ctx, int on);
/* Morton sort policy of this ctx's 8-layout builds with `dims` quantised dims: 0 = learn (the
 * first build picks MSD + window sort from the byte histograms and falls back to LSD when the top
 * bytes are too clustered; later builds remember), -1 = LSD digit passes, whose last pass writes
 * the indices (fused finalize), k > 0 = k MSD bytes + window sort.  Results are identical. */
zi_status zi_ctx_set_sort_policy(zi_ctx* ctx, int32_t dims, int32_t policy);
/* time only these kernels (comma-separated launch names; NULL or "": every kernel) */
zi_status zi_ctx_set_profile_filter(zi_ctx* ctx, const char* names);
zi_status zi_ctx_profile(const zi_ctx* ctx, int slot, double* ms, uint64_t* launches,
                         const char** name);

/* ---- host utilities with reference counterparts ---- */
int zi_less_most_significant_bit(int a, int b);                          /* morton.hpp:10-12 */
int zi_morton_less(const uint8_t* a, const uint8_t* b, uint32_t dims);   /* morton.hpp:18-29 */
int zi_subset_pixel_count(int patch_size, double coverage);             /* layouts.cpp:9-11 */
/* build_subset_layouts (layouts.cpp:13-60); rc_out holds 8*m*2 int32 (row, col) */
zi_status zi_subset_layouts(int patch_size, double coverage, int32_t* rc_out, int32_t* m_out);
/* subset_layout::anchor of layouts 0..7 (layouts.cpp: N, E, S, W edge midpoints, then NW, NE, SW,
 * SE corners); rc_out holds 8*2 int32 (row, col) */
zi_status zi_subset_layout_anchors(int patch_size, int32_t* rc_out);
zi_status zi_index_config_validate(const zi_index_config* cfg, int channels); /* builder.cpp:38-53 */
void zi_index_config_default(zi_index_config* cfg);

/* ---- z-curve index ---- */
/* zcurve_index::from_descriptors (zcurve.hpp:121-123, zcurve.cpp:108-138): coords n*dims
 * row-major, keys packed y<<16|x; sorted on the device by an LSD radix sort of the Morton key */
zi_status zi_index_from_descriptors(zi_ctx* ctx, const uint8_t* coords, const uint32_t* keys,
                                    uint64_t n, uint32_t dims, uint32_t layout_id, zi_index** out);
zi_status zi_index_destroy(zi_index* idx);
zi_status zi_index_size(const zi_index* idx, uint64_t* n, uint32_t* dims);
/* zcurve_index::coords()/keys() (zcurve.hpp:130-133): sorted coords n*dims + keys n */
zi_status zi_index_export(zi_index* idx, uint8_t* coords_out, uint32_t* keys_out);
/* knn_search (zcurve.hpp:158-162, zcurve.cpp:429-452): exact k-NN in (distance, key) order;
 * packed_out receives min(k, n) packed (dist<<32 | key) ascending. mu is validated only. */
zi_status zi_knn_search(zi_index* idx, const uint8_t* query, uint32_t k, uint32_t mu, int32_t norm,
                        uint64_t* packed_out, uint32_t* count_out);
/* batched form for the cfg-5 sweep: queries nq*dims, packed_out nq*k, counts_out nq */
zi_status zi_knn_search_batch(zi_index* idx, const uint8_t* queries, uint64_t nq, uint32_t k,
                              int32_t norm, uint64_t* packed_out, uint32_t* counts_out);

/* timed device-resident batch (bench helper): queries uploaded once, `reps` launches timed with
 * CUDA events; ms_per_batch = mean device time of one launch over nq queries; stats3 (optional)
 * = {bbox tests, entries scored, results} of one launch.  Results of the last launch are copied
 * to packed_out / counts_out when non-NULL. */
zi_status zi_knn_batch_bench(zi_index* idx, const uint8_t* queries, uint64_t nq, uint32_t k, int32_t norm,
                             int32_t reps, double* ms_per_batch, uint64_t* stats3, uint64_t* packed_out,
                             uint32_t* counts_out);

/* ---- dictionary: collect_dictionary (builder.hpp:52-55, builder.cpp:74-108) ---- */
zi_status zi_dictionary_collect(zi_ctx* ctx, const uint8_t* known, int32_t width, int32_t height,
                                int32_t patch_size, uint32_t* keys_out, uint64_t cap, uint64_t* n_out);

/* ---- multi_index::build (builder.hpp:90-91, builder.cpp:202-224) ----
 * image: height*width*channels u8 (row-major, channel-interleaved); known: height*width
 * (nonzero = KNOWN).  All 8 layout indices are built on the device. */
zi_status zi_multi_index_build(zi_ctx* ctx, const uint8_t* image, const uint8_t* known,
                               int32_t width, int32_t height, int32_t channels,
                               const zi_index_config* cfg, zi_multi_index** out);
/* multi_index::build with the dictionary returned in the same call: keys_out (keys_cap entries,
 * pinned host memory for the copy to overlap) receives the n dictionary keys while the indices
 * are built -- the image upload and the dictionary download run on the copy engines alongside
 * the build's kernels.  Synchronous: keys_out is filled and the indices are ready on return. */
zi_status zi_multi_index_build_to(zi_ctx* ctx, const uint8_t* image, const uint8_t* known,
                                  int32_t width, int32_t height, int32_t channels,
                                  const zi_index_config* cfg, uint32_t* keys_out, uint64_t keys_cap,
                                  uint64_t* n_out, zi_multi_index** out);
/* rebuild from the device-resident image/mask (bench: inputs already in HBM) */
zi_status zi_multi_index_rebuild(zi_multi_index* mi);
zi_status zi_multi_index_destroy(zi_multi_index* mi);
zi_status zi_multi_index_get_info(const zi_multi_index* mi, zi_multi_index_info* info);
zi_status zi_multi_index_dictionary(zi_multi_index* mi, uint32_t* keys_out);
/* patch_index fields (builder.hpp:60-75): layout rc m*2, pca mean (m*C), components
 * (dims rows of m*C), eigenvalues (dims), quantizer lo/hi (dims).  NULL pointers are skipped. */
zi_status zi_multi_index_layout(zi_multi_index* mi, int32_t layout, int32_t* rc, double* mean,
                                double* components, double* eigenvalues, double* lo, double* hi);
zi_status zi_multi_index_layout_index(zi_multi_index* mi, int32_t layout, uint8_t* coords_out,
                                      uint32_t* keys_out);
/* borrowed view of one layout's zcurve_index (valid until mi is destroyed or rebuilt) */
zi_status zi_multi_index_get_index(zi_multi_index* mi, int32_t layout, zi_index** out);
/* ---- one layout: build_index (builder.hpp:77-81, builder.cpp:129-195) ----
 * The reference's per-layout entry point over a caller-given dictionary (keys packed y<<16|x,
 * every window inside the image) and subset layout (layout_rc: m (row, col) pairs).  The PCA fit
 * (moments of the dictionary restricted to the layout, pca.cpp:20-67), projection, quantiser and
 * Morton sort run on the device.  Errors: ZI_E_INVALID (config / layout / window outside the
 * image), ZI_E_EMPTY_DICT (n == 0). */
zi_status zi_index_build(zi_ctx* ctx, const uint8_t* image, int32_t width, int32_t height, int32_t channels,
                         const uint32_t* keys, uint64_t n, const int32_t* layout_rc, int32_t m,
                         const zi_index_config* cfg, zi_patch_index** out);
zi_status zi_patch_index_destroy(zi_patch_index* pi);
/* patch_index fields: dims (effective D), mc (= m*channels); mean (mc), components (dims rows of
 * mc), eigenvalues (dims), quantizer lo / hi (dims); build_seconds (device time of the whole
 * build) and sort_seconds (the sort + finalize).  NULL pointers are skipped. */
zi_status zi_patch_index_model(const zi_patch_index* pi, int32_t* dims, int32_t* mc, double* mean, double* components,
                               double* eigenvalues, double* lo, double* hi, double* build_seconds,
                               double* sort_seconds);
/* borrowed view of the layout's zcurve_index (valid until pi is destroyed) */
zi_status zi_patch_index_get_index(zi_patch_index* pi, zi_index** out);
/* patch_index::make_query (builder.hpp:72, builder.cpp:110-127): target K*K*C values + K*K known
 * flags -> dims quantised bytes; unknown layout pixels take the PCA mean.  On the device, in the
 * canonical fp64 order of the build. */
zi_status zi_make_query(zi_patch_index* pi, const uint8_t* target_values, const uint8_t* target_known, uint8_t* out);
/* the same for layout `layout` of a multi-index (multi_index::indices[layout].make_query) */
zi_status zi_multi_index_make_query(zi_multi_index* mi, int32_t layout, const uint8_t* target_values,
                                    const uint8_t* target_known, uint8_t* out);
/* brute_force_best(image, target, dictionary, norm) (engine.hpp:98-99, engine.cpp:220-236) over a
 * caller-given image and dictionary (uploaded per call; the multi-index form below reuses the
 * device-resident ones).  An empty dictionary returns cost 0xffffffff. */
zi_status zi_brute_force_scan(zi_ctx* ctx, const uint8_t* image, int32_t width, int32_t height, int32_t channels,
                              const uint32_t* keys, uint64_t n, const uint8_t* target_values,
                              const uint8_t* target_known, int32_t patch_size, int32_t norm, zi_best_patch* out);

/* ---- cfg5: index over fp32 feature vectors (BASELINE.json configs[4]) ----
 * The reference's patch-index semantics with every coordinate a pixel: PCA fit (pca.cpp:20-67,
 * canonical fp64 order in 32768-row stripes), project + quantise (builder.cpp:55-72,159-187),
 * from_descriptors keyed by row (bindings.cpp:109-125).  X: n x dim fp32, host memory; effective
 * dims = min(dims, dim, n).  Queries: unknown coordinate (known[j] == 0) -> mean (make_query,
 * builder.cpp:110-127), then the exact k-NN of zi_knn_search_batch. */
typedef struct zi_vector_index zi_vector_index;
zi_status zi_vector_index_build(zi_ctx* ctx, const float* X, uint64_t n, int32_t dim, int32_t dims,
                                zi_vector_index** out);
/* same, rows already in device memory (read during the build only; not retained) */
zi_status zi_vector_index_build_device(zi_ctx* ctx, const float* d_X, uint64_t n, int32_t dim, int32_t dims,
                                       zi_vector_index** out);
zi_status zi_vector_index_destroy(zi_vector_index* vi);
/* dims after the clamp; mean (dim), components (dims rows of dim), eigenvalues, lo, hi (dims);
 * NULL pointers are skipped; build_ms = device time of the build */
zi_status zi_vector_index_model(zi_vector_index* vi, int32_t* dims, double* mean, double* components,
                                double* eigenvalues, double* lo, double* hi, double* build_ms);
/* borrowed view of the z-curve index (keys = row ids); valid until vi is destroyed */
zi_status zi_vector_index_get_index(zi_vector_index* vi, zi_index** out);
/* queries (nq x dim fp32 + nq x dim known flags) -> quantised descriptors (nq x dims) */
zi_status zi_vector_make_queries(zi_vector_index* vi, const float* queries, const uint8_t* known, uint64_t nq,
                                 uint8_t* descriptors_out);
/* make_queries + exact k-NN: packed (dist<<32 | row) ascending, nq x k, counts[nq] */
zi_status zi_vector_knn_batch(zi_vector_index* vi, const float* queries, const uint8_t* known, uint64_t nq,
                              uint32_t k, int32_t norm, uint64_t* packed_out, uint32_t* counts_out);

/* ZIDX1 persistence (io_index.hpp:21-22, io_index.cpp:133-154): eight blocks, layout 0 first,
 * "ZIDX1" | u32 K | f64 coverage | u32 D | u32 layout | u64 n | u32 C | mean | components (D
 * rows) | eigenvalues | lo | hi | n x (D bytes, u32 x, u32 y).  Load re-sorts each block on the
 * device and recovers the dictionary from layout 0; `image` is the picture queries are refined
 * against (its channel count must match the file).  Errors: ZI_E_RUNTIME for bad magic / header,
 * truncation, key out of range or disagreeing blocks (the reference's std::runtime_error). */
zi_status zi_multi_index_save(zi_multi_index* mi, const char* path);
zi_status zi_multi_index_load(zi_ctx* ctx, const char* path, const uint8_t* image, int32_t w, int32_t h,
                              int32_t C, zi_multi_index** out);
/* exact int64 moments of the full K*K*C patch vector (s[F], S[F*F]) behind the PCA fit */
zi_status zi_multi_index_moments(zi_multi_index* mi, int64_t* s_out, int64_t* S_out);

/* ---- query ---- */
/* query_best_patch (engine.hpp:93-96, engine.cpp:178-213): select_index + make_query + exact
 * knn + masked-cost refine; target_values K*K*C, target_known K*K.  knn_out (optional)
 * receives the sorted candidate list (best->candidates entries). */
zi_status zi_query_best_patch(zi_multi_index* mi, const uint8_t* target_values,
                              const uint8_t* target_known, uint32_t k, int32_t norm,
                              zi_best_patch* out, uint64_t* knn_out);
/* brute_force_best (engine.hpp:98-99, engine.cpp:220-236) over the whole dictionary */
zi_status zi_brute_force_best(zi_multi_index* mi, const uint8_t* target_values,
                              const uint8_t* target_known, int32_t norm, zi_best_patch* out);

/* masked-cost refine of a caller-given candidate list: the refine step of query_best_patch
 * (engine.cpp:195-212) on its own, for the sharded query (the per-shard k-NN lists are merged
 * by the host, then the global top-k is refined here).  cands: packed (dist<<32 | key) */
zi_status zi_refine_best(zi_multi_index* mi, const uint8_t* target_values, const uint8_t* target_known,
                         const uint64_t* cands, uint32_t count, int32_t norm, zi_best_patch* out);

/* ---- range-partitioned multi_index over G ranks ----
 * No reference counterpart (the reference is one host process); the result is rank r holding
 * positions shard_ranges(n, G)[r] of every layout of multi_index::build (builder.cpp:202-224),
 * byte-identical.  The caller runs the collectives between the stages (sharding.py: NCCL over
 * torch.distributed); d_* are DEVICE pointers (the send buffers are owned by the shard, valid
 * until the next stage; the receive buffers are the caller's).  Stages, in order:
 *   create -> moments (all-reduce SUM of F+F*F int64) -> fit_project (all-reduce MIN lo, MAX hi:
 *   8*dims order-preserving int64 each) -> refine_ranges (all-reduce MIN / MAX again) ->
 *   quantize_sort (all-gather 8*S sample rows of words+1
 *   u32) -> zi_shard_splitters -> partition (all-gather counts [G][8]; all-to-all records,
 *   words+1 u32 each) -> receive (all-gather counts2; all-to-all) -> finish.
 * After finish, zi_shard_multi_index() is a multi_index whose 8 indices and dictionary are this
 * rank's slice: zi_query_best_patch with knn_out gives the local k-NN list, zi_brute_force_best
 * scans the slice, zi_refine_best refines a merged list. */
typedef struct zi_shard zi_shard;
zi_status zi_shard_create(zi_ctx* ctx, const uint8_t* image, const uint8_t* known, int32_t w, int32_t h,
                          int32_t C, const zi_index_config* cfg, int32_t rank, int32_t world, zi_shard** out);
zi_status zi_shard_destroy(zi_shard* sh);
/* restart the stages for the next build over the same device-resident image and mask, every
 * device buffer kept (bench: one sharded build per step) */
zi_status zi_shard_rebuild(zi_shard* sh);
/* world == 1, after quantize_sort: the locally sorted layouts are the index -- finalise them
 * without the exchange stages (partition / receive / finish) */
zi_status zi_shard_finish_local(zi_shard* sh);
/* info[10]: n_total, row_begin, row_end, F, dims, words, rank, world, stage, records held */
zi_status zi_shard_info(const zi_shard* sh, uint64_t* info);
zi_status zi_shard_moments(zi_shard* sh, int64_t* moments_out);
zi_status zi_shard_fit_project(zi_shard* sh, const int64_t* moments, int64_t* lo_out, int64_t* hi_out);
/* the global ranges of fit_project (approximate on the tensor-core path) -> this rank's exact
 * partial lo / hi (all-reduce MIN / MAX again before quantize_sort) */
zi_status zi_shard_refine_ranges(zi_shard* sh, const int64_t* lo, const int64_t* hi, int64_t* lo_out,
                                 int64_t* hi_out);
zi_status zi_shard_quantize_sort(zi_shard* sh, const int64_t* lo, const int64_t* hi, uint32_t samples_per_layout,
                                 uint32_t* samples_out);
/* host only: G-1 splitters per layout from all ranks' samples (count rows) */
zi_status zi_shard_splitters(const uint32_t* samples, uint64_t count, int32_t words, int32_t world,
                             uint32_t* splitters_out);
zi_status zi_shard_partition(zi_shard* sh, const uint32_t* splitters, uint64_t* counts_out,
                             const uint32_t** d_send);
/* host only: what rank `me` sends where after the first exchange (all_counts [src][dst][8]) */
zi_status zi_shard_rebalance_plan(const uint64_t* all_counts, int32_t world, uint64_t n_total, int32_t me,
                                  uint64_t* send_counts, uint64_t* send_starts);
zi_status zi_shard_receive(zi_shard* sh, const uint32_t* d_recv, const uint64_t* all_counts,
                           uint64_t* counts2_out, const uint32_t** d_send2);
zi_status zi_shard_finish(zi_shard* sh, const uint32_t* d_recv2, const uint64_t* all_counts2);
/* borrowed multi_index view of the shard (valid until zi_shard_destroy) */
zi_status zi_shard_multi_index(zi_shard* sh, zi_multi_index** out);

/* ---- inpaint (engine.hpp:112-118, engine.cpp:442-506) ----
 * records: capacity `cap` (the iteration count never exceeds the unknown pixel count). */
zi_status zi_inpaint(zi_ctx* ctx, const uint8_t* image, const uint8_t* known, int32_t width,
                     int32_t height, int32_t channels, const zi_index_config* cfg,
                     const zi_inpaint_config* icfg, uint8_t* image_out,
                     zi_iteration_record* records, uint64_t cap, uint64_t* n_records,
                     zi_run_stats* stats);
/* variant with prebuilt indices (engine.hpp:115-118): query-side knobs from cfg */
zi_status zi_inpaint_with_index(zi_multi_index* mi, const uint8_t* image, const uint8_t* known,
                                const zi_index_config* cfg, const zi_inpaint_config* icfg,
                                uint8_t* image_out, zi_iteration_record* records, uint64_t cap,
                                uint64_t* n_records, zi_run_stats* stats);

#ifdef __cplusplus
}
#endif
#endif /* ZINPAINT_B200_H */
