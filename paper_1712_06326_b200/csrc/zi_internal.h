// zi_internal.h -- internal types shared by the host runtime (C++) and the sm_100a kernels.
// Nothing here crosses the C ABI (include/zinpaint_b200.h).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <functional>
#include <vector>

#include "zinpaint_b200.h"

namespace zi {

// Internal exception; converted to a zi_status at the ABI boundary (api.cu).
struct error : std::runtime_error {
    zi_status code;
    error(zi_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define ZI_CUDA(x)                                                                              \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess)                                                                  \
            throw ::zi::error(e_ == cudaErrorMemoryAllocation ? ZI_E_OOM : ZI_E_CUDA,           \
                              std::string(#x) + ": " + cudaGetErrorString(e_));                 \
    } while (0)

inline void check_launch(const char* name) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw error(ZI_E_CUDA, std::string("launch ") + name + ": " + cudaGetErrorString(e));
}

// Stream of the API call in progress on this thread (set by api.cu's guard): device buffers are
// allocated and freed stream-ordered on it, from the device's default memory pool, which keeps
// its memory (release threshold = max) -- building index after index reuses the same HBM without
// cudaMalloc / cudaFree round trips.
extern thread_local cudaStream_t tls_alloc_stream;
// the ctx's private memory pool (nullptr: the device's current pool)
extern thread_local cudaMemPool_t tls_alloc_pool;

// Growable device buffer (pool allocated, never shrinks).
template <typename T>
struct dbuf {
    T* p = nullptr;
    size_t cap = 0;
    cudaStream_t s = nullptr;  // stream the buffer was allocated on (frees are ordered after its work)
    dbuf() = default;
    dbuf(const dbuf&) = delete;
    dbuf& operator=(const dbuf&) = delete;
    ~dbuf() { release(); }
    void release() {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        cap = 0;
    }
    T* ensure(size_t n) {
        if (n <= cap && p) return p;
        release();
        const size_t bytes = (n ? n : 1) * sizeof(T);
        s = tls_alloc_stream;
        if (tls_alloc_pool) ZI_CUDA(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&p), bytes, tls_alloc_pool, s));
        else ZI_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), bytes, s));
        cap = n ? n : 1;
        return p;
    }
};

// Pinned host staging buffer.
template <typename T>
struct hbuf {
    T* p = nullptr;
    size_t cap = 0;
    hbuf() = default;
    hbuf(const hbuf&) = delete;
    hbuf& operator=(const hbuf&) = delete;
    ~hbuf() {
        if (p) cudaFreeHost(p);
    }
    T* ensure(size_t n) {
        if (n <= cap && p) return p;
        if (p) cudaFreeHost(p);
        p = nullptr;
        ZI_CUDA(cudaMallocHost(reinterpret_cast<void**>(&p), (n ? n : 1) * sizeof(T)));
        cap = n ? n : 1;
        return p;
    }
};

// Raise a kernel's dynamic shared-memory limit to at least `bytes` on `device` (the attribute is
// per function and per device); thread-safe, remembers what each (function, device) already has.
void set_smem_attr(const void* fn, int device, size_t bytes);
template <typename F>
inline void smem_attr(int device, F* fn, size_t bytes) {
    set_smem_attr(reinterpret_cast<const void*>(fn), device, bytes);
}

// Per-kernel device timing (CUDA events on the ctx stream), used by bench.py for the
// roofline's "average launch duration measured live".
struct prof_slot {
    const char* name = nullptr;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> events;
    size_t used = 0;
    uint64_t launches = 0;
};

}  // namespace zi

struct zi_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    uint64_t launches = 0;
    bool profiling = false;
    std::vector<zi::prof_slot> prof;
    std::vector<std::string> prof_filter;  // kernels to time while profiling (empty: every kernel)
    int num_sms = 148;
    cudaMemPool_t pool = nullptr;  // private stream-ordered pool (never trimmed; rebuilds reuse its HBM)
    // shared scratch for sorts / collection
    zi::dbuf<uint8_t> scratch;
    zi::dbuf<uint32_t> counter;  // small integer scratch (tile counters etc.)
    zi::dbuf<uint8_t> flush;     // L2 flush buffer (bench hygiene)
    // hybrid sort depth learnt per (dims, layouts): 0 = from the byte entropies, -1 = all-LSD;
    // raised when a build's MSD split left too many records in oversized segments
    int sort_depth[33][2] = {};
    int flush_toggle = 1;
    zi::dbuf<int2> gm_wtab;      // fused moments: gather word table
    zi::dbuf<uint32_t> ss_buf;   // splitter sort: output records, samples, splitters, histograms
    // copy stream of zi_multi_index_build_to: the image upload and the dictionary download run
    // on the copy engines while the build's kernels run (created on first use)
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_alloc = nullptr, ev_img = nullptr, ev_dict = nullptr, ev_copy = nullptr;
};

// One z-curve-sorted index, device resident.
//   planes : P = ceil(dims/4) uint32 planes of n words; plane p holds dims 4p..4p+3 (dim 4p in
//            the low byte) of every entry, in Morton order -> coalesced 4-dim loads.
//   keys   : packed patch keys (y<<16|x), Morton order.
//   bbox   : per 256-entry block, per-dim min and max bytes, packed the same way as planes.
struct zi_index {
    zi_ctx* ctx = nullptr;
    uint64_t n = 0;
    uint32_t dims = 0, planes_n = 0, layout_id = 0;
    uint64_t nblk = 0;
    zi::dbuf<uint32_t> planes, keys, bbox_min, bbox_max;
    // query scratch
    zi::dbuf<uint8_t> qscratch;
    zi::hbuf<uint8_t> hstage;
};

struct zi_layout_state {
    std::vector<int32_t> rc;  // m*2
    std::vector<double> mean, comp, eig, lo, hi;
    zi_index index;
};

struct zi_multi_index {
    zi_ctx* ctx = nullptr;
    zi_index_config cfg{};
    int32_t w = 0, h = 0, C = 1, K = 9, m = 0, mc = 0, F = 0, dims = 0;
    uint64_t n = 0;
    double build_ms = 0.0, eigen_s = 0.0, wall_s = 0.0;
    zi::dbuf<uint8_t> image, known;
    zi::dbuf<uint32_t> dict;
    zi::dbuf<int32_t> layout_off;        // 8*m pixel offsets (r*w + c)*C
    zi::dbuf<int32_t> layout_local;      // 8*m local indices r*K + c
    zi::dbuf<double> pca_mean, pca_comp; // 8*mc, 8*mc*D ([layout][j][d])
    zi::dbuf<unsigned long long> minmax; // 8 * 2*D ordered-u64 lo / hi
    zi::dbuf<unsigned long long> moments;  // F + F*F (s, S)
    zi::dbuf<double> proj;               // D*n fp64 projections (reused across layouts)
    zi::dbuf<uint32_t> recs;             // (W+1)*n sort records (Morton words + payload)
    zi::dbuf<uint8_t> pt_scratch;        // tensor-core projection: digit matrices, bounds, fix-up list
    zi::dbuf<int2> pt_wtab;              // tensor-core projection: gather word table
    zi::dbuf<uint8_t> qscratch;          // query scratch
    zi::hbuf<uint8_t> hstage;            // pinned staging for targets/results
    void* hres = nullptr;                // mapped pinned query result (k_query_one publishes it)
    void* dres = nullptr;
    uint32_t qseq = 0;
    const void* qws_last = nullptr;      // query workspace of the last launch
    bool qws_clean = false;              // the last k_query_one left it reset
    zi::hbuf<unsigned long long> hmom;
    std::vector<int64_t> s, S;           // host copy of the moments
    // device PCA (k_pca.cu): feature columns [8][mc], eigenvalues [8][D], eigenvector scratch
    zi::dbuf<int32_t> pca_cols;
    zi::dbuf<double> pca_eig, pca_work;
    zi::dbuf<int> pca_status;
    bool pca_cols_ready = false;
    bool host_model = false;             // s, S, L[].mean/comp/eig mirror the device copies
    bool host_lohi = false;              // L[].lo/hi mirror the device min/max
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;  // build timing, read lazily (no sync at build end)
    bool build_ms_pending = false;
    bool loaded = false;                 // read from a ZIDX1 file (no mask, no moments)
    bool device_pca = false;             // last build solved the eigenproblems on the device
    // range-partitioned shard (shard.cu): this handle's indices hold one contiguous Morton range
    // of every layout and its dictionary slice is rows [row_begin, row_begin + n) of the n_total
    // dictionary rows in dict (every rank keeps the whole dictionary: payload rows are global)
    bool shard = false;
    uint64_t row_begin = 0, n_total = 0;
    // zi_multi_index_build_to: the image arrives on ctx->copy_stream (ev_img), and the dictionary
    // goes to dict_out on it as soon as it is collected (ev_copy)
    bool image_on_copy = false;
    uint32_t* dict_out = nullptr;
    uint64_t dict_cap = 0;
    // build records carry the patch key as payload (instead of (layout << 29) | row): set when the
    // sort's fused last pass writes the indices (no dictionary gather there)
    bool payload_key = false;
    zi_layout_state L[8];
};

// One layout index over a caller-given dictionary: build_index (proj/src/builder.cpp:129-195),
// the per-layout entry point of the reference (builder.hpp:77-81).  Same device pipeline as one
// layout of zi_multi_index: exact int64 moments, device eigen-solve, canonical fp64 projection,
// quantiser, Morton sort, finalize.
struct zi_patch_index {
    zi_ctx* ctx = nullptr;
    zi_index_config cfg{};
    int32_t w = 0, h = 0, C = 1, K = 9, m = 0, mc = 0, F = 0, dims = 0;
    uint64_t n = 0;
    std::vector<int32_t> rc;                 // m*2 (row, col)
    zi::dbuf<uint8_t> image;
    zi::dbuf<uint32_t> dict;
    zi::dbuf<int32_t> off, local, cols;      // pixel offsets, local r*K+c, feature columns
    zi::dbuf<unsigned long long> moments, minmax;
    zi::dbuf<double> mean, comp, eig, work, proj;
    zi::dbuf<int> status;
    zi::dbuf<uint32_t> recs;
    zi::dbuf<uint8_t> qbuf;                  // make_query staging
    zi::hbuf<uint8_t> hstage;
    std::vector<double> h_mean, h_comp, h_eig, h_lo, h_hi;  // comp: dims rows of mc
    bool device_pca = false;
    double build_ms = 0.0, sort_ms = 0.0;
    zi_index index;
};

// cfg5: z-curve index over fp32 feature vectors (k_vector.cu)
struct zi_vector_index {
    zi_ctx* ctx = nullptr;
    uint64_t n = 0;
    int dim = 0, dims = 0;
    zi::dbuf<float> X;                  // n x dim, device resident (owned copy)
    const float* Xd = nullptr;          // the rows the build reads (X.p or a caller's device buffer)
    zi::dbuf<double> mean, cov, comp, eig, pca_work, Y, scratch;
    zi::dbuf<unsigned long long> minmax;
    zi::dbuf<uint32_t> recs;
    zi::dbuf<uint8_t> qbuf;             // query staging
    zi_index index;
    bool host_model = false;
    std::vector<double> h_mean, h_comp, h_eig, h_lo, h_hi;
    double build_ms = 0.0;
};

namespace zi {

// ---- kernel entry points (implemented in the .cu files) ----
void launch_begin(zi_ctx* ctx, const char* name);  // counts launches; profiling events
void launch_end(zi_ctx* ctx, const char* name);

// collect_dictionary on the device: known (w*h) -> keys (row-major); returns n (syncs)
uint64_t collect_dictionary(zi_ctx* ctx, const uint8_t* d_known, int w, int h, int K,
                            dbuf<uint32_t>& keys_out);

// exact moments s (F) and S (F*F, full symmetric) of the K*K*C patch vectors
void gram_u8_tc(zi_ctx* ctx, const uint8_t* XT, int F, int Fpad, uint64_t npad, unsigned long long* out);
void patch_moments(zi_ctx* ctx, const uint8_t* d_img, int w, int C, int K, const uint32_t* d_keys,
                   uint64_t n, unsigned long long* d_out /* F + F*F */);
// the fused path of patch_moments (k_proj_tc.cu); false: outside its envelope
bool patch_moments_fused(zi_ctx* ctx, const uint8_t* d_img, int w, int C, int K, const uint32_t* d_keys, uint64_t n,
                         unsigned long long* d_out, dbuf<int2>& wtab);

// projection pass: Y[d*n + i] fp64 and ordered-u64 lo/hi in minmax (2*D)
void project(zi_ctx* ctx, const uint8_t* d_img, int w, int C, const uint32_t* d_keys, uint64_t n,
             const int32_t* d_off, int m, const double* d_mean, const double* d_comp, int D,
             double* d_Y, unsigned long long* d_minmax);

// quantise + Morton interleave -> key words (SoA, W words) + payload = dictionary key
// (records of all layouts in one array of N entries; this layout's entries start at layout*n;
// payload row = row_base + i, row_base > 0 for a shard's slice of the dictionary)
void quantize_interleave(zi_ctx* ctx, const double* d_Y, const unsigned long long* d_minmax, uint64_t n,
                         uint64_t N, uint32_t layout, int D, uint32_t* d_keyw, uint32_t* d_val,
                         uint32_t row_base = 0);
// row-major coords (n*D) -> Morton key words + payload copy
void interleave_coords(zi_ctx* ctx, const uint8_t* d_coords, const uint32_t* d_keys_in, uint64_t n,
                       int D, uint32_t* d_keyw, uint32_t* d_val);

// stable LSD radix sort of (key words, payload) by the D-byte Morton key; when
// payload_first, 4 leading passes order by the payload (ties of the Morton key -> key order).
// d_keyw: W*n words (SoA), d_val: n.  Result in place.
void morton_sort(zi_ctx* ctx, uint32_t* d_keyw, uint32_t* d_val, uint64_t n, int D, bool payload_first);
constexpr int kSortMaxWords = 9;  // up to 8 Morton key words (D <= 32) + payload
// Splitter sort (k_ssort.cu) of G groups of n records (group-major, SoA: nw-1 Morton words then
// the payload) by (Morton key, payload) inside each group; group_in_payload: the group id is the
// payload's top 3 bits (the 8-layout build).  out[k]: the buffers holding the sorted words (the
// input, or ctx->ss_buf), valid until the next sort on this context.
void sample_sort_groups(zi_ctx* ctx, uint32_t* const* words, int nw, uint64_t n, int G, int D, bool group_in_payload,
                        uint32_t** out);
// the build's sort: G groups (layouts) of n records, group-major; out[k] = word k of the sorted
// records (stride G*n), payload at out[W].  Onesweep LSD / hybrid sorts (k_sort.cu); ZI_SORT=splitter
// selects the experimental two-level splitter sort (k_ssort.cu) when the payload is ascending.
// sink (optional, G = 8 layout groups, D a multiple of 4 up to 16): when the sort ends in an LSD
// pass, that pass writes the layout indices' dim planes and keys instead of records; the return
// value tells whether it did (the caller then only adds the bboxes, finalize_index_bboxes)
struct final_sink {
    uint32_t* planes[8];   // per group (layout): [P][n] plane words
    uint32_t* keys[8];     // per group: [n] patch keys
    const uint32_t* dict;  // payload row -> patch key
};
bool morton_sort_records(zi_ctx* ctx, uint32_t* d_keyw, uint32_t* d_val, uint64_t n, int G, int D,
                         bool group_in_payload, uint32_t** out, bool payload_ascending = true,
                         const final_sink* sink = nullptr);
bool layouts_sort_fuses(zi_ctx* ctx, int D);  // the 8-layout sort will write the indices itself
// the index buffers finalize_index fills (the fused sort's last pass writes planes and keys)
void prepare_index(zi_index* idx, uint64_t n, int D);
// the per-256-entry bboxes of nidx (<= 8) equally sized indices whose planes are written
void finalize_index_bboxes(zi_ctx* ctx, zi_index* const* idx, int nidx);
// all 8 layouts at once: N = 8n records, Morton passes then one pass on the layout bits of the
// payload ((layout << 29) | row) -- stable, so each layout segment ends in reference order
// out (optional): the buffers holding the sorted words (out[k] = out[0] + k*N, the payload at
// out[W]) -- the sort's scratch buffer after an odd number of passes, valid until the next use
// of the context scratch; without it the records end in d_keyw / d_val
void morton_sort_layouts(zi_ctx* ctx, uint32_t* d_keyw, uint32_t* d_val, uint64_t N, int D, uint32_t** out = nullptr);

// projection + quantisation of all 8 layouts on the int8 tensor cores with the exact fp64 fix-up
// (k_proj_tc.cu): records and exact lo/hi identical to project + quantize_interleave; false when
// the configuration is outside its envelope (dims > 16, K*K*C > 384, ZI_PROJ_FP64 set)
bool project_quantize_tc(zi_multi_index* mi, uint32_t* d_keyw, uint32_t* d_val, uint64_t N);
// the same three phases for a shard, all-reduces in between: begin -> approximate ranges (ordered
// u64, 8 x 2 x dims; false: not eligible, use the fp64 path); quantize(global approximate
// ranges) -> exact lo / hi over the local candidates; fixup (with the global exact lo / hi in
// mi->minmax)
bool shard_tc_begin(zi_multi_index* mi, uint32_t* keyw, uint32_t* val, uint64_t Nrec, unsigned long long* amm_out);
void shard_tc_quantize(zi_multi_index* mi, uint32_t* keyw, uint32_t* val, uint64_t Nrec, const unsigned long long* amm,
                       unsigned long long* exact_out);
void shard_tc_fixup(zi_multi_index* mi, uint32_t* keyw, uint32_t* val, uint64_t Nrec);

// sorted key words + payload -> index planes, keys, bbox
void finalize_layout_indexes(zi_ctx* ctx, const uint32_t* d_keyw, const uint32_t* d_val, uint64_t N, uint64_t n, int D,
                             const uint32_t* d_dict, zi_index* const* idx, int nidx);
void finalize_index(zi_ctx* ctx, const uint32_t* d_keyw, const uint32_t* d_val, uint64_t N, uint64_t off,
                    uint64_t n, int D, const uint32_t* d_dict, zi_index* idx);

// decode the ordered-u64 min/max pair of layout `l` into host lo/hi
double ordered_to_double(unsigned long long u);

// ---- query side ----
struct query_result {
    uint64_t best;   // packed (cost<<32 | key)
    uint32_t lid;
    uint32_t count;  // number of knn candidates
};
// full query_best_patch on the device for the target staged at d_target (K*K*C values then K*K
// flags); knn list optionally copied out.
// while_waiting (optional): host work run once while the device answers (the fill loop's
// result-independent part of the paste)
query_result query_best_patch(zi_multi_index* mi, const uint8_t* h_tv, const uint8_t* h_tk,
                              uint32_t k, int norm, uint64_t* knn_out, const std::function<void()>* while_waiting = nullptr);
uint64_t brute_force_best(zi_multi_index* mi, const uint8_t* h_tv, const uint8_t* h_tk, int norm);
// the exhaustive scan over any device image + dictionary (brute_force_best with the reference's
// (image, target, dictionary, norm) arguments, engine.hpp:98-99)
uint64_t brute_force_scan(zi_ctx* ctx, const uint8_t* d_img, int w, int C, int K, const uint32_t* d_dict, uint64_t n,
                          const uint8_t* h_tv, const uint8_t* h_tk, int norm, dbuf<uint8_t>& scratch,
                          hbuf<uint8_t>& stage);
// patch_index::make_query (proj/src/builder.cpp:110-127) on the device for one layout model:
// d_local m local pixel indices, d_mean mc, d_comp [j][d], d_minmax 2*D ordered lo / hi
void make_query(zi_ctx* ctx, const uint8_t* h_tv, const uint8_t* h_tk, int K, int C, const int32_t* d_local, int m,
                const double* d_mean, const double* d_comp, const unsigned long long* d_minmax, int D, uint8_t* h_out,
                dbuf<uint8_t>& scratch, hbuf<uint8_t>& stage);
// masked-cost refine of a given candidate list (packed dist<<32 | key) -> packed (cost<<32 | key)
uint64_t refine_candidates(zi_multi_index* mi, const uint8_t* h_tv, const uint8_t* h_tk, const uint64_t* h_cands,
                           uint32_t count, int norm);
// knn over a bare index (zcurve_index + query bytes)
uint32_t knn_search(zi_index* idx, const uint8_t* h_query, uint32_t k, int norm, uint64_t* out);
void knn_search_batch(zi_index* idx, const uint8_t* h_queries, uint64_t nq, uint32_t k, int norm,
                      uint64_t* out, uint32_t* counts);
// device-resident batch (k <= 256): warp per query; stats (optional) = {blocks bbox-tested,
// entries scored, results}
void knn_batch_device(zi_ctx* ctx, zi_index* idx, const uint8_t* d_queries, uint64_t nq, uint32_t k, int norm,
                      unsigned long long* d_out, uint32_t* d_counts, unsigned long long* d_stats);

// ---- range-partitioned shard (shard.cu) ----
void shard_ranges(uint64_t n, int world, int r, uint64_t* b, uint64_t* e);
zi_shard* shard_create(zi_multi_index* mi, int rank, int world);
void shard_rebuild(zi_shard* sh);
void shard_finish_local(zi_shard* sh);
void shard_moments(zi_shard* sh, int64_t* out);
void shard_fit_project(zi_shard* sh, const int64_t* moments, int64_t* lo_out, int64_t* hi_out);
void shard_refine_ranges(zi_shard* sh, const int64_t* lo, const int64_t* hi, int64_t* lo_out, int64_t* hi_out);
void shard_quantize_sort(zi_shard* sh, const int64_t* lo, const int64_t* hi, uint32_t S, uint32_t* samples_out);
void shard_splitters(const uint32_t* samples, uint64_t count, int W, int world, uint32_t* out);
void shard_partition(zi_shard* sh, const uint32_t* splitters, uint64_t* counts_out, const uint32_t** d_send);
void shard_rebalance_plan(const uint64_t* all_counts, int world, uint64_t n_total, int me, uint64_t* send_counts,
                          uint64_t* send_starts);
void shard_receive(zi_shard* sh, const uint32_t* d_recv, const uint64_t* all_counts, uint64_t* counts2_out,
                   const uint32_t** d_send2);
void shard_finish(zi_shard* sh, const uint32_t* d_recv2, const uint64_t* all_counts2);
zi_multi_index* shard_multi_index(zi_shard* sh);
void shard_destroy(zi_shard* sh);
void shard_info(const zi_shard* sh, uint64_t* v);

// ---- host pieces ----
int subset_pixel_count(int K, double c);
int subset_layouts(int K, double c, std::vector<int32_t>& rc);  // returns m
void layout_anchors(int K, int32_t* rc);                         // 8 (row, col) anchors
void validate_config(const zi_index_config& cfg, int channels);
// covariance + eigen-solve + sign rule for one layout (host, deterministic)
void pca_fit_layout(const std::vector<int64_t>& s, const std::vector<int64_t>& S, int F, uint64_t n,
                    const std::vector<int32_t>& cols, int dims, std::vector<double>& mean,
                    std::vector<double>& comp /* dims*mc, row d */, std::vector<double>& eig);
void build_multi_index(zi_multi_index* mi);
// the 8 PCA models from the moments already in mi->moments over n_total patches (device solve,
// host fallback for mc > 224); leaves mi->pca_mean / pca_comp on the device
void fit_models(zi_multi_index* mi, uint64_t n_total);
// copy the moments, the 8 PCA models and the quantiser ranges to the host mirror (lazy: only
// the accessors need them); finish_build_timing reads the build's event pair
void sync_host_model(zi_multi_index* mi);
void finish_build_timing(zi_multi_index* mi);
// k_pca.cu: covariance + eigen-solve of all 8 layouts on the device; false if mc is too large.
// d_work must hold pca_work_doubles(mc, D) doubles.
size_t pca_work_doubles(int mc, int D);
// one model from a precomputed covariance (mc x mc, row-major, device): comp [j][d], eig [D]
bool pca_from_cov_on_device(zi_ctx* ctx, const double* d_cov, int mc, int D, double* d_comp, double* d_eig,
                            double* d_work);
bool pca_on_device(zi_ctx* ctx, const unsigned long long* d_moments, int F, uint64_t n, const int32_t* d_cols, int mc,
                   int D, double* d_mean, double* d_comp, double* d_eig, double* d_work, int* d_status);
// the same for `layouts` models (d_cols holds layouts*mc columns)
bool pca_on_device_n(zi_ctx* ctx, int layouts, const unsigned long long* d_moments, int F, uint64_t n,
                     const int32_t* d_cols, int mc, int D, double* d_mean, double* d_comp, double* d_eig,
                     double* d_work);
// build_index for one layout (build.cu)
void build_patch_index(zi_patch_index* pi);
void patch_index_sync_host(zi_patch_index* pi);

// vector index (k_vector.cu): upload + build, device-resident build, queries, host mirrors
void vector_index_build(zi_vector_index* vi, const float* h_X);
void build_vector_index_device(zi_vector_index* vi);
void vector_make_queries(zi_vector_index* vi, const float* d_Q, const uint8_t* d_known, uint64_t nq, uint8_t* d_out);
void vector_sync_host_model(zi_vector_index* vi);
// hybrid Morton sort of a single index (payload = row id, ties by row) -- k_sort.cu
void morton_sort_rows(zi_ctx* ctx, uint32_t* d_keyw, uint32_t* d_val, uint64_t n, int D);

// ZIDX1 persistence (persist.cpp, proj/src/io_index.cpp)
struct zidx_header {
    int K = 0, D = 0, C = 0;
    double coverage = 0.0;
    uint64_t count = 0;
};
zidx_header zidx_peek(const char* path);
void save_multi_index(zi_multi_index* mi, const char* path);
// mi: created for the file's (K, coverage, dims) with layouts and image uploaded
void load_multi_index_into(zi_multi_index* mi, const char* path);

// fill loop (host_engine.cpp): run_loop / inpaint (proj/src/engine.cpp:283-506)
void run_inpaint(zi_multi_index* mi, const uint8_t* image, const uint8_t* known, const zi_index_config& cfg,
                 const zi_inpaint_config& icfg, uint8_t* image_out, zi_iteration_record* records, uint64_t cap,
                 uint64_t* n_records, zi_run_stats* stats);

}  // namespace zi
