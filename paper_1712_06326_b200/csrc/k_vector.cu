// k_vector.cu -- cfg5: a z-curve index over fp32 feature vectors (BASELINE.json configs[4];
// SURVEY.md §8(d) cfg5 row).  The reference expresses this path as its patch-index machinery
// with every coordinate a "pixel": PCA fit (proj/src/pca.cpp:20-67), project + quantise
// (proj/src/builder.cpp:55-72, 159-187), from_descriptors with the row index as the key
// (proj/python/bindings.cpp:109-125), make_query with unknown coordinates -> mean
// (proj/src/builder.cpp:110-127), knn_search.
//
// Canonical fp64 order (pinned in oracle/zoracle.cpp zo_vec_*; Eigen's order is unpinned):
//   * rows are processed in stripes of kStripe = 32768; a stripe's column sum adds, in order, the
//     row-ordered sums of its 4096-row sub-chunks; mean_j = (stripe sums added in order) / n;
//   * Gram G = sum over stripes (in order) of the stripe's row-ordered fma chain of
//     xc_i * xc_j (xc = (double)x - mean); cov = G / (n - 1);  the per-stripe chains run on the
//     FP64 tensor cores (mma.m8n8k4.f64 == four sequential fma's in k order);
//   * projection y_d = fma(comp[j][d], xc_j, y_d), j ascending, on the FP64 tensor cores, with
//     the quantiser's min / max folded into the same kernel;
//   * eigen-solve: k_pca.cu on the covariance (tolerance-checked, like the image path).
#include <algorithm>
#include <vector>

#include "common.cuh"

namespace zi {

constexpr int kStripe = 32768;      // canonical stripe of the mean / Gram sums
constexpr int kGramRows = 32;       // rows staged in shared memory per round (8 k-steps)

__device__ inline void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// per-stripe column sums: row-ordered sums of kSub-row sub-chunks, added in sub-chunk order
// (the canonical order: oracle zo_vec_mean_cov).  Thread (sub-chunk u, column j); part[s * dim + j]
constexpr int kSub = 4096;
constexpr int kSubs = kStripe / kSub;  // 8
__global__ void __launch_bounds__(1024) k_vec_colsum(const float* __restrict__ X, uint64_t n, int dim,
                                                     double* __restrict__ part) {
    __shared__ double s_sub[kSubs][128];
    const uint64_t r0 = static_cast<uint64_t>(blockIdx.x) * kStripe;
    for (int j0 = 0; j0 < dim; j0 += 128) {
        const int u = threadIdx.x / 128, j = j0 + threadIdx.x % 128;
        if (j < dim) {
            const uint64_t a = r0 + static_cast<uint64_t>(u) * kSub;
            const uint64_t lim = r0 + kStripe < n ? r0 + kStripe : n;
            const uint64_t e = a + kSub < lim ? a + kSub : lim;
            double s = 0.0;
            uint64_t r = a;
            for (; r + 8 <= e; r += 8) {  // 8 loads in flight, then the row-ordered adds
                float v[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) v[q] = __ldg(X + (r + q) * dim + j);
#pragma unroll
                for (int q = 0; q < 8; ++q) s = __dadd_rn(s, static_cast<double>(v[q]));
            }
            for (; r < e; ++r) s = __dadd_rn(s, static_cast<double>(__ldg(X + r * dim + j)));
            s_sub[u][threadIdx.x % 128] = s;  // a sub-chunk past the end sums to +0.0
        }
        __syncthreads();
        if (threadIdx.x < 128 && j0 + static_cast<int>(threadIdx.x) < dim) {
            double t = 0.0;
            for (int q = 0; q < kSubs; ++q) t = __dadd_rn(t, s_sub[q][threadIdx.x]);
            part[static_cast<size_t>(blockIdx.x) * dim + j0 + threadIdx.x] = t;
        }
        __syncthreads();
    }
}

__global__ void k_vec_mean(const double* __restrict__ part, int nstripe, int dim, uint64_t n, double* __restrict__ mean) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= dim) return;
    double s = 0.0;
    for (int t = 0; t < nstripe; ++t) s = __dadd_rn(s, part[static_cast<size_t>(t) * dim + j]);
    mean[j] = __ddiv_rn(s, static_cast<double>(n));
}

__device__ inline void cp_async16_v(void* dst, const void* src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
}

// Per-stripe Gram tiles (ti <= tj, 8x8) on the FP64 tensor cores: k = data rows in order;
// part[(s * ntiles + tile) * 64 + r * 8 + c] = G_s[8 ti + r][8 tj + c].  Rounds of kGramRows rows:
// the raw fp32 rows of round b+1 stream in with cp.async (one contiguous 16-byte-aligned block)
// while round b's k-steps run; each round is converted once to xc = (double)x - mean in shared
// memory (fp64, 32-byte row skew: conflict-free fragments).
// Blocked variant: warp w owns a 4x4 block of 8x8 tiles (block (bi, bj), bi <= bj, of the upper
// triangle), so a k-step loads 4 A and 4 B fragments for 16 MMAs (the per-tile variant loads 2
// per MMA and is shared-memory bound).  Tiles below the diagonal of a diagonal block are computed
// but not stored.  One warp per block, up to 10 blocks per CTA (two CTAs per SM: the 512 stripes of n = 2^24 then run in under two waves with twice the warps per SM).
constexpr int kGramMaxWarps = 10;  // 10 = the 4x4-tile blocks of the upper triangle at dim <= 128
__global__ void __launch_bounds__(kGramMaxWarps * 32, 2) k_vec_gram_blk(const float* __restrict__ X, uint64_t n, int dim,
                                                                        int Pd, const double* __restrict__ mean,
                                                                        int nblocks, double* __restrict__ part) {
    extern __shared__ __align__(16) double s_x[];  // kGramRows x (Pd + 4) fp64, then 2 raw fp32 rounds
    const int ld = Pd + 4;
    float* s_raw = reinterpret_cast<float*>(s_x + kGramRows * ld);
    const int raw_words = ((kGramRows * dim + 3) / 4) * 4;
    const int T = Pd / 8, Tb = (T + 3) / 4, ntiles = T * (T + 1) / 2;
    const int nthr = blockDim.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r = lane >> 2, c = lane & 3;
    const uint64_t r0 = static_cast<uint64_t>(blockIdx.x) * kStripe;
    const uint64_t r1 = r0 + kStripe < n ? r0 + kStripe : n;
    const int blk = blockIdx.y * kGramMaxWarps + warp;
    const bool active = blk < nblocks;
    int bi = 0, bj = 0;
    {
        int rem = active ? blk : 0;
        while (bi < Tb && rem >= Tb - bi) {
            rem -= Tb - bi;
            ++bi;
        }
        bj = bi + rem;
    }
    int offA[4], offB[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        offA[u] = c * ld + (4 * bi + u) * 8 + r;
        offB[u] = c * ld + (4 * bj + u) * 8 + r;
    }
    double acc[4][4][2];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v][0] = acc[u][v][1] = 0.0;
    auto issue = [&](uint64_t b, int buf) {
        const uint64_t rows = b + kGramRows <= r1 ? kGramRows : r1 - b;
        const uint64_t words = rows * dim;
        const float* src = X + b * dim;
        float* dst = s_raw + buf * raw_words;
        const uint64_t full = words / 4;
        for (uint64_t e = tid; e < full; e += nthr) cp_async16_v(dst + 4 * e, src + 4 * e);
        for (uint64_t e = full * 4 + tid; e < words; e += nthr) dst[e] = __ldg(src + e);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    issue(r0, 0);
    int buf = 0;
    for (uint64_t b = r0; b < r1; b += kGramRows, buf ^= 1) {
        if (b + kGramRows < r1) {
            issue(b + kGramRows, buf ^ 1);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        const float* raw = s_raw + buf * raw_words;
        const int rows = static_cast<int>(b + kGramRows <= r1 ? kGramRows : r1 - b);
        for (int e = tid; e < kGramRows * Pd; e += nthr) {
            const int rr = e / Pd, j = e - rr * Pd;
            s_x[rr * ld + j] = (rr < rows && j < dim) ? __dsub_rn(static_cast<double>(raw[rr * dim + j]), mean[j]) : 0.0;
        }
        __syncthreads();
        if (active) {
#pragma unroll 2
            for (int ks = 0; ks < kGramRows / 4; ++ks) {
                const double* xr = s_x + (ks * 4) * ld;
                double af[4], bf[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    af[u] = xr[offA[u]];
                    bf[u] = xr[offB[u]];
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) dmma(acc[u][v][0], acc[u][v][1], af[u], bf[v]);
            }
        }
    }
    if (!active) return;
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int ti = 4 * bi + u, tj = 4 * bj + v;
            if (ti >= T || tj >= T || ti > tj) continue;
            const int t = ti * T - ti * (ti - 1) / 2 + (tj - ti);  // upper-triangle row-major index
            double* o = part + (static_cast<size_t>(blockIdx.x) * ntiles + t) * 64 + r * 8 + 2 * c;
            o[0] = acc[u][v][0];
            o[1] = acc[u][v][1];
        }
}

// cov[i][j] = cov[j][i] = (sum over stripes, in order) / (n - 1)
__global__ void k_vec_gram_reduce(const double* __restrict__ part, int nstripe, int ntiles, int T, int dim, uint64_t n,
                                  double* __restrict__ cov) {
    const int t = blockIdx.x, e = threadIdx.x;  // one block of 64 threads per tile
    int a = 0, rem = t;
    while (a < T && rem >= T - a) {
        rem -= T - a;
        ++a;
    }
    const int i = a * 8 + (e >> 3), j = (a + rem) * 8 + (e & 7);
    if (i >= dim || j >= dim || i > j) return;
    double s = 0.0;
    for (int st = 0; st < nstripe; ++st) s = __dadd_rn(s, part[(static_cast<size_t>(st) * ntiles + t) * 64 + e]);
    const double v = n > 1 ? __ddiv_rn(s, static_cast<double>(n - 1)) : s;
    cov[static_cast<size_t>(i) * dim + j] = v;
    cov[static_cast<size_t>(j) * dim + i] = v;
}

// projection of fp32 rows onto comp ([j][d]) on the FP64 tensor cores (see k_project), with the
// quantiser's min / max folded in
constexpr int kVpThreads = 256;
constexpr int kVpGroups = 4;
template <int D>
__global__ void __launch_bounds__(kVpThreads) k_vec_project(const float* __restrict__ X, uint64_t n, int dim,
                                                            const double* __restrict__ mean,
                                                            const double* __restrict__ comp, double* __restrict__ Y,
                                                            unsigned long long* __restrict__ minmax) {
    constexpr int NT = (D + 7) / 8;
    constexpr int G = kVpGroups;
    extern __shared__ double sm[];
    const int KS = (dim + 3) / 4;
    double* s_B = sm;                                          // [KS][NT][32]
    double* s_mean = s_B + static_cast<size_t>(KS) * NT * 32;  // [KS*4]
    for (int idx = threadIdx.x; idx < KS * NT * 32; idx += kVpThreads) {
        const int ks = idx / (NT * 32), t = (idx / 32) % NT, ln = idx % 32;
        const int j = ks * 4 + ln % 4, d = t * 8 + ln / 4;
        s_B[idx] = (j < dim && d < D) ? comp[j * D + d] : 0.0;
    }
    for (int j = threadIdx.x; j < KS * 4; j += kVpThreads) s_mean[j] = j < dim ? mean[j] : 0.0;
    __shared__ unsigned long long s_mm[2][D];
    if (threadIdx.x < 2 * D) s_mm[threadIdx.x / D][threadIdx.x % D] = threadIdx.x < D ? ~0ull : 0ull;
    __syncthreads();
    const int lane = threadIdx.x & 31, r = lane >> 2, c = lane & 3;
    const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (kVpThreads / 32);
    for (uint64_t base = (static_cast<uint64_t>(blockIdx.x) * (kVpThreads / 32) + (threadIdx.x >> 5)) * (8 * G);
         base < n; base += warps * 8 * G) {
        const float* xp[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const uint64_t i = base + 8 * g + r;
            xp[g] = X + (i < n ? i : n - 1) * dim;
        }
        double acc[G][NT][2];
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
            for (int t = 0; t < NT; ++t) acc[g][t][0] = acc[g][t][1] = 0.0;
        float xn[G];
#pragma unroll
        for (int g = 0; g < G; ++g) xn[g] = c < dim ? __ldg(xp[g] + c) : 0.f;
        for (int ks = 0; ks < KS; ++ks) {
            float xcur[G];
#pragma unroll
            for (int g = 0; g < G; ++g) xcur[g] = xn[g];
            const int jn = (ks + 1) * 4 + c;
            if (ks + 1 < KS)
#pragma unroll
                for (int g = 0; g < G; ++g) xn[g] = jn < dim ? __ldg(xp[g] + jn) : 0.f;
            const double mj = s_mean[ks * 4 + c];
            double bf[NT];
#pragma unroll
            for (int t = 0; t < NT; ++t) bf[t] = s_B[(ks * NT + t) * 32 + lane];
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const double a = __dsub_rn(static_cast<double>(xcur[g]), mj);
#pragma unroll
                for (int t = 0; t < NT; ++t) dmma(acc[g][t][0], acc[g][t][1], a, bf[t]);
            }
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const uint64_t i = base + 8 * g + r;
            if (i < n) {
#pragma unroll
                for (int t = 0; t < NT; ++t)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int d = 8 * t + 2 * c + e;
                        if (d < D) {
                            const double y = acc[g][t][e];
                            Y[static_cast<size_t>(d) * n + i] = y;
                            const unsigned long long o = double_to_ordered(y);
                            atomicMin(&s_mm[0][d], o);
                            atomicMax(&s_mm[1][d], o);
                        }
                    }
            }
        }
    }
    __syncthreads();
    if (threadIdx.x < D) {
        atomicMin(minmax + threadIdx.x, s_mm[0][threadIdx.x]);
        atomicMax(minmax + D + threadIdx.x, s_mm[1][threadIdx.x]);
    }
}

// make_query (proj/src/builder.cpp:110-127) for vectors: unknown coordinate -> mean, project in
// the canonical order, quantise with the index's lo / hi.  One warp per query, lane d = dim d.
__global__ void __launch_bounds__(32) k_vec_make_query(const float* __restrict__ Q, const uint8_t* __restrict__ known,
                                                       uint64_t nq, int dim, int D, const double* __restrict__ mean,
                                                       const double* __restrict__ comp,
                                                       const unsigned long long* __restrict__ minmax,
                                                       uint8_t* __restrict__ out) {
    const uint64_t q = blockIdx.x;
    const int d = threadIdx.x;
    if (q >= nq || d >= D) return;
    const float* x = Q + q * dim;
    const uint8_t* kn = known + q * dim;
    double y = 0.0;
    for (int j = 0; j < dim; ++j) {
        const double v = kn[j] ? static_cast<double>(x[j]) : mean[j];
        y = __fma_rn(comp[j * D + d], __dsub_rn(v, mean[j]), y);
    }
    out[q * D + d] = static_cast<uint8_t>(quantize_rn(ordered_to_double_hd(minmax[d]), ordered_to_double_hd(minmax[D + d]), y));
}

// ---------------------------------------------------------------- host side
template <int D>
static void launch_vec_project(zi_ctx* ctx, const float* X, uint64_t n, int dim, const double* mean, const double* comp,
                               double* Y, unsigned long long* mm) {
    constexpr int NT = (D + 7) / 8;
    const int KS = (dim + 3) / 4;
    const size_t smem = (static_cast<size_t>(KS) * NT * 32 + static_cast<size_t>(KS) * 4) * sizeof(double);
    smem_attr(ctx->device, k_vec_project<D>, smem);
    const uint64_t warps = (n + 8 * kVpGroups - 1) / (8 * kVpGroups);
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((warps + kVpThreads / 32 - 1) / (kVpThreads / 32),
                                                                   static_cast<uint64_t>(ctx->num_sms) * 8));
    ZI_LAUNCH(ctx, "vec_project", k_vec_project<D>, grid, kVpThreads, smem, X, n, dim, mean, comp, Y, mm);
}

void vector_index_build(zi_vector_index* vi, const float* h_X) {
    zi_ctx* ctx = vi->ctx;
    const uint64_t n = vi->n;
    const int dim = vi->dim;
    vi->X.ensure(n * dim);
    ZI_CUDA(cudaMemcpyAsync(vi->X.p, h_X, n * dim * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
    vi->Xd = vi->X.p;
    build_vector_index_device(vi);
}

void build_vector_index_device(zi_vector_index* vi) {
    zi_ctx* ctx = vi->ctx;
    const uint64_t n = vi->n;
    const int dim = vi->dim, D = vi->dims;
    const float* X = vi->Xd;
    const int nstripe = static_cast<int>((n + kStripe - 1) / kStripe);
    // mean
    vi->mean.ensure(dim);
    dbuf<double>& part = vi->scratch;
    const int Pd = (dim + 7) / 8 * 8, T = Pd / 8, ntiles = T * (T + 1) / 2;
    part.ensure(std::max<size_t>(static_cast<size_t>(nstripe) * dim, static_cast<size_t>(nstripe) * ntiles * 64));
    ZI_LAUNCH(ctx, "vec_colsum", k_vec_colsum, nstripe, 1024, 0, X, n, dim, part.p);
    ZI_LAUNCH(ctx, "vec_mean", k_vec_mean, (dim + 127) / 128, 128, 0, part.p, nstripe, dim, n, vi->mean.p);
    // covariance
    const size_t raw_words = ((static_cast<size_t>(kGramRows) * dim + 3) / 4) * 4;
    const size_t gsmem = static_cast<size_t>(kGramRows) * (Pd + 4) * sizeof(double) + 2 * raw_words * sizeof(float);
    {
        const int Tb = (T + 3) / 4, nblocks = Tb * (Tb + 1) / 2;
        const int warps = std::min(nblocks, kGramMaxWarps);
        const unsigned gy = static_cast<unsigned>((nblocks + kGramMaxWarps - 1) / kGramMaxWarps);
        smem_attr(ctx->device, k_vec_gram_blk, gsmem);
        ZI_LAUNCH(ctx, "vec_gram", k_vec_gram_blk, dim3(nstripe, gy), warps * 32, gsmem, X, n, dim, Pd, vi->mean.p,
                  nblocks, part.p);
    }
    vi->cov.ensure(static_cast<size_t>(dim) * dim);
    ZI_LAUNCH(ctx, "vec_gram_reduce", k_vec_gram_reduce, ntiles, 64, 0, part.p, nstripe, ntiles, T, dim, n, vi->cov.p);
    // eigen-solve (k_pca.cu), components [j][d]
    vi->comp.ensure(static_cast<size_t>(dim) * D);
    vi->eig.ensure(32);
    vi->pca_work.ensure(pca_work_doubles(dim, D));
    if (!pca_from_cov_on_device(ctx, vi->cov.p, dim, D, vi->comp.p, vi->eig.p, vi->pca_work.p))
        throw error(ZI_E_INVALID, "vector index: dim must be in [3, 224] and dims <= 32");
    // projection + min/max, quantise + interleave, sort by (Morton, row), finalize
    vi->minmax.ensure(2 * D);
    ZI_CUDA(cudaMemsetAsync(vi->minmax.p, 0xff, D * sizeof(unsigned long long), ctx->stream));
    ZI_CUDA(cudaMemsetAsync(vi->minmax.p + D, 0x00, D * sizeof(unsigned long long), ctx->stream));
    vi->Y.ensure(static_cast<size_t>(D) * n);
    switch (D) {
#define ZI_VP(DD) \
    case DD: launch_vec_project<DD>(ctx, X, n, dim, vi->mean.p, vi->comp.p, vi->Y.p, vi->minmax.p); break;
        ZI_VP(1) ZI_VP(2) ZI_VP(3) ZI_VP(4) ZI_VP(5) ZI_VP(6) ZI_VP(7) ZI_VP(8)
        ZI_VP(9) ZI_VP(10) ZI_VP(11) ZI_VP(12) ZI_VP(13) ZI_VP(14) ZI_VP(15) ZI_VP(16)
        ZI_VP(17) ZI_VP(18) ZI_VP(19) ZI_VP(20) ZI_VP(21) ZI_VP(22) ZI_VP(23) ZI_VP(24)
        ZI_VP(25) ZI_VP(26) ZI_VP(27) ZI_VP(28) ZI_VP(29) ZI_VP(30) ZI_VP(31) ZI_VP(32)
#undef ZI_VP
        default: throw error(ZI_E_INVALID, "dims must be in [1, 32]");
    }
    const int W = (D + 3) / 4;
    vi->recs.ensure(static_cast<size_t>(W + 1) * n);
    uint32_t* keyw = vi->recs.p;
    uint32_t* val = vi->recs.p + static_cast<size_t>(W) * n;
    quantize_interleave(ctx, vi->Y.p, vi->minmax.p, n, n, 0, D, keyw, val);
    uint32_t* sorted[10];
    morton_sort_records(ctx, keyw, val, n, 1, D, false, sorted);
    vi->index.ctx = ctx;
    vi->index.layout_id = 0;
    finalize_index(ctx, sorted[0], sorted[W], n, 0, n, D, nullptr, &vi->index);
    vi->host_model = false;
}

void vector_make_queries(zi_vector_index* vi, const float* d_Q, const uint8_t* d_known, uint64_t nq, uint8_t* d_out) {
    if (nq == 0) return;
    ZI_LAUNCH(vi->ctx, "vec_make_query", k_vec_make_query, static_cast<unsigned>(nq), 32, 0, d_Q, d_known, nq, vi->dim,
              vi->dims, vi->mean.p, vi->comp.p, vi->minmax.p, d_out);
}

void vector_sync_host_model(zi_vector_index* vi) {
    if (vi->host_model) return;
    const int dim = vi->dim, D = vi->dims;
    std::vector<double> comp(static_cast<size_t>(dim) * D);
    std::vector<unsigned long long> mm(2 * D);
    vi->h_mean.resize(dim);
    vi->h_eig.resize(D);
    zi_ctx* ctx = vi->ctx;
    ZI_CUDA(cudaMemcpyAsync(vi->h_mean.data(), vi->mean.p, dim * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    ZI_CUDA(cudaMemcpyAsync(comp.data(), vi->comp.p, comp.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    ZI_CUDA(cudaMemcpyAsync(vi->h_eig.data(), vi->eig.p, D * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    ZI_CUDA(cudaMemcpyAsync(mm.data(), vi->minmax.p, mm.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                            ctx->stream));
    ZI_CUDA(cudaStreamSynchronize(ctx->stream));
    vi->h_comp.assign(static_cast<size_t>(D) * dim, 0.0);  // rows d of dim (the reference's column d)
    for (int j = 0; j < dim; ++j)
        for (int d = 0; d < D; ++d) vi->h_comp[static_cast<size_t>(d) * dim + j] = comp[static_cast<size_t>(j) * D + d];
    vi->h_lo.resize(D);
    vi->h_hi.resize(D);
    for (int d = 0; d < D; ++d) {
        vi->h_lo[d] = ordered_to_double(mm[d]);
        vi->h_hi[d] = ordered_to_double(mm[D + d]);
    }
    vi->host_model = true;
}

}  // namespace zi
