// k_query.cu -- per-iteration query kernels (sm_100a):
//   K6 query_prep   select_index + make_query   proj/src/engine.cpp:162-176; builder.cpp:110-127
//   K7 seed         lower_bound in Morton order + window scoring (subinterval analogue,
//                   proj/src/zcurve.cpp:140-179) -> first k-th bound
//   K8 knn_scan     bbox-pruned exact scan; prune iff (lb<<32) > bound, the reference's
//                   prunable() predicate (proj/src/zcurve.cpp:290-292) on packed values
//   K8b knn_merge   exact top-k in (distance, key) order (knn_list::sorted, zcurve.cpp:51-62)
//   K9 refine       masked_cost_at over the candidates, min (cost, key)  engine.cpp:197-210, 48-76
//   K10 brute_force masked cost over the whole dictionary             engine.cpp:220-236
//
// Exactness argument: every bound used is the packed (dist,key) value of the k-th element of
// some SUBSET of the index, so it is >= the true k-th value; an entry is dropped only if it is
// above such a bound, or if k smaller entries exist in the same CTA buffer.  Packed values are
// unique (keys are), so the final k smallest are exactly the reference's knn_search result.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace zi {

constexpr int kScanThreads = 256;
constexpr int kScanCap = 4096;     // CTA candidate buffer (u64)
constexpr int kMergeThreads = 1024;
constexpr int kMergeCap = 4096;
constexpr uint32_t kMaxScanK = 2048;  // above: exhaustive sort path

// device workspace of one query
struct qws {
    unsigned long long bound;
    unsigned long long best;
    uint32_t q4[8];
    uint8_t q[32];
    uint32_t lid;
    uint32_t count;
    uint32_t overflow;  // fused single-CTA query gave up (too many candidates): host falls back
    uint32_t dbg_total, dbg_m;  // merge: candidates in all CTA lists / candidates <= the final bound
    uint32_t done;              // k_query_one: CTAs finished (the last one merges)
    uint32_t gcount;            // k_query_one: candidates appended to the compact global list
    unsigned long long final_bound;
    unsigned long long tphase[10];  // debug: %globaltimer at phase boundaries (CTA 0 / last CTA)
};

// Fill-loop query result in mapped pinned host memory: written by the last CTA of k_query_one,
// then `seq` is published after a system-scope fence -- the host spins on it instead of a D2H copy
// plus a stream synchronisation.
struct qres {
    unsigned long long best;
    uint32_t lid, count, overflow;
    volatile uint32_t seq;
};

struct index_view {
    const uint32_t* planes;
    const uint32_t* keys;
    const uint32_t* bmin;
    const uint32_t* bmax;
    uint64_t n, nblk;
    int P, D;
};

// the 8 layout views; kernels after the prep pick views.v[ws->lid] on the device, so the
// query needs no host round trip between select_index and the scan
struct views8 {
    index_view v[8];
};

__device__ inline void block_bitonic_sort(unsigned long long* a, int n) {
    for (int size = 2; size <= n; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < (n >> 1); t += blockDim.x) {
                const int i = 2 * stride * (t / stride) + (t % stride);
                const int j = i + stride;
                const bool up = (i & size) == 0;
                const unsigned long long x = a[i], y = a[j];
                if ((x > y) == up) {
                    a[i] = y;
                    a[j] = x;
                }
            }
            __syncthreads();
        }
}

__device__ inline int pow2ceil(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

__device__ inline uint32_t entry_byte(const index_view& v, uint64_t i, int d) {
    return plane_byte(v.planes[static_cast<size_t>(d >> 2) * v.n + i], d);
}

// morton_less(entry_i, q)  (proj/include/zinpaint/morton.hpp:18-29)
__device__ inline bool entry_less_query(const index_view& v, uint64_t i, const uint8_t* q) {
    uint32_t best_diff = 0;
    int best_dim = 0;
    for (int d = 0; d < v.D; ++d) {
        const uint32_t diff = entry_byte(v, i, d) ^ q[d];
        if (less_msb(best_diff, diff)) {
            best_diff = diff;
            best_dim = d;
        }
    }
    return entry_byte(v, i, best_dim) < q[best_dim];
}

__device__ inline uint32_t entry_dist(const index_view& v, uint64_t i, const uint32_t* q4, int norm) {
    uint32_t acc = 0;
    for (int p = 0; p < v.P; ++p) acc = dist4(v.planes[static_cast<size_t>(p) * v.n + i], q4[p], norm, acc);
    return acc;
}

// Packed (dist<<32 | key) of the 8 entries lane, lane+32, ..., lane+224 of 256-entry block b;
// all 8*(P+1) loads are issued before any arithmetic (P = dim planes, a compile-time constant).
template <int P>
__device__ inline void score_block(const index_view& v, uint64_t b, const uint32_t (&q4)[8], int norm,
                                   unsigned long long (&c)[8]) {
    const int lane = threadIdx.x & 31;
    const uint64_t base = b * 256 + lane;
    uint32_t w[8][P], kk[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const uint64_t i = base + e * 32;
        const bool ok = i < v.n;
#pragma unroll
        for (int p = 0; p < P; ++p) w[e][p] = ok ? __ldg(v.planes + static_cast<size_t>(p) * v.n + i) : 0u;
        kk[e] = ok ? __ldg(v.keys + i) : 0u;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        uint32_t dist = 0;
#pragma unroll
        for (int p = 0; p < P; ++p) dist = dist4(w[e][p], q4[p], norm, dist);
        c[e] = base + e * 32 < v.n ? pack_candidate(dist, kk[e]) : kU64Max;
    }
}

// K7': seed from the bbox table -- each warp finds the block with the smallest lower bound among
// its share of all blocks, scores it, and the k-th smallest packed value of those 2048 entries
// (any k real entries give a valid bound) becomes the starting bound.  Needs 2048 u64 of s_buf
// and blockDim.x == 256.
template <int P>
__device__ void seed_bound_bbox(const index_view& v, const uint32_t (&q4)[8], uint32_t k, int norm,
                                unsigned long long* s_buf, qws* ws) {
    __shared__ unsigned long long s_wmin[8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    unsigned long long mine = kU64Max;
    for (uint64_t b = static_cast<uint64_t>(warp) * 32 + lane; b < v.nblk; b += 256) {
        uint32_t lb = 0;
#pragma unroll
        for (int p = 0; p < P; ++p)
            lb = gap4(q4[p], v.bmin[static_cast<size_t>(p) * v.nblk + b], v.bmax[static_cast<size_t>(p) * v.nblk + b], norm, lb);
        const unsigned long long c = (static_cast<unsigned long long>(lb) << 32) | b;
        mine = c < mine ? c : mine;
    }
    mine = warp_min(mine);
    if (lane == 0) s_wmin[warp] = mine;
    __syncthreads();
    const unsigned long long sb = s_wmin[warp];
    unsigned long long c[8];
    if (sb != kU64Max) {
        score_block<P>(v, sb & 0xffffffffull, q4, norm, c);
    } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) c[e] = kU64Max;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) s_buf[warp * 256 + e * 32 + lane] = c[e];
    __syncthreads();
    block_bitonic_sort(s_buf, 2048);
    if (tid == 0) {
        ws->bound = k <= 2048 ? s_buf[k - 1] : kU64Max;
        ws->best = kU64Max;
        ws->count = 0;
        ws->overflow = 0;
    }
}

// K7: lower_bound of q in Morton order (256-ary search), then score a window of `win`
// entries around it and take the k-th smallest packed value as the starting bound.
__device__ void seed_bound(const index_view& v, const uint8_t* s_q, const uint32_t* s_q4, uint32_t k, int norm,
                           int win, unsigned long long* s_buf, qws* ws) {
    __shared__ uint64_t s_lo, s_hi;
    const int tid = threadIdx.x;
    if (tid == 0) {
        s_lo = 0;
        s_hi = v.n;
    }
    __syncthreads();
    while (true) {
        const uint64_t lo = s_lo, hi = s_hi;
        const uint64_t len = hi - lo;
        if (len <= static_cast<uint64_t>(blockDim.x)) {
            const bool less = tid < static_cast<int>(len) && entry_less_query(v, lo + tid, s_q);
            const int c = __syncthreads_count(less);
            if (tid == 0) s_lo = lo + c;
            __syncthreads();
            break;
        }
        const int np = blockDim.x;
        const uint64_t piv = lo + (static_cast<uint64_t>(tid) + 1) * len / (np + 1);
        const bool less = entry_less_query(v, piv, s_q);
        const int c = __syncthreads_count(less);
        if (tid == 0) {
            const uint64_t nlo = c > 0 ? lo + static_cast<uint64_t>(c) * len / (np + 1) + 1 : lo;
            const uint64_t nhi = c < np ? lo + (static_cast<uint64_t>(c) + 1) * len / (np + 1) : hi;
            s_lo = nlo;
            s_hi = nhi;
        }
        __syncthreads();
    }
    const uint64_t pos = s_lo;
    const uint64_t wn = v.n < static_cast<uint64_t>(win) ? v.n : static_cast<uint64_t>(win);
    uint64_t start = pos > wn / 2 ? pos - wn / 2 : 0;
    if (start + wn > v.n) start = v.n - wn;
    for (int t = tid; t < win; t += blockDim.x) {
        unsigned long long c = kU64Max;
        if (static_cast<uint64_t>(t) < wn) {
            const uint64_t i = start + t;
            c = pack_candidate(entry_dist(v, i, s_q4, norm), v.keys[i]);
        }
        s_buf[t] = c;
    }
    __syncthreads();
    block_bitonic_sort(s_buf, win);
    if (tid == 0) {
        ws->bound = (wn >= k && k <= static_cast<uint32_t>(win)) ? s_buf[k - 1] : kU64Max;
        ws->best = kU64Max;
        ws->count = 0;
    }
}

template <int P>
__global__ void __launch_bounds__(256) k_seed_query(index_view v, const uint8_t* __restrict__ query, qws* ws,
                                                    uint32_t k, int norm, int win) {
    extern __shared__ unsigned long long s_buf[];
    __shared__ uint8_t s_q[32];
    __shared__ uint32_t s_q4[8];
    if (threadIdx.x < 32) s_q[threadIdx.x] = threadIdx.x < v.D ? query[threadIdx.x] : 0;
    __syncthreads();
    if (threadIdx.x < 8) {
        uint32_t w = 0;
        for (int b = 0; b < 4; ++b) w |= static_cast<uint32_t>(s_q[threadIdx.x * 4 + b]) << (8 * b);
        s_q4[threadIdx.x] = w;
        ws->q4[threadIdx.x] = w;
    }
    if (threadIdx.x < 32) ws->q[threadIdx.x] = s_q[threadIdx.x];
    if (threadIdx.x == 0) ws->lid = 0;
    __syncthreads();
    uint32_t q4[8];
#pragma unroll
    for (int p = 0; p < 8; ++p) q4[p] = s_q4[p];
    (void)win;
    seed_bound_bbox<P>(v, q4, k, norm, s_buf, ws);
}

// multi-index: select_index + make_query on the device, then the seed on the chosen layout
struct mi_view {
    index_view idx[8];
    const int32_t* local;  // 8*m  (r*K + c)
    const double* mean;    // 8*mc
    const double* comp;    // 8*mc*D  ([layout][j][d])
    const unsigned long long* minmax;  // 8*2D
    int m, C, K, D;
};

// Dynamic smem: the seed window (win u64) | x row of the chosen layout (mc doubles) |
// components of the chosen layout ([j][d], mc*D doubles) | target (K*K*C + K*K bytes).
template <int P>
__global__ void __launch_bounds__(256) k_query_prep(mi_view mv, const uint8_t* __restrict__ target, qws* ws,
                                                    uint32_t k, int norm, int win) {
    extern __shared__ unsigned long long s_buf[];
    __shared__ int s_ov[8];
    __shared__ int s_lid;
    __shared__ uint8_t s_q[32];
    __shared__ uint32_t s_q4[8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int KK = mv.K * mv.K, mc = mv.m * mv.C;
    double* s_xc = reinterpret_cast<double*>(s_buf + win);     // mc
    double* s_comp = s_xc + mc;                                  // mc * D
    uint8_t* s_t = reinterpret_cast<uint8_t*>(s_comp + static_cast<size_t>(mc) * mv.D);
    const int tbytes = KK * mv.C + KK;
    for (int i = tid; i < tbytes; i += blockDim.x) s_t[i] = target[i];
    __syncthreads();
    const uint8_t* tv = s_t;
    const uint8_t* tk = s_t + KK * mv.C;
    // select_index (proj/src/engine.cpp:162-176): strict '>' from 0, ties -> lowest id
    if (warp < 8) {
        int ov = 0;
        for (int p = lane; p < mv.m; p += 32) ov += tk[mv.local[warp * mv.m + p]] != 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ov += __shfl_xor_sync(0xffffffffu, ov, o);
        if (lane == 0) s_ov[warp] = ov;
    }
    __syncthreads();
    if (tid == 0) {
        int best = 0, bid = 0;
        for (int l = 0; l < 8; ++l)
            if (s_ov[l] > best) {
                best = s_ov[l];
                bid = l;
            }
        s_lid = bid;
        ws->lid = static_cast<uint32_t>(bid);
    }
    if (tid < 32) s_q[tid] = 0;
    __syncthreads();
    const int lid = s_lid;
    // make_query (proj/src/builder.cpp:110-127): xc_j = x_j - mean_j with unknown pixels at the
    // mean (xc = +0.0 exactly), staged in parallel; then the canonical fp64 chain per dim
    {
        const double* mean = mv.mean + static_cast<size_t>(lid) * mc;
        const int32_t* loc = mv.local + lid * mv.m;
        for (int j = tid; j < mc; j += blockDim.x) {
            const int l = loc[j / mv.C];
            const double mj = mean[j];
            const double x = tk[l] ? static_cast<double>(tv[l * mv.C + j % mv.C]) : mj;
            s_xc[j] = __dsub_rn(x, mj);
        }
        const double* comp = mv.comp + static_cast<size_t>(lid) * mc * mv.D;
        for (int i = tid; i < mc * mv.D; i += blockDim.x) s_comp[i] = comp[i];
    }
    __syncthreads();
    if (tid < mv.D) {
        const int d = tid;
        double y = 0.0;
        for (int j = 0; j < mc; ++j) y = __fma_rn(s_comp[j * mv.D + d], s_xc[j], y);
        const unsigned long long* mm = mv.minmax + static_cast<size_t>(lid) * 2 * mv.D;
        s_q[d] = quantize_rn(ordered_to_double_hd(mm[d]), ordered_to_double_hd(mm[mv.D + d]), y);
    }
    __syncthreads();
    if (tid < 8) {
        uint32_t w = 0;
        for (int b = 0; b < 4; ++b) w |= static_cast<uint32_t>(s_q[tid * 4 + b]) << (8 * b);
        s_q4[tid] = w;
        ws->q4[tid] = w;
    }
    if (tid < 32) ws->q[tid] = s_q[tid];
    __syncthreads();
    uint32_t q4[8];
#pragma unroll
    for (int p = 0; p < 8; ++p) q4[p] = s_q4[p];
    seed_bound_bbox<P>(mv.idx[lid], q4, k, norm, s_buf, ws);
}

// keep the <= k smallest of buf[0..cnt) (sorted), tighten the bounds
__device__ void compact_buffer(unsigned long long* buf, int* s_cnt, unsigned long long* s_bound, uint32_t k,
                               qws* ws, bool publish) {
    const int cnt = *s_cnt;
    if (cnt == 0) return;
    const int sz = pow2ceil(cnt < 2 ? 2 : cnt);
    for (int t = cnt + threadIdx.x; t < sz; t += blockDim.x) buf[t] = kU64Max;
    __syncthreads();
    block_bitonic_sort(buf, sz);
    if (threadIdx.x == 0) {
        int keep = cnt < static_cast<int>(k) ? cnt : static_cast<int>(k);
        if (cnt >= static_cast<int>(k)) {
            const unsigned long long kth = buf[k - 1];
            if (kth < *s_bound) *s_bound = kth;
            if (publish) atomicMin(&ws->bound, kth);
        }
        // entries above the bound can never be in the answer
        while (keep > 0 && buf[keep - 1] > *s_bound) --keep;
        *s_cnt = keep;
    }
    __syncthreads();
}

// K8: one CTA = interleaved 256-entry blocks; 8 warps score one block each per round.
template <int P>
__global__ void __launch_bounds__(kScanThreads) k_knn_scan(views8 V, qws* ws, uint32_t k, int norm,
                                                           uint32_t* __restrict__ cand_cnt,
                                                           unsigned long long* __restrict__ cand) {
    __shared__ unsigned long long s_buf[kScanCap];
    __shared__ int s_cnt;
    __shared__ unsigned long long s_bound;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const index_view v = V.v[ws->lid & 7];
    uint32_t q4[8];
#pragma unroll
    for (int p = 0; p < 8; ++p) q4[p] = ws->q4[p];
    if (tid == 0) {
        s_cnt = 0;
        s_bound = *reinterpret_cast<volatile unsigned long long*>(&ws->bound);
    }
    __syncthreads();
    const uint64_t G = gridDim.x;
    const uint64_t rounds = (v.nblk + 8 * G - 1) / (8 * G);
    for (uint64_t r = 0; r < rounds; ++r) {
        const uint64_t b = blockIdx.x + (r * 8 + warp) * G;
        const unsigned long long bound = s_bound;
        if (b < v.nblk) {
            uint32_t lb = 0;
#pragma unroll
            for (int p = 0; p < P; ++p)
                lb = gap4(q4[p], v.bmin[static_cast<size_t>(p) * v.nblk + b], v.bmax[static_cast<size_t>(p) * v.nblk + b],
                          norm, lb);
            if ((static_cast<unsigned long long>(lb) << 32) <= bound) {
                unsigned long long c[8];
                score_block<P>(v, b, q4, norm, c);
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    if (c[e] != kU64Max && c[e] <= bound) s_buf[atomicAdd(&s_cnt, 1)] = c[e];
            }
            (void)lane;
        }
        __syncthreads();
        if (s_cnt > kScanCap - 8 * 256) {
            compact_buffer(s_buf, &s_cnt, &s_bound, k, ws, true);
        } else if (tid == 0) {
            const unsigned long long g = *reinterpret_cast<volatile unsigned long long*>(&ws->bound);
            if (g < s_bound) s_bound = g;
        }
        __syncthreads();
    }
    compact_buffer(s_buf, &s_cnt, &s_bound, k, ws, true);
    const int cnt = s_cnt;
    for (int t = tid; t < cnt; t += blockDim.x) cand[static_cast<size_t>(blockIdx.x) * k + t] = s_buf[t];
    if (tid == 0) cand_cnt[blockIdx.x] = static_cast<uint32_t>(cnt);
}

// K8b: merge the per-CTA lists into the exact top-k (sorted); out[0..count)
__global__ void __launch_bounds__(kMergeThreads) k_knn_merge(qws* ws, uint32_t k, int G,
                                                             const uint32_t* __restrict__ cand_cnt,
                                                             const unsigned long long* __restrict__ cand,
                                                             unsigned long long* __restrict__ out) {
    __shared__ unsigned long long s_buf[kMergeCap];
    __shared__ uint32_t s_pref[1025];  // G <= 1024 CTA lists
    __shared__ int s_cnt;
    __shared__ unsigned long long s_bound;
    __shared__ uint32_t s_warp[32];
    const int tid = threadIdx.x;
    // prefix over the CTA list lengths (G <= 1024)
    uint32_t carry = 0;
    for (int base = 0; base < G; base += kMergeThreads) {
        const int i = base + tid;
        const uint32_t c = i < G ? cand_cnt[i] : 0;
        uint32_t x = c;
        const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_warp[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint32_t t = s_warp[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
                if (lane >= o) t += y;
            }
            s_warp[lane] = t;
        }
        __syncthreads();
        const uint32_t ex = carry + (warp ? s_warp[warp - 1] : 0) + x - c;
        if (i < G) s_pref[i] = ex;
        carry += s_warp[31];
        __syncthreads();
    }
    if (tid == 0) {
        s_pref[G] = carry;
        s_cnt = 0;
        s_bound = ws->bound;
    }
    __syncthreads();
    const uint32_t total = s_pref[G];
    // fast path: everything <= the final bound fits -> exact ranks by counting (values are unique)
    {
        const unsigned long long bound = s_bound;
        for (uint32_t f = tid; f < total; f += kMergeThreads) {
            int lo = 0, hi = G;
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (s_pref[mid] <= f) lo = mid;
                else hi = mid;
            }
            const unsigned long long c = cand[static_cast<size_t>(lo) * k + (f - s_pref[lo])];
            if (c <= bound) {
                const int slot = atomicAdd(&s_cnt, 1);
                if (slot < kMergeCap) s_buf[slot] = c;
            }
        }
        __syncthreads();
        const int m = s_cnt;
        if (tid == 0) {
            ws->dbg_total = total;
            ws->dbg_m = static_cast<uint32_t>(m);
        }
        if (m <= kMergeThreads) {
            if (tid < m) {
                const unsigned long long c = s_buf[tid];
                int r = 0;
                for (int u = 0; u < m; ++u) r += s_buf[u] < c;
                if (r < static_cast<int>(k)) out[r] = c;
            }
            if (tid == 0) ws->count = static_cast<uint32_t>(m < static_cast<int>(k) ? m : static_cast<int>(k));
            return;
        }
        __syncthreads();
        if (tid == 0) s_cnt = 0;
        __syncthreads();
    }
    const int chunk = kMergeCap - static_cast<int>(k);
    for (uint32_t f0 = 0; f0 < total; f0 += chunk) {
        const unsigned long long bound = s_bound;
        for (uint32_t f = f0 + tid; f < f0 + chunk && f < total; f += kMergeThreads) {
            // owner list of flat index f
            int lo = 0, hi = G;  // s_pref[lo] <= f < s_pref[hi]
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (s_pref[mid] <= f) lo = mid;
                else hi = mid;
            }
            const unsigned long long c = cand[static_cast<size_t>(lo) * k + (f - s_pref[lo])];
            if (c <= bound) s_buf[atomicAdd(&s_cnt, 1)] = c;
        }
        __syncthreads();
        compact_buffer(s_buf, &s_cnt, &s_bound, k, ws, false);
    }
    const int cnt = s_cnt;
    for (int t = tid; t < cnt; t += kMergeThreads) out[t] = s_buf[t];
    if (tid == 0) ws->count = static_cast<uint32_t>(cnt);
}

// K9: refine -- masked_cost_at (proj/src/engine.cpp:48-76) per candidate, warp per candidate,
// min over packed (cost, key) (engine.cpp:202-209).
// cnt candidates of `list` (global or shared); s_t: >= K*K*C + 2*K*K + 2 bytes of shared memory
__device__ void refine_list(const uint8_t* __restrict__ img, int w, int C, int K, const uint8_t* __restrict__ target,
                            const unsigned long long* list, int cnt, int norm, uint8_t* s_t, qws* ws,
                            int cost_slots = 1 << 30) {
    __shared__ int s_nloc;
    __shared__ unsigned long long s_best;
    const int KK = K * K;
    uint16_t* s_loc = reinterpret_cast<uint16_t*>(s_t + ((KK * C + 1) & ~1));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    for (int i = threadIdx.x; i < KK * C; i += blockDim.x) s_t[i] = target[i];
    if (warp == 0) {  // known locals, ascending (known_locals_of, engine.cpp:16-22), via ballots
        int c = 0;
        for (int base = 0; base < KK; base += 32) {
            const bool kn = base + lane < KK && target[KK * C + base + lane] != 0;
            const unsigned m = __ballot_sync(0xffffffffu, kn);
            if (kn) s_loc[c + __popc(m & ((1u << lane) - 1u))] = static_cast<uint16_t>(base + lane);
            c += __popc(m);
        }
        if (lane == 0) {
            s_nloc = c;
            s_best = kU64Max;
        }
    }
    __syncthreads();
    const int nloc = s_nloc;
    if (cnt > cost_slots) {  // very large k: one warp per candidate
        for (int e = warp; e < cnt; e += nwarp) {
            const uint32_t key = static_cast<uint32_t>(list[e] & 0xffffffffu);
            uint32_t acc = 0;
            for (int li = lane; li < nloc; li += 32) {
                const int l = s_loc[li];
                const uint8_t* s = img + (static_cast<size_t>((key >> 16) + l / K) * w + (key & 0xffff) + l % K) * C;
                for (int c = 0; c < C; ++c) {
                    const int d = static_cast<int>(s_t[l * C + c]) - static_cast<int>(__ldg(s + c));
                    acc += norm == 0 ? static_cast<uint32_t>(d * d) : static_cast<uint32_t>(d < 0 ? -d : d);
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) atomicMin(&s_best, pack_candidate(acc, key));
        }
        __syncthreads();
        if (threadIdx.x == 0) ws->best = s_best;
        return;
    }
    // all (candidate, known pixel) pairs in parallel; per-candidate sums in shared memory
    uint32_t* s_cost = reinterpret_cast<uint32_t*>(
        s_t + ((((KK * C + 1) & ~1) + 2 * KK + 15) & ~15));  // cnt words, 16-byte aligned
    for (int e = threadIdx.x; e < cnt; e += blockDim.x) s_cost[e] = 0;
    __syncthreads();
    const int pairs = cnt * nloc;
    const int stride = blockDim.x;
    // 4 independent pairs per step so their image loads are in flight together
    for (int p0 = threadIdx.x; p0 < pairs; p0 += 4 * stride) {
        uint8_t sv[4][3];
        int pe[4], pl[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int pi = p0 + u * stride;
            pe[u] = -1;
            if (pi < pairs) {
                const int e = pi / nloc, li = pi - e * nloc;
                const uint32_t key = static_cast<uint32_t>(list[e] & 0xffffffffu);
                const int l = s_loc[li];
                const uint8_t* s = img + (static_cast<size_t>((key >> 16) + l / K) * w + (key & 0xffff) + l % K) * C;
                pe[u] = e;
                pl[u] = l;
#pragma unroll
                for (int c = 0; c < 3; ++c) sv[u][c] = c < C ? __ldg(s + c) : 0;
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (pe[u] < 0) continue;
            const uint8_t* t = s_t + pl[u] * C;
            uint32_t acc = 0;
            for (int c = 0; c < C; ++c) {
                const int d = static_cast<int>(t[c]) - static_cast<int>(sv[u][c]);
                acc += norm == 0 ? static_cast<uint32_t>(d * d) : static_cast<uint32_t>(d < 0 ? -d : d);
            }
            atomicAdd(&s_cost[pe[u]], acc);
        }
    }
    __syncthreads();
    unsigned long long mine = kU64Max;
    for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
        const unsigned long long c = pack_candidate(s_cost[e], static_cast<uint32_t>(list[e] & 0xffffffffu));
        mine = c < mine ? c : mine;
    }
    mine = warp_min(mine);
    if (lane == 0) atomicMin(&s_best, mine);
    (void)warp;
    (void)nwarp;
    __syncthreads();
    if (threadIdx.x == 0) ws->best = s_best;
}

constexpr int kRefineSlots = 4096;

__global__ void __launch_bounds__(1024) k_refine(const uint8_t* __restrict__ img, int w, int C, int K,
                                                 const uint8_t* __restrict__ target, qws* ws,
                                                 const unsigned long long* __restrict__ list, int norm) {
    extern __shared__ uint8_t s_t[];
    refine_list(img, w, C, K, target, list, static_cast<int>(ws->count), norm, s_t, ws, kRefineSlots);
}

__device__ inline void warp_bitonic_sort(unsigned long long* a, int n);

__device__ inline unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define ZI_TPHASE(i) \
    if (threadIdx.x == 0 && (blockIdx.x == 0 || (i) >= 6)) ws->tphase[i] = gtimer();

// Exact top-k selection in shared memory (any blockDim): buf[0..m) holds unique packed values;
// a histogram of their distances finds the bin holding the k-th, the boundary bin is ranked
// exactly, and the k winners are sorted into sel[0..min(k,m)).  Returns that count, or -1 when
// the boundary bin holds more than tmp_cap values (caller falls back).  hist: nbins+1 words.
__device__ int select_topk(const unsigned long long* buf, int m, uint32_t k, unsigned long long* sel,
                           unsigned long long* tmp, int tmp_cap, uint32_t* hist, int nbins, uint32_t maxd,
                           bool sort_result) {
    __shared__ int s_nsel, s_ntmp, s_B, s_cumB;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nt = blockDim.x;
    if (m > static_cast<int>(k)) {
        for (int i = tid; i <= nbins; i += nt) hist[i] = 0;
        if (tid == 0) {
            s_nsel = 0;
            s_ntmp = 0;
            s_B = -1;
        }
        __syncthreads();
        // bin = floor(dist * nbins / (maxd + 1)) as a multiply-shift: monotone in dist, < nbins
        const uint64_t scale = (static_cast<uint64_t>(nbins) << 32) / (static_cast<uint64_t>(maxd) + 1);
        for (int i = tid; i < m; i += nt) {
            const uint32_t bin = static_cast<uint32_t>(((buf[i] >> 32) * scale) >> 32);
            atomicAdd(&hist[bin < static_cast<uint32_t>(nbins) ? bin : nbins - 1], 1u);
        }
        __syncthreads();
        if (warp == 0) {  // first bin where the running count reaches k
            uint32_t run = 0;
            for (int base = 0; base < nbins; base += 32) {
                uint32_t x = base + lane < nbins ? hist[base + lane] : 0;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                const unsigned hit = __ballot_sync(0xffffffffu, run + x >= k);
                if (hit) {
                    const int src = __ffs(hit) - 1;
                    const uint32_t incl = __shfl_sync(0xffffffffu, x, src);
                    if (lane == 0) {
                        s_B = base + src;
                        s_cumB = static_cast<int>(run + incl - hist[base + src]);
                    }
                    break;
                }
                run += __shfl_sync(0xffffffffu, x, 31);
            }
        }
        __syncthreads();
        const int B = s_B, cumB = s_cumB;
        if (B < 0 || B >= nbins) {
            if (tid == 0) printf("select_topk: no boundary bin (m=%d k=%u maxd=%u)\n", m, k, maxd);
            return -1;
        }
        if (static_cast<int>(hist[B]) > tmp_cap) return -1;
        for (int i = tid; i < m; i += nt) {
            const unsigned long long c = buf[i];
            const int bin = static_cast<int>(((c >> 32) * scale) >> 32);
            if (bin < B) sel[atomicAdd(&s_nsel, 1)] = c;
            else if (bin == B) tmp[atomicAdd(&s_ntmp, 1)] = c;
        }
        __syncthreads();
        const int ntmp = s_ntmp, need = static_cast<int>(k) - cumB;
        for (int i = tid; i < ntmp; i += nt) {
            const unsigned long long c = tmp[i];
            int r = 0;
            for (int u = 0; u < ntmp; ++u) r += tmp[u] < c;
            if (r < need) sel[cumB + r] = c;
        }
        __syncthreads();
    } else {
        for (int i = tid; i < m; i += nt) sel[i] = buf[i];
        __syncthreads();
    }
    const int cnt = m < static_cast<int>(k) ? m : static_cast<int>(k);
    if (!sort_result) return cnt;
    int sz = 32;
    while (sz < cnt) sz <<= 1;
    for (int i = cnt + tid; i < sz; i += nt) sel[i] = kU64Max;
    __syncthreads();
    if (sz <= 256) {  // one warp, no block barriers
        if (warp == 0) warp_bitonic_sort(sel, sz);
        __syncthreads();
    } else {
        block_bitonic_sort(sel, sz);
    }
    return cnt;
}

__device__ inline int select_sorted_topk(const unsigned long long* buf, int m, uint32_t k, unsigned long long* sel,
                                         unsigned long long* tmp, int tmp_cap, uint32_t* hist, int nbins,
                                         uint32_t maxd) {
    return select_topk(buf, m, k, sel, tmp, tmp_cap, hist, nbins, maxd, true);
}

// K8c: exact top-k of the CTA lists (multi-CTA scan) in one CTA, optionally fused with the
// refine (K9).  ws->overflow = 2 when the candidates do not fit: the host then runs k_knn_merge
// + k_refine instead (identical result).
constexpr int kSelThreads = 1024;
constexpr int kSelCap = 16384;
constexpr int kSelBins = 2048;
constexpr int kSelBinCap = 1024;

struct gather_result {
    int m;
    uint32_t maxd, total;
};

__device__ gather_result gather_lists(qws* ws, uint32_t k, int G, const uint32_t* __restrict__ cand_cnt,
                                      const unsigned long long* __restrict__ cand, unsigned long long* buf, int cap,
                                      uint32_t* s_pref) {
    __shared__ uint32_t s_warp[32];
    __shared__ int s_cnt;
    __shared__ uint32_t s_maxd;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nt = blockDim.x, nw = nt >> 5;
    uint32_t carry = 0;
    for (int base = 0; base < G; base += nt) {
        const int i = base + tid;
        const uint32_t c = i < G ? cand_cnt[i] : 0;
        uint32_t x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_warp[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint32_t t = lane < nw ? s_warp[lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
                if (lane >= o) t += y;
            }
            s_warp[lane] = t;
        }
        __syncthreads();
        if (i < G) s_pref[i] = carry + (warp ? s_warp[warp - 1] : 0) + x - c;
        carry += s_warp[nw - 1];
        __syncthreads();
    }
    if (tid == 0) {
        s_pref[G] = carry;
        s_cnt = 0;
        s_maxd = 0;
    }
    __syncthreads();
    const uint32_t total = s_pref[G];
    const unsigned long long bound = *reinterpret_cast<volatile unsigned long long*>(&ws->bound);
    for (uint32_t f = tid; f < total; f += nt) {
        int lo = 0, hi = G;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (s_pref[mid] <= f) lo = mid;
            else hi = mid;
        }
        if (f - s_pref[lo] >= k) continue;  // defensive: a list never exceeds k entries
        const unsigned long long c = cand[static_cast<size_t>(lo) * k + (f - s_pref[lo])];
        if (c <= bound) {
            const int slot = atomicAdd(&s_cnt, 1);
            if (slot < cap) buf[slot] = c;
            atomicMax(&s_maxd, static_cast<uint32_t>(c >> 32));
        }
    }
    __syncthreads();
    gather_result r;
    r.m = s_cnt;
    r.maxd = s_maxd;
    r.total = total;
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kSelThreads) k_knn_select(qws* ws, uint32_t k, int G,
                                                            const uint32_t* __restrict__ cand_cnt,
                                                            const unsigned long long* __restrict__ cand,
                                                            unsigned long long* __restrict__ out,
                                                            const uint8_t* __restrict__ img, int w, int C, int K,
                                                            const uint8_t* __restrict__ target, int norm) {
    extern __shared__ unsigned long long s_dyn[];
    unsigned long long* buf = s_dyn;                         // kSelCap
    unsigned long long* sel = buf + kSelCap;                 // 2048 (k <= 2048)
    unsigned long long* tmp = sel + 2048;                    // kSelBinCap
    uint32_t* hist = reinterpret_cast<uint32_t*>(tmp + kSelBinCap);  // kSelBins (+1)
    __shared__ uint32_t s_pref[1025];
    const gather_result gr = gather_lists(ws, k, G, cand_cnt, cand, buf, kSelCap, s_pref);
    const int m = gr.m;
    const uint32_t maxd = gr.maxd, total = gr.total;
    int cnt = m > kSelCap ? -1 : select_sorted_topk(buf, m, k, sel, tmp, kSelBinCap, hist, kSelBins, maxd);
    if (cnt < 0) {
        if (threadIdx.x == 0) ws->overflow = 2;
        return;
    }
    for (int i = threadIdx.x; i < cnt; i += kSelThreads) out[i] = sel[i];
    if (threadIdx.x == 0) {
        ws->count = static_cast<uint32_t>(cnt);
        ws->dbg_total = total;
        ws->dbg_m = static_cast<uint32_t>(m);
        ws->overflow = 0;
    }
    if (target != nullptr) {
        __syncthreads();
        refine_list(img, w, C, K, target, sel, cnt, norm, reinterpret_cast<uint8_t*>(buf), ws);
    }
}

// K10: exhaustive masked-cost scan over the dictionary (brute_force_best)
__global__ void __launch_bounds__(256) k_brute(const uint8_t* __restrict__ img, int w, int C, int K,
                                               const uint32_t* __restrict__ dict, uint64_t n,
                                               const uint8_t* __restrict__ target, int norm,
                                               unsigned long long* __restrict__ best) {
    // shared: the known target values in known-local order (known_locals_of, engine.cpp:16-22)
    // and each value's byte offset from the patch origin, so the scan loop is two broadcast loads,
    // one image byte and one multiply-add per value
    extern __shared__ uint8_t s_t[];
    __shared__ int s_nv;
    __shared__ unsigned long long s_best;
    const int KK = K * K;
    int* s_off = reinterpret_cast<int*>(s_t + ((KK * C + 3) & ~3));
    if (threadIdx.x < 32) {  // warp 0: ballot-compacted known locals, ascending
        int cnt = 0;
        for (int base = 0; base < KK; base += 32) {
            const int l = base + threadIdx.x;
            const bool kn = l < KK && target[KK * C + l] != 0;
            const unsigned m = __ballot_sync(0xffffffffu, kn);
            if (kn) {
                const int slot = cnt + __popc(m & ((1u << threadIdx.x) - 1u));
                const int ly = l / K, lx = l - ly * K;
                for (int c = 0; c < C; ++c) {
                    s_t[slot * C + c] = target[l * C + c];
                    s_off[slot * C + c] = (ly * w + lx) * C + c;
                }
            }
            cnt += __popc(m);
        }
        if (threadIdx.x == 0) {
            s_nv = cnt * C;
            s_best = kU64Max;
        }
    }
    __syncthreads();
    const int nv = s_nv;
    unsigned long long mine = kU64Max;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint32_t key = dict[i];
        const uint8_t* base = img + (static_cast<size_t>(key >> 16) * w + (key & 0xffffu)) * C;
        uint32_t acc = 0;
        if (norm == 0) {
#pragma unroll 4
            for (int v = 0; v < nv; ++v) {
                const int d = static_cast<int>(s_t[v]) - static_cast<int>(__ldg(base + s_off[v]));
                acc += static_cast<uint32_t>(d * d);
            }
        } else {
#pragma unroll 4
            for (int v = 0; v < nv; ++v) {
                const int d = static_cast<int>(s_t[v]) - static_cast<int>(__ldg(base + s_off[v]));
                acc += static_cast<uint32_t>(d < 0 ? -d : d);
            }
        }
        const unsigned long long c = pack_candidate(acc, key);
        mine = c < mine ? c : mine;
    }
    mine = warp_min(mine);
    if ((threadIdx.x & 31) == 0) atomicMin(&s_best, mine);
    __syncthreads();
    if (threadIdx.x == 0) atomicMin(best, s_best);
}

// The exhaustive scan for gray images (C == 1), four dictionary entries per thread: when the four
// keys are consecutive columns of one row (the common case: the dictionary is every fully known
// window in row-major order) one unaligned 4-byte load holds a known pixel of all four patches,
// and the four costs are accumulated byte-wise (__vabsdiffu4, then __dp4a per byte lane).  Other
// quads fall back to one patch at a time.  Same (cost, key) minimum as k_brute.
__global__ void __launch_bounds__(256) k_brute4(const uint8_t* __restrict__ img, int w, int K,
                                                const uint32_t* __restrict__ dict, uint64_t n,
                                                const uint8_t* __restrict__ target, int norm,
                                                unsigned long long* __restrict__ best) {
    // shared: the known target values replicated x4, and their byte offsets from the patch origin
    extern __shared__ uint32_t s_t4[];
    __shared__ int s_nv;
    __shared__ unsigned long long s_best;
    const int KK = K * K;
    int* s_off = reinterpret_cast<int*>(s_t4 + KK);
    if (threadIdx.x < 32) {
        int cnt = 0;
        for (int base = 0; base < KK; base += 32) {
            const int l = base + threadIdx.x;
            const bool kn = l < KK && target[KK + l] != 0;
            const unsigned m = __ballot_sync(0xffffffffu, kn);
            if (kn) {
                const int slot = cnt + __popc(m & ((1u << threadIdx.x) - 1u));
                const int ly = l / K, lx = l - ly * K;
                s_t4[slot] = static_cast<uint32_t>(target[l]) * 0x01010101u;
                s_off[slot] = ly * w + lx;
            }
            cnt += __popc(m);
        }
        if (threadIdx.x == 0) {
            s_nv = cnt;
            s_best = kU64Max;
        }
    }
    __syncthreads();
    const int nv = s_nv;
    unsigned long long mine = kU64Max;
    const uint64_t nq = (n + 3) / 4;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t qd = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; qd < nq; qd += stride) {
        const uint64_t i0 = 4 * qd;
        uint32_t key[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) key[u] = i0 + u < n ? __ldg(dict + i0 + u) : 0xffffffffu;
        if (i0 + 3 < n && key[3] == key[0] + 3u) {
            const uint32_t a0 = (key[0] >> 16) * static_cast<uint32_t>(w) + (key[0] & 0xffffu);
            uint32_t acc[4] = {0u, 0u, 0u, 0u};
#pragma unroll 4
            for (int v = 0; v < nv; ++v) {
                const uint32_t a = a0 + static_cast<uint32_t>(s_off[v]);
                const uint32_t* wp = reinterpret_cast<const uint32_t*>(img + (a & ~3u));
                const uint32_t s4 = __funnelshift_r(__ldg(wp), __ldg(wp + 1), (a & 3u) * 8u);
                const uint32_t d = __vabsdiffu4(s4, s_t4[v]);
                if (norm == 0) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) acc[u] = __dp4a(d & (0xffu << (8 * u)), d, acc[u]);
                } else {
#pragma unroll
                    for (int u = 0; u < 4; ++u) acc[u] = __dp4a(d & (0xffu << (8 * u)), 0x01010101u, acc[u]);
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const unsigned long long c = pack_candidate(acc[u], key[u]);
                mine = c < mine ? c : mine;
            }
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (i0 + u >= n) continue;
                const uint8_t* base = img + (static_cast<size_t>(key[u] >> 16) * w + (key[u] & 0xffffu));
                uint32_t acc = 0;
                for (int v = 0; v < nv; ++v) {
                    const int dd = static_cast<int>(s_t4[v] & 0xffu) - static_cast<int>(__ldg(base + s_off[v]));
                    acc += norm == 0 ? static_cast<uint32_t>(dd * dd) : static_cast<uint32_t>(dd < 0 ? -dd : dd);
                }
                const unsigned long long c = pack_candidate(acc, key[u]);
                mine = c < mine ? c : mine;
            }
        }
    }
    mine = warp_min(mine);
    if ((threadIdx.x & 31) == 0) atomicMin(&s_best, mine);
    __syncthreads();
    if (threadIdx.x == 0) atomicMin(best, s_best);
}

// The exhaustive scan for gray images, eight dictionary entries per thread.  When the eight keys
// are consecutive columns of one row, three aligned word loads + two funnel shifts per known value
// give that pixel for all eight patches; the byte differences (__vabsdiffu4) of four values are
// transposed with byte permutes so that one __dp4a adds four values of one patch (8 PRMT + 8 DP4A
// per 4 values x 8 patches, instead of a mask + __dp4a per patch and value).  The known values and
// their offsets are read as 16-byte vectors; a tail of nv % 4 values and non-consecutive octets
// take the per-lane path.  Same (cost, key) minimum as k_brute.
__device__ __forceinline__ void transpose4x4_bytes(uint32_t d0, uint32_t d1, uint32_t d2, uint32_t d3, uint32_t (&t)[4]) {
    const uint32_t a = __byte_perm(d0, d1, 0x5140), b = __byte_perm(d0, d1, 0x7362);
    const uint32_t c = __byte_perm(d2, d3, 0x5140), e = __byte_perm(d2, d3, 0x7362);
    t[0] = __byte_perm(a, c, 0x5410);
    t[1] = __byte_perm(a, c, 0x7632);
    t[2] = __byte_perm(b, e, 0x5410);
    t[3] = __byte_perm(b, e, 0x7632);
}

__global__ void __launch_bounds__(256) k_brute8(const uint8_t* __restrict__ img, int w, int K,
                                                const uint32_t* __restrict__ dict, uint64_t n,
                                                const uint8_t* __restrict__ target, int norm,
                                                unsigned long long* __restrict__ best) {
    // shared: the known target values replicated x4 and their byte offsets from the patch origin,
    // padded to a multiple of 4 entries (16-byte aligned arrays)
    extern __shared__ __align__(16) uint32_t s_t4[];
    __shared__ int s_nv;
    __shared__ unsigned long long s_best;
    const int KK = K * K, KP = (KK + 3) & ~3;
    int* s_off = reinterpret_cast<int*>(s_t4 + KP);
    if (threadIdx.x < 32) {
        int cnt = 0;
        for (int base = 0; base < KK; base += 32) {
            const int l = base + threadIdx.x;
            const bool kn = l < KK && target[KK + l] != 0;
            const unsigned m = __ballot_sync(0xffffffffu, kn);
            if (kn) {
                const int slot = cnt + __popc(m & ((1u << threadIdx.x) - 1u));
                const int ly = l / K, lx = l - ly * K;
                s_t4[slot] = static_cast<uint32_t>(target[l]) * 0x01010101u;
                s_off[slot] = ly * w + lx;
            }
            cnt += __popc(m);
        }
        if (threadIdx.x == 0) {
            s_nv = cnt;
            s_best = kU64Max;
        }
    }
    __syncthreads();
    const int nv = s_nv, nv4 = nv & ~3;
    const bool l2 = norm == 0;
    unsigned long long mine = kU64Max;
    const uint64_t no = (n + 7) / 8;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t oc = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; oc < no; oc += stride) {
        const uint64_t i0 = 8 * oc;
        uint32_t key[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) key[u] = i0 + u < n ? __ldg(dict + i0 + u) : 0xffffffffu;
        uint32_t acc[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] = 0u;
        if (i0 + 7 < n && key[7] == key[0] + 7u) {
            const uint32_t a0 = (key[0] >> 16) * static_cast<uint32_t>(w) + (key[0] & 0xffffu);
            auto pix8 = [&](int off, uint32_t& lo, uint32_t& hi) {
                const uint32_t a = a0 + static_cast<uint32_t>(off);
                const uint32_t* wp = reinterpret_cast<const uint32_t*>(img + (a & ~3u));
                const uint32_t x0 = __ldg(wp), x1 = __ldg(wp + 1), x2 = __ldg(wp + 2), sh = (a & 3u) * 8u;
                lo = __funnelshift_r(x0, x1, sh);
                hi = __funnelshift_r(x1, x2, sh);
            };
            for (int v = 0; v < nv4; v += 4) {
                const uint4 t4 = *reinterpret_cast<const uint4*>(s_t4 + v);
                const int4 o4 = *reinterpret_cast<const int4*>(s_off + v);
                uint32_t lo[4], hi[4];
                pix8(o4.x, lo[0], hi[0]);
                pix8(o4.y, lo[1], hi[1]);
                pix8(o4.z, lo[2], hi[2]);
                pix8(o4.w, lo[3], hi[3]);
                const uint32_t tv[4] = {t4.x, t4.y, t4.z, t4.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    lo[u] = __vabsdiffu4(lo[u], tv[u]);
                    hi[u] = __vabsdiffu4(hi[u], tv[u]);
                }
                uint32_t tl[4], th[4];
                transpose4x4_bytes(lo[0], lo[1], lo[2], lo[3], tl);
                transpose4x4_bytes(hi[0], hi[1], hi[2], hi[3], th);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    acc[u] = __dp4a(tl[u], l2 ? tl[u] : 0x01010101u, acc[u]);
                    acc[4 + u] = __dp4a(th[u], l2 ? th[u] : 0x01010101u, acc[4 + u]);
                }
            }
            for (int v = nv4; v < nv; ++v) {
                uint32_t lo, hi;
                pix8(s_off[v], lo, hi);
                const uint32_t dl = __vabsdiffu4(lo, s_t4[v]), dh = __vabsdiffu4(hi, s_t4[v]);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t ml = dl & (0xffu << (8 * u)), mh = dh & (0xffu << (8 * u));
                    acc[u] = __dp4a(ml, l2 ? dl : 0x01010101u, acc[u]);
                    acc[4 + u] = __dp4a(mh, l2 ? dh : 0x01010101u, acc[4 + u]);
                }
            }
        } else {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (i0 + u >= n) continue;
                const uint8_t* base = img + (static_cast<size_t>(key[u] >> 16) * w + (key[u] & 0xffffu));
                uint32_t a = 0;
                for (int v = 0; v < nv; ++v) {
                    const int dd = static_cast<int>(s_t4[v] & 0xffu) - static_cast<int>(__ldg(base + s_off[v]));
                    a += l2 ? static_cast<uint32_t>(dd * dd) : static_cast<uint32_t>(dd < 0 ? -dd : dd);
                }
                acc[u] = a;
            }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (i0 + u < n) {
                const unsigned long long c = pack_candidate(acc[u], key[u]);
                mine = c < mine ? c : mine;
            }
        }
    }
    mine = warp_min(mine);
    if ((threadIdx.x & 31) == 0) atomicMin(&s_best, mine);
    __syncthreads();
    if (threadIdx.x == 0) atomicMin(best, s_best);
}

// exhaustive path for k > kMaxScanK: pack every entry, radix-sort the u64 packed values
__global__ void __launch_bounds__(256) k_pack_all(views8 V, const qws* ws, int norm, uint32_t* __restrict__ lo,
                                                  uint32_t* __restrict__ hi) {
    const index_view v = V.v[ws->lid & 7];
    uint32_t q4[8];
#pragma unroll
    for (int p = 0; p < 8; ++p) q4[p] = ws->q4[p];
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < v.n; i += stride) {
        lo[i] = v.keys[i];
        hi[i] = entry_dist(v, i, q4, norm);
    }
}

__global__ void k_gather_topk(const uint32_t* __restrict__ lo, const uint32_t* __restrict__ hi, uint32_t cnt,
                              qws* ws, unsigned long long* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < cnt) out[i] = (static_cast<unsigned long long>(hi[i]) << 32) | lo[i];
    if (i == 0) ws->count = cnt;
}

// ===================================================================== one-launch query (fill loop)
// query_best_patch in ONE launch over G CTAs: every CTA stages the target and recomputes
// select_index + make_query (a few microseconds, no host round trip); each CTA owns a contiguous
// Morton range of blocks, seeds a local bound from its best block by bbox lower bound, shares it
// through atomicMin on ws->bound, and keeps its exact local top-k; the last CTA to finish
// (threadfence + ticket) selects the global top-k, refines it and resets the ticket/bound.
// masked costs (proj/src/engine.cpp:48-76) of list[0..cnt) into s_cost, CTA-cooperative: all
// (candidate, known pixel) pairs in parallel, four image loads in flight per thread
__device__ void cost_candidates(const uint8_t* __restrict__ img, int w, int C, int K, const uint8_t* s_tv,
                                const uint16_t* s_loc, int nloc, const unsigned long long* list, int cnt, int norm,
                                uint32_t* s_cost) {
    for (int e = threadIdx.x; e < cnt; e += blockDim.x) s_cost[e] = 0;
    __syncthreads();
    const int pairs = cnt * nloc;
    const int stride = blockDim.x;
    for (int p0 = threadIdx.x; p0 < pairs; p0 += 4 * stride) {
        uint8_t sv[4][3];
        int pe[4], pl[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int pi = p0 + u * stride;
            pe[u] = -1;
            if (pi < pairs) {
                const int e = pi / nloc, li = pi - e * nloc;
                const uint32_t key = static_cast<uint32_t>(list[e] & 0xffffffffu);
                const int l = s_loc[li];
                const uint8_t* src = img + (static_cast<size_t>((key >> 16) + l / K) * w + (key & 0xffff) + l % K) * C;
                pe[u] = e;
                pl[u] = l;
#pragma unroll
                for (int c = 0; c < 3; ++c) sv[u][c] = c < C ? __ldg(src + c) : 0;
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (pe[u] < 0) continue;
            const uint8_t* t = s_tv + pl[u] * C;
            uint32_t acc = 0;
            for (int c = 0; c < C; ++c) {
                const int d = static_cast<int>(t[c]) - static_cast<int>(sv[u][c]);
                acc += norm == 0 ? static_cast<uint32_t>(d * d) : static_cast<uint32_t>(d < 0 ? -d : d);
            }
            atomicAdd(&s_cost[pe[u]], acc);
        }
    }
    __syncthreads();
}

// k-th smallest of m unique packed values in buf (kU64Max when m <= k): distance histogram ->
// boundary bin -> exact rank inside it.  Returns kU64Max - 1 on a degenerate boundary bin
// (more than tmp_cap values), which the caller treats as an overflow.
__device__ unsigned long long kth_packed(const unsigned long long* buf, int m, uint32_t k, unsigned long long* tmp,
                                         int tmp_cap, uint32_t* hist, int nbins, uint32_t maxd) {
    __shared__ int s_ntmp, s_B, s_cumB;
    __shared__ unsigned long long s_T;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nt = blockDim.x;
    if (m <= static_cast<int>(k)) return kU64Max;
    for (int i = tid; i <= nbins; i += nt) hist[i] = 0;
    if (tid == 0) {
        s_ntmp = 0;
        s_B = -1;
        s_T = kU64Max - 1;
    }
    __syncthreads();
    const uint64_t scale = (static_cast<uint64_t>(nbins) << 32) / (static_cast<uint64_t>(maxd) + 1);
    for (int i = tid; i < m; i += nt) {
        const uint32_t bin = static_cast<uint32_t>(((buf[i] >> 32) * scale) >> 32);
        atomicAdd(&hist[bin < static_cast<uint32_t>(nbins) ? bin : nbins - 1], 1u);
    }
    __syncthreads();
    if (warp == 0) {
        uint32_t run = 0;
        for (int base = 0; base < nbins; base += 32) {
            uint32_t x = base + lane < nbins ? hist[base + lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            const unsigned hit = __ballot_sync(0xffffffffu, run + x >= k);
            if (hit) {
                const int src = __ffs(hit) - 1;
                const uint32_t incl = __shfl_sync(0xffffffffu, x, src);
                if (lane == 0) {
                    s_B = base + src;
                    s_cumB = static_cast<int>(run + incl - hist[base + src]);
                }
                break;
            }
            run += __shfl_sync(0xffffffffu, x, 31);
        }
    }
    __syncthreads();
    const int B = s_B, cumB = s_cumB;
    if (B < 0 || static_cast<int>(hist[B]) > tmp_cap) return kU64Max - 1;
    for (int i = tid; i < m; i += nt) {
        const unsigned long long c = buf[i];
        const uint32_t bin0 = static_cast<uint32_t>(((c >> 32) * scale) >> 32);
        const int bin = static_cast<int>(bin0 < static_cast<uint32_t>(nbins) ? bin0 : nbins - 1);
        if (bin == B) tmp[atomicAdd(&s_ntmp, 1)] = c;
    }
    __syncthreads();
    const int ntmp = s_ntmp, need = static_cast<int>(k) - cumB;  // need-th smallest (1-based) in tmp
    for (int i = tid; i < ntmp; i += nt) {
        const unsigned long long c = tmp[i];
        int r = 0;
        for (int u = 0; u < ntmp; ++u) r += tmp[u] < c;
        if (r == need - 1) s_T = c;
    }
    __syncthreads();
    return s_T;
}

constexpr int kOneThreads = 256;
constexpr int kOneCap = 4096;
constexpr uint32_t kOneMaxK = 1024;
constexpr int kOneBins = 2048;
constexpr int kOneBinCap = 1024;

template <int P>
__global__ void __launch_bounds__(kOneThreads) k_query_one(mi_view mv, const uint8_t* __restrict__ img, int w,
                                                          const uint8_t* __restrict__ target, qws* ws, uint32_t k,
                                                          int norm, uint32_t* __restrict__ cand_cnt,
                                                          unsigned long long* __restrict__ cand,
                                                          uint32_t* __restrict__ ccost,
                                                          unsigned long long* __restrict__ out, qres* res,
                                                          uint32_t seq, int want_list) {
    // kOneCap | sel (kOneMaxK) | tmp | hist | costs (kOneCap u32) | xc | comp | target | locals
    extern __shared__ unsigned long long s_buf[];
    unsigned long long* sel = s_buf + kOneCap;
    unsigned long long* tmp = sel + kOneMaxK;
    uint32_t* hist = reinterpret_cast<uint32_t*>(tmp + kOneBinCap);
    uint32_t* s_cost = hist + kOneBins + 2;
    const int KK = mv.K * mv.K, mc = mv.m * mv.C, C = mv.C, D = mv.D;
    double* s_xc = reinterpret_cast<double*>(s_cost + kOneCap);
    double* s_comp = s_xc + mc;
    uint8_t* s_t = reinterpret_cast<uint8_t*>(s_comp + static_cast<size_t>(mc) * D);
    uint16_t* s_loc = reinterpret_cast<uint16_t*>(s_t + ((KK * C + KK + 1) & ~1));
    __shared__ int s_nloc;
    __shared__ int s_ov[8];
    __shared__ int s_lid, s_cnt, s_last;
    __shared__ uint8_t s_q[32];
    __shared__ unsigned long long s_bound, s_wmin[8];
    __shared__ uint32_t s_pref[1025];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tbytes = KK * C + KK;
    ZI_TPHASE(0)
    for (int i = tid; i < tbytes; i += kOneThreads) s_t[i] = target[i];
    if (tid < 32) s_q[tid] = 0;
    if (tid == 0) s_cnt = 0;
    __syncthreads();
    if (warp == 0) {  // known locals, ascending (known_locals_of, engine.cpp:16-22), via ballots
        int c = 0;
        for (int base = 0; base < KK; base += 32) {
            const bool kn = base + lane < KK && s_t[KK * C + base + lane] != 0;
            const unsigned mk = __ballot_sync(0xffffffffu, kn);
            if (kn) s_loc[c + __popc(mk & ((1u << lane) - 1u))] = static_cast<uint16_t>(base + lane);
            c += __popc(mk);
        }
        if (lane == 0) s_nloc = c;
    }
    const uint8_t* tv = s_t;
    const uint8_t* tk = s_t + KK * C;
    {  // select_index (engine.cpp:162-176)
        int ov = 0;
        for (int p = lane; p < mv.m; p += 32) ov += tk[mv.local[warp * mv.m + p]] != 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ov += __shfl_xor_sync(0xffffffffu, ov, o);
        if (lane == 0) s_ov[warp] = ov;
    }
    __syncthreads();
    if (tid == 0) {
        int best = 0, bid = 0;
        for (int l = 0; l < 8; ++l)
            if (s_ov[l] > best) {
                best = s_ov[l];
                bid = l;
            }
        s_lid = bid;
    }
    __syncthreads();
    const int lid = s_lid;
    {  // make_query (builder.cpp:110-127), canonical fp64 order
        const double* mean = mv.mean + static_cast<size_t>(lid) * mc;
        const int32_t* loc = mv.local + lid * mv.m;
        for (int j = tid; j < mc; j += kOneThreads) {
            const int l = loc[j / C];
            const double mj = mean[j];
            const double x = tk[l] ? static_cast<double>(tv[l * C + j % C]) : mj;
            s_xc[j] = __dsub_rn(x, mj);
        }
        const double* comp = mv.comp + static_cast<size_t>(lid) * mc * D;
        for (int i = tid; i < mc * D; i += kOneThreads) s_comp[i] = comp[i];
    }
    __syncthreads();
    if (tid < D) {
        double y = 0.0;
        for (int j = 0; j < mc; ++j) y = __fma_rn(s_comp[j * D + tid], s_xc[j], y);
        const unsigned long long* mm = mv.minmax + static_cast<size_t>(lid) * 2 * D;
        s_q[tid] = quantize_rn(ordered_to_double_hd(mm[tid]), ordered_to_double_hd(mm[D + tid]), y);
    }
    __syncthreads();
    uint32_t q4[8];
#pragma unroll
    for (int p = 0; p < 8; ++p)
        q4[p] = static_cast<uint32_t>(s_q[4 * p]) | (static_cast<uint32_t>(s_q[4 * p + 1]) << 8) |
                (static_cast<uint32_t>(s_q[4 * p + 2]) << 16) | (static_cast<uint32_t>(s_q[4 * p + 3]) << 24);
    ZI_TPHASE(1)
    const index_view v = mv.idx[lid];
    const uint64_t nblk = v.nblk, G = gridDim.x;
    const uint64_t per = (nblk + G - 1) / G;
    const uint64_t bb0 = blockIdx.x * per < nblk ? blockIdx.x * per : nblk;
    const uint64_t bb1 = bb0 + per < nblk ? bb0 + per : nblk;
    // local seed: the range's block with the smallest bbox lower bound
    {
        unsigned long long mine = kU64Max;
        for (uint64_t b = bb0 + tid; b < bb1; b += kOneThreads) {
            uint32_t lb = 0;
#pragma unroll
            for (int p = 0; p < P; ++p)
                lb = gap4(q4[p], v.bmin[static_cast<size_t>(p) * nblk + b], v.bmax[static_cast<size_t>(p) * nblk + b], norm, lb);
            const unsigned long long c = (static_cast<unsigned long long>(lb) << 32) | b;
            mine = c < mine ? c : mine;
        }
        mine = warp_min(mine);
        if (lane == 0) s_wmin[warp] = mine;
    }
    __syncthreads();
    if (warp == 0) {
        unsigned long long bm = lane < 8 ? s_wmin[lane] : kU64Max;
        bm = warp_min(bm);
        unsigned long long c[8];
        if (bm != kU64Max) {
            score_block<P>(v, bm & 0xffffffffull, q4, norm, c);
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) c[e] = kU64Max;
        }
        // k-th smallest distance of these 256 entries by radix descent (no sort): at least k
        // entries have dist <= T, so (T<<32 | 0xffffffff) is a valid bound
        int valid = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) valid += c[e] != kU64Max;
        valid = __reduce_add_sync(0xffffffffu, valid);
        unsigned long long lbound = kU64Max;
        if (k <= 256 && valid >= static_cast<int>(k)) {
            uint32_t T = 0;
            int need = static_cast<int>(k);
            for (int bit = 31; bit >= 0; --bit) {
                int cnt = 0;
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    cnt += c[e] != kU64Max && (static_cast<uint32_t>(c[e] >> 32) >> bit) == (T >> bit);
                cnt = __reduce_add_sync(0xffffffffu, cnt);
                if (cnt < need) {
                    need -= cnt;
                    T |= 1u << bit;
                }
            }
            lbound = (static_cast<unsigned long long>(T) << 32) | 0xffffffffull;
        }
        if (lane == 0) {
            s_bound = lbound;
            if (lbound != kU64Max) atomicMin(&ws->bound, lbound);
        }
    }
    __syncthreads();
    ZI_TPHASE(2)
    // scan the range: 8 blocks per round, one per warp
    const uint64_t rounds = (bb1 - bb0 + 7) / 8;
    for (uint64_t r = 0; r < rounds; ++r) {
        const uint64_t b = bb0 + r * 8 + warp;
        unsigned long long bound = s_bound;
        const unsigned long long g = *reinterpret_cast<volatile unsigned long long*>(&ws->bound);
        bound = g < bound ? g : bound;
        if (b < bb1) {
            uint32_t lb = 0;
#pragma unroll
            for (int p = 0; p < P; ++p)
                lb = gap4(q4[p], v.bmin[static_cast<size_t>(p) * nblk + b], v.bmax[static_cast<size_t>(p) * nblk + b], norm, lb);
            if ((static_cast<unsigned long long>(lb) << 32) <= bound) {
                unsigned long long c[8];
                score_block<P>(v, b, q4, norm, c);
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    if (c[e] != kU64Max && c[e] <= bound) s_buf[atomicAdd(&s_cnt, 1)] = c[e];
            }
        }
        __syncthreads();
        if (s_cnt > kOneCap - 8 * 256) compact_buffer(s_buf, &s_cnt, &s_bound, k, ws, true);
        __syncthreads();
    }
    ZI_TPHASE(3)
    {  // exact local top-k (unsorted) by histogram selection, straight into the CTA's slot
        const int m0 = s_cnt;
        uint32_t mx = 0;
        for (int t = tid; t < m0; t += kOneThreads) mx = max(mx, static_cast<uint32_t>(s_buf[t] >> 32));
        mx = __reduce_max_sync(0xffffffffu, mx);
        __shared__ uint32_t s_mx;
        if (tid == 0) s_mx = 0;
        __syncthreads();
        if (lane == 0) atomicMax(&s_mx, mx);
        __syncthreads();
        int cnt = select_topk(s_buf, m0, k, sel, tmp, kOneBinCap, hist, 256, s_mx, false);
        if (cnt < 0) {  // degenerate boundary bin: exact sort-based compaction instead
            compact_buffer(s_buf, &s_cnt, &s_bound, k, ws, true);
            cnt = s_cnt;
            for (int t = tid; t < cnt; t += kOneThreads) sel[t] = s_buf[t];
            __syncthreads();
        }
        __shared__ unsigned long long s_kth, s_gb;
        __shared__ int s_keep;
        if (tid == 0) {
            s_kth = 0;
            s_keep = 0;
        }
        __syncthreads();
        // publish this CTA's k-th first (a valid global bound when it holds k candidates), then
        // keep only the local winners that can still make the global top-k
        unsigned long long kth = 0;
        for (int t = tid; t < cnt; t += kOneThreads) kth = sel[t] > kth ? sel[t] : kth;
        if (cnt >= static_cast<int>(k)) {
            atomicMax(&s_kth, kth);
            __syncthreads();
            if (tid == 0) atomicMin(&ws->bound, s_kth);
        }
        __syncthreads();
        if (tid == 0) s_gb = *reinterpret_cast<volatile unsigned long long*>(&ws->bound);
        __syncthreads();
        const unsigned long long gb = s_gb;
        for (int t = tid; t < cnt; t += kOneThreads)
            if (sel[t] <= gb) tmp[atomicAdd(&s_keep, 1)] = sel[t];
        __syncthreads();
        const int keep = s_keep;
        // refine ahead of the merge: every CTA costs its own surviving winners (in parallel across
        // CTAs), so the last CTA only selects the global k and takes the min over their costs
        cost_candidates(img, w, C, mv.K, s_t, s_loc, s_nloc, tmp, keep, norm, s_cost);
        __shared__ uint32_t s_gbase;
        if (tid == 0) s_gbase = atomicAdd(&ws->gcount, static_cast<uint32_t>(keep));
        __syncthreads();
        for (int t = tid; t < keep; t += kOneThreads) {
            cand[s_gbase + t] = tmp[t];
            ccost[s_gbase + t] = s_cost[t];
        }
    }
    ZI_TPHASE(4)
    // the last CTA merges
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(&ws->done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    ZI_TPHASE(6)
    int m;
    uint32_t maxd, total;
    {  // compact global list -> candidates <= the final bound
        __shared__ int s_m;
        __shared__ uint32_t s_maxd;
        if (tid == 0) {
            s_m = 0;
            s_maxd = 0;
        }
        __syncthreads();
        total = *reinterpret_cast<volatile uint32_t*>(&ws->gcount);
        const unsigned long long bound = *reinterpret_cast<volatile unsigned long long*>(&ws->bound);
        for (uint32_t f = tid; f < total; f += kOneThreads) {
            const unsigned long long c = cand[f];
            if (c <= bound) {
                const int slot = atomicAdd(&s_m, 1);
                if (slot < kOneCap) {
                    s_buf[slot] = c;
                    s_cost[slot] = ccost[f];
                }
                atomicMax(&s_maxd, static_cast<uint32_t>(c >> 32));
            }
        }
        __syncthreads();
        m = s_m;
        maxd = s_maxd;
        (void)s_pref;
    }
    ZI_TPHASE(7)
    // the global k-th packed value; winners = candidates <= it; best = min (cost, key) over them
    const unsigned long long T = m > kOneCap ? kU64Max - 1 : kth_packed(s_buf, m, k, tmp, kOneBinCap, hist, 256, maxd);
    int cnt = T == kU64Max - 1 ? -1 : (m < static_cast<int>(k) ? m : static_cast<int>(k));
    if (cnt >= 0 && want_list) cnt = select_sorted_topk(s_buf, m, k, sel, tmp, kOneBinCap, hist, 256, maxd);
    ZI_TPHASE(8)
    if (tid == 0) {
        ws->lid = static_cast<uint32_t>(lid);
        ws->dbg_total = total;
        ws->dbg_m = static_cast<uint32_t>(m);
        ws->final_bound = ws->bound;
        ws->done = 0;
        ws->gcount = 0;
    }
    if (cnt < 0) {
        if (tid == 0) {
            ws->overflow = 2;
            cand_cnt[0] = total;  // the compact list as ONE list for k_knn_merge
            if (res) {
                res->lid = static_cast<uint32_t>(lid);
                res->overflow = 2;
                __threadfence_system();
                res->seq = seq;
            }
        }
        return;  // host: k_knn_merge + k_refine over the same list
    }
    if (want_list)
        for (int i = tid; i < cnt; i += kOneThreads) out[i] = sel[i];
    {
        __shared__ unsigned long long s_best;
        if (tid == 0) s_best = kU64Max;
        __syncthreads();
        unsigned long long mine = kU64Max;
        for (int i = tid; i < m; i += kOneThreads)
            if (s_buf[i] <= T) {
                const unsigned long long c = pack_candidate(s_cost[i], static_cast<uint32_t>(s_buf[i] & 0xffffffffu));
                mine = c < mine ? c : mine;
            }
        mine = warp_min(mine);
        if (lane == 0) atomicMin(&s_best, mine);
        __syncthreads();
        if (tid == 0) ws->best = s_best;
    }
    ZI_TPHASE(9)
    if (tid == 0) {
        ws->count = static_cast<uint32_t>(cnt);
        ws->overflow = 0;
        ws->bound = kU64Max;  // the workspace is left ready for the next query (no host memsets)
        if (res) {
            res->best = ws->best;
            res->lid = static_cast<uint32_t>(lid);
            res->count = static_cast<uint32_t>(cnt);
            res->overflow = 0;
            __threadfence_system();
            res->seq = seq;
        }
    }
}

// ===================================================================== low-latency fill-loop query
// query_best_patch (engine.cpp:178-213) in ONE launch, tuned for latency (k <= kLatMaxK):
//  * the target (K*K*C values + K*K flags) travels in the kernel parameters: no H2D copy;
//  * every CTA redoes select_index + make_query (a few hundred FMAs);
//  * blocks are dealt round-robin (block b -> CTA b % G), so the dense Morton region around the
//    query is spread over all CTAs instead of landing on one;
//  * each thread computes the bbox lower bounds of its blocks at once; the CTA scores its best
//    block for a local k-th bound (atomicMin into the global bound), compacts the blocks whose
//    bound can still win, and its 16 warps score them independently (no per-block barriers);
//  * the CTA's exact local top-k is costed (refine ahead of the merge) and appended to a global
//    list; the last CTA (ticket) takes the global k-th and the (cost, key) minimum, resets the
//    workspace and publishes the result to mapped host memory.
// Exactness: as k_query_one -- every bound is the k-th packed value of a subset of the index.
constexpr int kLatThreads = 512;
constexpr int kLatWarps = kLatThreads / 32;
constexpr int kLatCap = 8192;  // a power of two: compact_buffer sorts the whole buffer
constexpr uint32_t kLatMaxK = 256;
constexpr int kLatMaxTarget = 1024;
constexpr int kLatBlkRegs = 8;  // bbox bounds per thread (shared memory): nblk <= G * 512 * 8

struct qlat_params {
    mi_view mv;
    const uint8_t* img;
    int w;
    qws* ws;
    uint32_t k;
    int norm;
    unsigned long long* cand;
    uint32_t* ccost;
    unsigned long long* out;
    qres* res;
    uint32_t seq;
    int want_list;
    int tbytes;
    unsigned long long* dbg;  // ZI_DEBUG_QUERY: per-CTA %globaltimer at start and before the ticket
    uint8_t target[kLatMaxTarget];
};

template <int P>
__global__ void __launch_bounds__(kLatThreads, P <= 3 ? 2 : 1) k_query_lat(const __grid_constant__ qlat_params prm) {
    // s_buf kLatCap | sel kLatMaxK | tmp kOneBinCap | hist | costs kLatCap | xc | target | locals;
    // the survivor list (<= kLatThreads * kLatBlkRegs blocks) aliases sel .. costs, which are only
    // used after the scoring
    extern __shared__ unsigned long long s_buf[];
    unsigned long long* sel = s_buf + kLatCap;
    unsigned long long* tmp = sel + kLatMaxK;
    uint32_t* hist = reinterpret_cast<uint32_t*>(tmp + kOneBinCap);
    uint32_t* s_cost = hist + 256 + 2;
    unsigned long long* s_surv = sel;
    static_assert((kLatMaxK + kOneBinCap) * 8 + (258 + kLatCap) * 4 >= kLatThreads * kLatBlkRegs * 8, "survivor list");
    const mi_view& mv = prm.mv;
    const int KK = mv.K * mv.K, mc = mv.m * mv.C, C = mv.C, D = mv.D;
    double* s_xc = reinterpret_cast<double*>(s_cost + kLatCap);
    uint8_t* s_t = reinterpret_cast<uint8_t*>(s_xc + mc);
    uint16_t* s_loc = reinterpret_cast<uint16_t*>(s_t + ((KK * C + KK + 1) & ~1));
    __shared__ int s_nloc, s_lid, s_cnt, s_last, s_nsurv, s_ovf;
    __shared__ int s_ov[8];
    __shared__ uint8_t s_q[32];
    __shared__ unsigned long long s_bound, s_wmin[kLatWarps];
    qws* ws = prm.ws;
    const uint32_t k = prm.k;
    const int norm = prm.norm;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    ZI_TPHASE(0)
    if (prm.dbg && tid == 0) prm.dbg[4 * blockIdx.x] = gtimer();
    for (int i = tid; i < prm.tbytes; i += kLatThreads) s_t[i] = prm.target[i];
    if (tid < 32) s_q[tid] = 0;
    if (tid == 0) {
        s_cnt = 0;
        s_nsurv = 0;
        s_ovf = 0;
    }
    __syncthreads();
    const uint8_t* tv = s_t;
    const uint8_t* tk = s_t + KK * C;
    if (warp == 8) {  // known locals, ascending (known_locals_of, engine.cpp:16-22)
        int c = 0;
        for (int base = 0; base < KK; base += 32) {
            const bool kn = base + lane < KK && tk[base + lane] != 0;
            const unsigned mk = __ballot_sync(0xffffffffu, kn);
            if (kn) s_loc[c + __popc(mk & ((1u << lane) - 1u))] = static_cast<uint16_t>(base + lane);
            c += __popc(mk);
        }
        if (lane == 0) s_nloc = c;
    }
    if (warp < 8) {  // select_index (engine.cpp:162-176)
        int ov = 0;
        for (int p = lane; p < mv.m; p += 32) ov += tk[mv.local[warp * mv.m + p]] != 0;
        ov = __reduce_add_sync(0xffffffffu, ov);
        if (lane == 0) s_ov[warp] = ov;
    }
    __syncthreads();
    if (tid == 0) {
        int best = 0, bid = 0;
        for (int l = 0; l < 8; ++l)
            if (s_ov[l] > best) {
                best = s_ov[l];
                bid = l;
            }
        s_lid = bid;
    }
    __syncthreads();
    const int lid = s_lid;
    // make_query (builder.cpp:110-127): x - mean and the layout's components ([j][d], staged in
    // the candidate buffer, unused until the seed) in shared memory, then the canonical fp64
    // chain per dim
    double* s_comp = reinterpret_cast<double*>(s_buf);
    {
        const double* mean = mv.mean + static_cast<size_t>(lid) * mc;
        const int32_t* loc = mv.local + lid * mv.m;
        for (int j = tid; j < mc; j += kLatThreads) {
            const int l = loc[j / C];
            const double mj = mean[j];
            const double x = tk[l] ? static_cast<double>(tv[l * C + j % C]) : mj;
            s_xc[j] = __dsub_rn(x, mj);
        }
        const double* comp = mv.comp + static_cast<size_t>(lid) * mc * D;
        for (int i = tid; i < mc * D; i += kLatThreads) s_comp[i] = __ldg(comp + i);
    }
    __syncthreads();
    if (tid < D) {
        double y = 0.0;
        int j = 0;
        for (; j + 8 <= mc; j += 8) {
            double cc[8], xx[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                cc[u] = s_comp[(j + u) * D + tid];
                xx[u] = s_xc[j + u];
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) y = __fma_rn(cc[u], xx[u], y);
        }
        for (; j < mc; ++j) y = __fma_rn(s_comp[j * D + tid], s_xc[j], y);
        const unsigned long long* mm = mv.minmax + static_cast<size_t>(lid) * 2 * D;
        s_q[tid] = quantize_rn(ordered_to_double_hd(mm[tid]), ordered_to_double_hd(mm[D + tid]), y);
    }
    __syncthreads();
    uint32_t q4[8];
#pragma unroll
    for (int p = 0; p < 8; ++p)
        q4[p] = static_cast<uint32_t>(s_q[4 * p]) | (static_cast<uint32_t>(s_q[4 * p + 1]) << 8) |
                (static_cast<uint32_t>(s_q[4 * p + 2]) << 16) | (static_cast<uint32_t>(s_q[4 * p + 3]) << 24);
    ZI_TPHASE(1)
    const index_view v = mv.idx[lid];
    const uint64_t nblk = v.nblk, G = gridDim.x, c0 = blockIdx.x;
    // bbox lower bounds of this CTA's blocks b = c0 + G*i, i = tid + kLatThreads*r, kept as packed
    // (lb<<32 | b) in the upper half of s_buf (the candidates start at its bottom)
    unsigned long long* s_lbb = s_buf + (kLatCap - kLatThreads * kLatBlkRegs);
    unsigned long long mine = kU64Max;
#pragma unroll 4
    for (int r = 0; r < kLatBlkRegs; ++r) {
        const uint64_t b = c0 + G * (static_cast<uint64_t>(tid) + static_cast<uint64_t>(kLatThreads) * r);
        unsigned long long e = kU64Max;
        if (b < nblk) {
            uint32_t lb = 0;
#pragma unroll
            for (int p = 0; p < P; ++p)
                lb = gap4(q4[p], __ldg(v.bmin + static_cast<size_t>(p) * nblk + b),
                          __ldg(v.bmax + static_cast<size_t>(p) * nblk + b), norm, lb);
            e = (static_cast<unsigned long long>(lb) << 32) | b;
            mine = e < mine ? e : mine;
        }
        s_lbb[tid + kLatThreads * r] = e;
    }
    mine = warp_min(mine);
    if (lane == 0) s_wmin[warp] = mine;
    __syncthreads();
    const unsigned long long seed = [&] {
        unsigned long long m = kU64Max;
#pragma unroll
        for (int w = 0; w < kLatWarps; ++w) m = s_wmin[w] < m ? s_wmin[w] : m;
        return m;
    }();
    if (warp == 0) {  // score the best block: its k-th distance bounds the answer
        unsigned long long c[8];
        if (seed != kU64Max) {
            score_block<P>(v, seed & 0xffffffffull, q4, norm, c);
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) c[e] = kU64Max;
        }
        int valid = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) valid += c[e] != kU64Max;
        valid = __reduce_add_sync(0xffffffffu, valid);
        unsigned long long lbound = kU64Max;
        if (valid >= static_cast<int>(k)) {  // k-th smallest distance by radix descent
            uint32_t T = 0;
            int need = static_cast<int>(k);
            for (int bit = 31; bit >= 0; --bit) {
                int cnt = 0;
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    cnt += c[e] != kU64Max && (static_cast<uint32_t>(c[e] >> 32) >> bit) == (T >> bit);
                cnt = __reduce_add_sync(0xffffffffu, cnt);
                if (cnt < need) {
                    need -= cnt;
                    T |= 1u << bit;
                }
            }
            lbound = (static_cast<unsigned long long>(T) << 32) | 0xffffffffull;
        }
        const unsigned long long g = *reinterpret_cast<volatile unsigned long long*>(&ws->bound);
        const unsigned long long bnd = g < lbound ? g : lbound;
#pragma unroll
        for (int e = 0; e < 8; ++e)  // the seed block's own candidates
            if (c[e] != kU64Max && c[e] <= bnd) s_buf[atomicAdd(&s_cnt, 1)] = c[e];
        if (lane == 0) {
            s_bound = lbound;
            if (lbound < g) atomicMin(&ws->bound, lbound);
        }
    }
    __syncthreads();
    ZI_TPHASE(2)
    {  // blocks that can still hold a winner (the seed block is done)
        const unsigned long long g = *reinterpret_cast<volatile unsigned long long*>(&ws->bound);
        const unsigned long long bnd = g < s_bound ? g : s_bound;
        for (int r = 0; r < kLatBlkRegs; ++r) {
            const unsigned long long e = s_lbb[tid + kLatThreads * r];
            if (e != kU64Max && e != seed && (e & 0xffffffff00000000ull) <= bnd) s_surv[atomicAdd(&s_nsurv, 1)] = e;
        }
    }
    __syncthreads();
    const int nsurv = s_nsurv;
    // score the survivors, kLatWarps blocks at a time; a round never overfills the buffer
    for (int s0 = 0; s0 < nsurv; s0 += kLatWarps) {
        const int si = s0 + warp;
        if (si < nsurv) {
            const unsigned long long g = *reinterpret_cast<volatile unsigned long long*>(&ws->bound);
            const unsigned long long bnd = g < s_bound ? g : s_bound;
            const unsigned long long e0 = s_surv[si];
            if ((e0 & 0xffffffff00000000ull) <= bnd) {
                unsigned long long c[8];
                score_block<P>(v, e0 & 0xffffffffull, q4, norm, c);
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    if (c[e] != kU64Max && c[e] <= bnd) s_buf[atomicAdd(&s_cnt, 1)] = c[e];
            }
        }
        if (s0 + kLatWarps < nsurv) {
            __syncthreads();
            if (s_cnt > kLatCap - kLatWarps * 256) compact_buffer(s_buf, &s_cnt, &s_bound, k, ws, true);
            __syncthreads();
        }
    }
    __syncthreads();
    ZI_TPHASE(3)
    if (prm.dbg && tid == 0) {
        prm.dbg[4 * blockIdx.x + 2] = static_cast<unsigned long long>(nsurv);
        prm.dbg[4 * blockIdx.x + 3] = static_cast<unsigned long long>(s_cnt);
    }
    {  // exact local top-k (unsorted), then the winners that can still make the global top-k
        const int m0 = s_cnt;
        uint32_t mx = 0;
        for (int t = tid; t < m0; t += kLatThreads) mx = max(mx, static_cast<uint32_t>(s_buf[t] >> 32));
        mx = __reduce_max_sync(0xffffffffu, mx);
        __shared__ uint32_t s_mx;
        if (tid == 0) s_mx = 0;
        __syncthreads();
        if (lane == 0) atomicMax(&s_mx, mx);
        __syncthreads();
        int cnt = select_topk(s_buf, m0, k, sel, tmp, kOneBinCap, hist, 256, s_mx, false);
        if (cnt < 0) {  // degenerate boundary bin: exact sort-based compaction instead
            compact_buffer(s_buf, &s_cnt, &s_bound, k, ws, true);
            cnt = s_cnt;
            for (int t = tid; t < cnt; t += kLatThreads) sel[t] = s_buf[t];
            __syncthreads();
        }
        __shared__ unsigned long long s_kth, s_gb;
        __shared__ int s_keep;
        if (tid == 0) {
            s_kth = 0;
            s_keep = 0;
        }
        __syncthreads();
        unsigned long long kth = 0;
        for (int t = tid; t < cnt; t += kLatThreads) kth = sel[t] > kth ? sel[t] : kth;
        if (cnt >= static_cast<int>(k)) {
            atomicMax(&s_kth, kth);
            __syncthreads();
            if (tid == 0) atomicMin(&ws->bound, s_kth);
        }
        __syncthreads();
        if (tid == 0) s_gb = *reinterpret_cast<volatile unsigned long long*>(&ws->bound);
        __syncthreads();
        const unsigned long long gb = s_gb;
        for (int t = tid; t < cnt; t += kLatThreads)
            if (sel[t] <= gb) tmp[atomicAdd(&s_keep, 1)] = sel[t];
        __syncthreads();
        const int keep = s_keep;
        cost_candidates(prm.img, prm.w, C, mv.K, s_t, s_loc, s_nloc, tmp, keep, norm, s_cost);
        __shared__ uint32_t s_gbase;
        if (tid == 0) s_gbase = atomicAdd(&ws->gcount, static_cast<uint32_t>(keep));
        __syncthreads();
        for (int t = tid; t < keep; t += kLatThreads) {
            prm.cand[s_gbase + t] = tmp[t];
            prm.ccost[s_gbase + t] = s_cost[t];
        }
    }
    ZI_TPHASE(4)
    if (prm.dbg && tid == 0) prm.dbg[4 * blockIdx.x + 1] = gtimer();
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(&ws->done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    ZI_TPHASE(6)
    int m;
    uint32_t maxd, total;
    {  // compact global list -> candidates <= the final bound
        __shared__ int s_m;
        __shared__ uint32_t s_maxd;
        if (tid == 0) {
            s_m = 0;
            s_maxd = 0;
        }
        __syncthreads();
        total = *reinterpret_cast<volatile uint32_t*>(&ws->gcount);
        const unsigned long long bound = *reinterpret_cast<volatile unsigned long long*>(&ws->bound);
        for (uint32_t f = tid; f < total; f += kLatThreads) {
            const unsigned long long c = __ldcg(prm.cand + f);
            if (c <= bound) {
                const int slot = atomicAdd(&s_m, 1);
                if (slot < kLatCap) {
                    s_buf[slot] = c;
                    s_cost[slot] = __ldcg(prm.ccost + f);
                }
                atomicMax(&s_maxd, static_cast<uint32_t>(c >> 32));
            }
        }
        __syncthreads();
        m = s_m;
        maxd = s_maxd;
    }
    ZI_TPHASE(7)
    const unsigned long long T = m > kLatCap ? kU64Max - 1 : kth_packed(s_buf, m, k, tmp, kOneBinCap, hist, 256, maxd);
    int cnt = T == kU64Max - 1 ? -1 : (m < static_cast<int>(k) ? m : static_cast<int>(k));
    if (cnt >= 0 && prm.want_list) cnt = select_sorted_topk(s_buf, m, k, sel, tmp, kOneBinCap, hist, 256, maxd);
    ZI_TPHASE(8)
    if (tid == 0) {
        ws->lid = static_cast<uint32_t>(lid);
        ws->dbg_total = total;
        ws->dbg_m = static_cast<uint32_t>(m);
        ws->final_bound = ws->bound;
        ws->done = 0;
        ws->gcount = 0;
    }
    if (cnt < 0) {
        if (tid == 0) {
            ws->overflow = 2;
            if (prm.res) {
                prm.res->lid = static_cast<uint32_t>(lid);
                prm.res->overflow = 2;
                __threadfence_system();
                prm.res->seq = prm.seq;
            }
        }
        return;  // host: the multi-launch path re-runs this query
    }
    if (prm.want_list)
        for (int i = tid; i < cnt; i += kLatThreads) prm.out[i] = sel[i];
    {
        __shared__ unsigned long long s_best;
        if (tid == 0) s_best = kU64Max;
        __syncthreads();
        unsigned long long best = kU64Max;
        for (int i = tid; i < m; i += kLatThreads)
            if (s_buf[i] <= T) {
                const unsigned long long c = pack_candidate(s_cost[i], static_cast<uint32_t>(s_buf[i] & 0xffffffffu));
                best = c < best ? c : best;
            }
        best = warp_min(best);
        if (lane == 0) atomicMin(&s_best, best);
        __syncthreads();
        if (tid == 0) ws->best = s_best;
    }
    ZI_TPHASE(9)
    if (tid == 0) {
        ws->count = static_cast<uint32_t>(cnt);
        ws->overflow = 0;
        ws->bound = kU64Max;  // the workspace is left ready for the next query
        if (prm.res) {
            prm.res->best = ws->best;
            prm.res->lid = static_cast<uint32_t>(lid);
            prm.res->count = static_cast<uint32_t>(cnt);
            prm.res->overflow = 0;
            __threadfence_system();
            prm.res->seq = prm.seq;
        }
    }
}

// ===================================================================== fused single-CTA query
// The fill loop's per-iteration query in ONE launch (1024 threads): stage the target,
// select_index, make_query, seed the bound from the 8 blocks with the smallest bbox lower bound,
// bbox-pruned pass over every block appending candidates <= bound, exact top-k by sort, refine.
// If more than kFusedCap candidates survive it sets ws->overflow and the host re-runs the
// multi-CTA path (k_query_prep / k_knn_scan / k_knn_merge / k_refine) -- results identical.
constexpr int kFusedThreads = 512;
constexpr int kFusedCap = 8192;
constexpr uint32_t kFusedMaxK = 1024;

template <int P>
__global__ void __launch_bounds__(kFusedThreads) k_query_fused(mi_view mv, const uint8_t* __restrict__ img, int w,
                                                              const uint8_t* __restrict__ target, qws* ws, uint32_t k,
                                                              int norm, unsigned long long* __restrict__ out_list) {
    extern __shared__ unsigned long long s_buf[];  // kFusedCap candidates | xc | comp | target | locals
    __shared__ int s_ov[8];
    __shared__ int s_lid, s_cnt, s_nloc, s_overflow;
    __shared__ uint8_t s_q[32];
    __shared__ unsigned long long s_seed[32];
    __shared__ unsigned long long s_best;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int KK = mv.K * mv.K, mc = mv.m * mv.C, C = mv.C, D = mv.D;
    double* s_xc = reinterpret_cast<double*>(s_buf + kFusedCap);
    double* s_comp = s_xc + mc;
    uint8_t* s_t = reinterpret_cast<uint8_t*>(s_comp + static_cast<size_t>(mc) * D);
    uint16_t* s_loc = reinterpret_cast<uint16_t*>(s_t + ((KK * C + KK + 1) & ~1));
    const int tbytes = KK * C + KK;
    for (int i = tid; i < tbytes; i += kFusedThreads) s_t[i] = target[i];
    if (tid == 0) {
        s_cnt = 0;
        s_overflow = 0;
        s_best = kU64Max;
    }
    if (tid < 32) s_q[tid] = 0;
    __syncthreads();
    const uint8_t* tv = s_t;
    const uint8_t* tk = s_t + KK * C;
    // select_index (engine.cpp:162-176) + known locals (engine.cpp:16-22)
    if (warp < 8) {
        int ov = 0;
        for (int p = lane; p < mv.m; p += 32) ov += tk[mv.local[warp * mv.m + p]] != 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ov += __shfl_xor_sync(0xffffffffu, ov, o);
        if (lane == 0) s_ov[warp] = ov;
    } else if (warp == 8) {
        int c = 0;
        for (int base = 0; base < KK; base += 32) {
            const bool kn = base + lane < KK && tk[base + lane] != 0;
            const unsigned m = __ballot_sync(0xffffffffu, kn);
            if (kn) s_loc[c + __popc(m & ((1u << lane) - 1u))] = static_cast<uint16_t>(base + lane);
            c += __popc(m);
        }
        if (lane == 0) s_nloc = c;
    }
    __syncthreads();
    if (tid == 0) {
        int best = 0, bid = 0;
        for (int l = 0; l < 8; ++l)
            if (s_ov[l] > best) {
                best = s_ov[l];
                bid = l;
            }
        s_lid = bid;
    }
    __syncthreads();
    const int lid = s_lid;
    // make_query (builder.cpp:110-127), canonical fp64 order
    {
        const double* mean = mv.mean + static_cast<size_t>(lid) * mc;
        const int32_t* loc = mv.local + lid * mv.m;
        for (int j = tid; j < mc; j += kFusedThreads) {
            const int l = loc[j / C];
            const double mj = mean[j];
            const double x = tk[l] ? static_cast<double>(tv[l * C + j % C]) : mj;
            s_xc[j] = __dsub_rn(x, mj);
        }
        const double* comp = mv.comp + static_cast<size_t>(lid) * mc * D;
        for (int i = tid; i < mc * D; i += kFusedThreads) s_comp[i] = comp[i];
    }
    __syncthreads();
    if (tid < D) {
        double y = 0.0;
        for (int j = 0; j < mc; ++j) y = __fma_rn(s_comp[j * D + tid], s_xc[j], y);
        const unsigned long long* mm = mv.minmax + static_cast<size_t>(lid) * 2 * D;
        s_q[tid] = quantize_rn(ordered_to_double_hd(mm[tid]), ordered_to_double_hd(mm[D + tid]), y);
    }
    __syncthreads();
    uint32_t q4[8];
#pragma unroll
    for (int p = 0; p < 8; ++p)
        q4[p] = static_cast<uint32_t>(s_q[4 * p]) | (static_cast<uint32_t>(s_q[4 * p + 1]) << 8) |
                (static_cast<uint32_t>(s_q[4 * p + 2]) << 16) | (static_cast<uint32_t>(s_q[4 * p + 3]) << 24);
    const index_view v = mv.idx[lid];
    const uint64_t nblk = v.nblk;
    // seed: every warp's best block by bbox lower bound; score the 8 best of those
    {
        unsigned long long mine = kU64Max;
        for (uint64_t b = static_cast<uint64_t>(warp) * 32 + lane; b < nblk; b += kFusedThreads) {
            uint32_t lb = 0;
#pragma unroll
            for (int p = 0; p < P; ++p)
                lb = gap4(q4[p], v.bmin[static_cast<size_t>(p) * nblk + b], v.bmax[static_cast<size_t>(p) * nblk + b], norm, lb);
            const unsigned long long c = (static_cast<unsigned long long>(lb) << 32) | b;
            mine = c < mine ? c : mine;
        }
        mine = warp_min(mine);
        if (lane == 0) s_seed[warp] = mine;
    }
    __syncthreads();
    if (warp == 0) {  // sort the warp minima (bitonic in registers)
        unsigned long long x = lane < kFusedThreads / 32 ? s_seed[lane] : kU64Max;
        for (int size = 2; size <= 32; size <<= 1)
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                const unsigned long long y = __shfl_xor_sync(0xffffffffu, x, stride);
                const bool up = (lane & size) == 0;
                const bool lower = (lane & stride) == 0;
                x = (lower == up) ? (x < y ? x : y) : (x < y ? y : x);
            }
        s_seed[lane] = x;
    }
    __syncthreads();
    if (warp < 8) {
        const unsigned long long sb = s_seed[warp];
        unsigned long long c[8];
        if (sb != kU64Max) {
            score_block<P>(v, sb & 0xffffffffull, q4, norm, c);
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) c[e] = kU64Max;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) s_buf[warp * 256 + e * 32 + lane] = c[e];
    }
    __syncthreads();
    block_bitonic_sort(s_buf, 2048);
    const unsigned long long seed_bound_v = (k <= 2048) ? s_buf[k - 1] : kU64Max;  // MAX if fewer than k
    __syncthreads();
    // pass over every block
    {
        const unsigned long long bound = seed_bound_v;
        for (uint64_t b0 = static_cast<uint64_t>(warp) * 32; b0 < nblk; b0 += kFusedThreads) {
            const uint64_t b = b0 + lane;
            uint32_t lb = 0xffffffffu;
            if (b < nblk) {
                lb = 0;
#pragma unroll
                for (int p = 0; p < P; ++p)
                    lb = gap4(q4[p], v.bmin[static_cast<size_t>(p) * nblk + b], v.bmax[static_cast<size_t>(p) * nblk + b], norm,
                              lb);
            }
            unsigned live = __ballot_sync(0xffffffffu, b < nblk && (static_cast<unsigned long long>(lb) << 32) <= bound);
            while (live) {
                const int src = __ffs(live) - 1;
                live &= live - 1;
                unsigned long long c[8];
                score_block<P>(v, b0 + src, q4, norm, c);
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const bool take = c[e] != kU64Max && c[e] <= bound;
                    const unsigned m = __ballot_sync(0xffffffffu, take);
                    int base = 0;
                    if (lane == 0 && m) base = atomicAdd(&s_cnt, __popc(m));
                    base = __shfl_sync(0xffffffffu, base, 0);
                    if (take) {
                        const int slot = base + __popc(m & ((1u << lane) - 1u));
                        if (slot < kFusedCap) s_buf[slot] = c[e];
                        else s_overflow = 1;
                    }
                }
            }
        }
    }
    __syncthreads();
    if (s_overflow) {
        if (tid == 0) {
            ws->overflow = 1;
            ws->lid = static_cast<uint32_t>(lid);
        }
        return;
    }
    const int m = s_cnt;
    {
        int sz = 2;
        while (sz < m) sz <<= 1;
        for (int t = m + tid; t < sz; t += kFusedThreads) s_buf[t] = kU64Max;
        __syncthreads();
        block_bitonic_sort(s_buf, sz);
    }
    const int cnt = m < static_cast<int>(k) ? m : static_cast<int>(k);
    // refine (engine.cpp:197-210): warp per candidate, min packed (cost, key)
    const int nloc = s_nloc;
    for (int e = warp; e < cnt; e += kFusedThreads / 32) {
        const uint32_t key = static_cast<uint32_t>(s_buf[e] & 0xffffffffu);
        const int sx = key & 0xffff, sy = key >> 16;
        uint32_t acc = 0;
        for (int li = lane; li < nloc; li += 32) {
            const int l = s_loc[li];
            const int ly = l / mv.K, lx = l % mv.K;
            const uint8_t* sp = img + (static_cast<size_t>(sy + ly) * w + sx + lx) * C;
            const uint8_t* tp = tv + l * C;
            for (int ch = 0; ch < C; ++ch) {
                const int d = static_cast<int>(tp[ch]) - static_cast<int>(__ldg(sp + ch));
                acc += norm == 0 ? static_cast<uint32_t>(d * d) : static_cast<uint32_t>(d < 0 ? -d : d);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) atomicMin(&s_best, pack_candidate(acc, key));
    }
    if (out_list)
        for (int t = tid; t < cnt; t += kFusedThreads) out_list[t] = s_buf[t];
    __syncthreads();
    if (tid == 0) {
        ws->best = s_best;
        ws->count = static_cast<uint32_t>(cnt);
        ws->lid = static_cast<uint32_t>(lid);
        ws->overflow = 0;
    }
}

// ===================================================================== batched k-NN (warp per query)
// cfg-5 style throughput path: one warp answers one query end to end -- 32-ary Morton
// lower_bound, a seed window for the first k-th bound, then every 256-entry block visited in
// outward order from the seed block (32 bboxes per warp step, pruned iff (lb<<32) > bound),
// candidates <= bound appended to a private shared-memory buffer that is sorted and cut to k
// when it fills.  Same exactness argument as the multi-CTA scan.
constexpr int kWarpBuf = 1024;     // u64 candidates per warp
constexpr uint32_t kWarpMaxK = 256;
constexpr int kBatchWarps = 4;

__device__ inline void warp_bitonic_sort(unsigned long long* a, int n) {
    const int lane = threadIdx.x & 31;
    for (int size = 2; size <= n; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = lane; t < (n >> 1); t += 32) {
                const int i = 2 * stride * (t / stride) + (t % stride);
                const int j = i + stride;
                const bool up = (i & size) == 0;
                const unsigned long long x = a[i], y = a[j];
                if ((x > y) == up) {
                    a[i] = y;
                    a[j] = x;
                }
            }
            __syncwarp();
        }
}

// sort buf[0..cnt), keep the k smallest that are <= bound; returns the new count and tightens bound
__device__ inline int warp_compact(unsigned long long* buf, int cnt, uint32_t k, unsigned long long& bound) {
    const int lane = threadIdx.x & 31;
    if (cnt == 0) return 0;
    int sz = 32;
    while (sz < cnt) sz <<= 1;
    for (int t = cnt + lane; t < sz; t += 32) buf[t] = kU64Max;
    __syncwarp();
    warp_bitonic_sort(buf, sz);
    if (cnt >= static_cast<int>(k)) {
        const unsigned long long kth = buf[k - 1];
        if (kth < bound) bound = kth;
        cnt = static_cast<int>(k);
    }
    while (cnt > 0 && buf[cnt - 1] > bound) --cnt;  // warp-uniform
    return cnt;
}

__device__ inline int64_t outward_block(int64_t b0, int64_t v, int64_t nblk) {
    const int64_t b = (v & 1) ? b0 - (v + 1) / 2 : b0 + v / 2;
    return (b >= 0 && b < nblk) ? b : -1;
}

template <int P>
__global__ void __launch_bounds__(32 * kBatchWarps) k_knn_batch(index_view v, const uint8_t* __restrict__ queries,
                                                               uint64_t nq, uint32_t k, int norm, int win,
                                                               unsigned long long* __restrict__ out,
                                                               uint32_t* __restrict__ counts,
                                                               unsigned long long* __restrict__ stats) {
    __shared__ unsigned long long s_buf[kBatchWarps][kWarpBuf];
    __shared__ uint8_t s_q[kBatchWarps][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long* buf = s_buf[warp];
    uint8_t* q = s_q[warp];
    unsigned long long st_blocks = 0, st_scored = 0, st_cand = 0;
    const uint32_t lt_mask = (1u << lane) - 1u;
    for (uint64_t qi = static_cast<uint64_t>(blockIdx.x) * kBatchWarps + warp; qi < nq;
         qi += static_cast<uint64_t>(gridDim.x) * kBatchWarps) {
        q[lane] = lane < v.D ? queries[qi * v.D + lane] : 0;
        __syncwarp();
        uint32_t q4[8];
#pragma unroll
        for (int p = 0; p < 8; ++p)
            q4[p] = static_cast<uint32_t>(q[4 * p]) | (static_cast<uint32_t>(q[4 * p + 1]) << 8) |
                    (static_cast<uint32_t>(q[4 * p + 2]) << 16) | (static_cast<uint32_t>(q[4 * p + 3]) << 24);
        // 32-ary lower_bound in Morton order; invariant: position in [lo, hi]
        uint64_t lo = 0, hi = v.n;
        while (hi - lo > 32) {
            const uint64_t len = hi - lo;
            const uint64_t piv = lo + (static_cast<uint64_t>(lane) + 1) * len / 33;
            const int c = __popc(__ballot_sync(0xffffffffu, entry_less_query(v, piv, q)));
            const uint64_t nlo = c > 0 ? lo + static_cast<uint64_t>(c) * len / 33 + 1 : lo;
            const uint64_t nhi = c < 32 ? lo + (static_cast<uint64_t>(c) + 1) * len / 33 : hi;
            lo = nlo;
            hi = nhi;
        }
        {
            const bool less = lo + lane < hi && entry_less_query(v, lo + lane, q);
            lo += __popc(__ballot_sync(0xffffffffu, less));
        }
        const uint64_t pos = lo;
        // seed window -> first bound
        unsigned long long bound = kU64Max;
        {
            const uint64_t wn = v.n < static_cast<uint64_t>(win) ? v.n : static_cast<uint64_t>(win);
            uint64_t start = pos > wn / 2 ? pos - wn / 2 : 0;
            if (start + wn > v.n) start = v.n - wn;
            for (int t = lane; t < win; t += 32)
                buf[t] = static_cast<uint64_t>(t) < wn
                             ? pack_candidate(entry_dist(v, start + t, q4, norm), v.keys[start + t])
                             : kU64Max;
            __syncwarp();
            warp_bitonic_sort(buf, win);
            if (wn >= k) bound = buf[k - 1];
            __syncwarp();
        }
        // outward scan over all blocks
        int cnt = 0;
        const int64_t nblk = static_cast<int64_t>(v.nblk);
        const int64_t b0 = static_cast<int64_t>(pos / 256 < v.nblk ? pos / 256 : v.nblk - 1);
        const int64_t span = 2 * (b0 + 1 > nblk - b0 ? b0 + 1 : nblk - b0);
        for (int64_t vb = 0; vb < span; vb += 32) {
            const int64_t b = outward_block(b0, vb + lane, nblk);
            uint32_t lb = 0xffffffffu;
            if (b >= 0) {
                lb = 0;
#pragma unroll
                for (int p = 0; p < P; ++p)
                    lb = gap4(q4[p], v.bmin[static_cast<size_t>(p) * v.nblk + b], v.bmax[static_cast<size_t>(p) * v.nblk + b],
                              norm, lb);
                ++st_blocks;
            }
            unsigned live = __ballot_sync(0xffffffffu, b >= 0 && (static_cast<unsigned long long>(lb) << 32) <= bound);
            while (live) {
                const int src = __ffs(live) - 1;
                live &= live - 1;
                const int64_t bb = __shfl_sync(0xffffffffu, b, src);
                const uint32_t blb = __shfl_sync(0xffffffffu, lb, src);
                if ((static_cast<unsigned long long>(blb) << 32) > bound) continue;  // bound tightened meanwhile
                if (cnt > kWarpBuf - 256) cnt = warp_compact(buf, cnt, k, bound);
                unsigned long long c[8];
                score_block<P>(v, static_cast<uint64_t>(bb), q4, norm, c);
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const bool take = c[e] != kU64Max && c[e] <= bound;
                    st_scored += c[e] != kU64Max;
                    const unsigned m = __ballot_sync(0xffffffffu, take);
                    if (take) buf[cnt + __popc(m & lt_mask)] = c[e];
                    cnt += __popc(m);
                }
                __syncwarp();
            }
        }
        cnt = warp_compact(buf, cnt, k, bound);
        for (int t = lane; t < cnt; t += 32) out[qi * k + t] = buf[t];
        if (lane == 0) counts[qi] = static_cast<uint32_t>(cnt);
        st_cand += static_cast<unsigned long long>(cnt);
        __syncwarp();
    }
    if (stats) {
        atomicAdd(stats + 0, st_blocks);
        atomicAdd(stats + 1, st_scored);
        if (lane == 0) atomicAdd(stats + 2, st_cand);
    }
}

// ===================================================================== host side
void radix_sort_words(zi_ctx* ctx, uint32_t** words, int nw, uint64_t n, const std::vector<int2>& passes,
                      const uint32_t* hist_host, bool device_bases);

static index_view view_of(const zi_index* idx) {
    index_view v;
    v.planes = idx->planes.p;
    v.keys = idx->keys.p;
    v.bmin = idx->bbox_min.p;
    v.bmax = idx->bbox_max.p;
    v.n = idx->n;
    v.nblk = idx->nblk;
    v.P = static_cast<int>(idx->planes_n);
    v.D = static_cast<int>(idx->dims);
    return v;
}

static int seed_window(uint32_t k) {
    int w = 256;
    while (w < static_cast<int>(2 * k) && w < 4096) w <<= 1;
    return w;
}

struct query_scratch {
    qws* ws;
    uint32_t* cand_cnt;
    unsigned long long* cand;
    uint32_t* ccost;  // k_query_one: masked cost of each cand entry
    unsigned long long* out;
    uint8_t* target;
    int G;
};

static query_scratch carve(dbuf<uint8_t>& buf, const zi_ctx* ctx, uint64_t nblk, uint32_t k, size_t target_bytes) {
    query_scratch s;
    s.G = static_cast<int>(std::min<uint64_t>(std::min<uint64_t>(std::max<uint64_t>(nblk, 1), static_cast<uint64_t>(ctx->num_sms) * 2), 1024));
    const size_t kk = std::max<uint32_t>(k, 1);
    const size_t kscan = std::min<size_t>(kk, kMaxScanK);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off = (off + bytes + 255) & ~size_t(255);
        return o;
    };
    const size_t o_ws = take(sizeof(qws));
    const size_t o_cc = take(s.G * sizeof(uint32_t));
    const size_t o_c = take(static_cast<size_t>(s.G) * kscan * sizeof(unsigned long long));
    const size_t o_cc2 = take(static_cast<size_t>(s.G) * kscan * sizeof(uint32_t));
    const size_t o_out = take(kk * sizeof(unsigned long long));
    const size_t o_t = take(target_bytes + 64);
    uint8_t* b = buf.ensure(off);
    s.ws = reinterpret_cast<qws*>(b + o_ws);
    s.cand_cnt = reinterpret_cast<uint32_t*>(b + o_cc);
    s.cand = reinterpret_cast<unsigned long long*>(b + o_c);
    s.ccost = reinterpret_cast<uint32_t*>(b + o_cc2);
    s.out = reinterpret_cast<unsigned long long*>(b + o_out);
    s.target = b + o_t;
    return s;
}

// scan + merge, or the exhaustive sort for very large k; result sorted in s.out, count in ws.
// The layout actually searched is ws->lid (set by the prep kernel).
struct refine_args {
    const uint8_t* img;
    int w, C, K;
};

// Returns true when the refine (if requested) already ran inside the selection kernel.
static bool run_knn(zi_ctx* ctx, const views8& V, uint64_t n, uint64_t nblk, const query_scratch& s, uint32_t k,
                    int norm, const refine_args* ra = nullptr) {
    (void)nblk;
    if (k <= kMaxScanK) {
        switch (V.v[0].P) {
#define ZI_SCAN_CASE(PP) \
    case PP: ZI_LAUNCH(ctx, "knn_scan", k_knn_scan<PP>, s.G, kScanThreads, 0, V, s.ws, k, norm, s.cand_cnt, s.cand); break;
            ZI_SCAN_CASE(1) ZI_SCAN_CASE(2) ZI_SCAN_CASE(3) ZI_SCAN_CASE(4)
            ZI_SCAN_CASE(5) ZI_SCAN_CASE(6) ZI_SCAN_CASE(7) ZI_SCAN_CASE(8)
#undef ZI_SCAN_CASE
            default: throw error(ZI_E_INVALID, "dims above 32");
        }
        smem_attr(ctx->device, k_knn_select, 200 * 1024);
        const size_t smem = (kSelCap + 2048 + kSelBinCap) * sizeof(unsigned long long) + (kSelBins + 1) * sizeof(uint32_t);
        ZI_LAUNCH(ctx, "knn_select", k_knn_select, 1, kSelThreads, smem, s.ws, k, s.G, s.cand_cnt, s.cand, s.out,
                  ra ? ra->img : nullptr, ra ? ra->w : 0, ra ? ra->C : 1, ra ? ra->K : 1, ra ? s.target : nullptr, norm);
        return ra != nullptr;
    }
    // exhaustive: sort all n packed values (two-word LSD radix), take the first min(k, n)
    uint32_t* lohi = ctx->counter.ensure(2 * n + 64);
    uint32_t* lo = lohi;
    uint32_t* hi = lohi + n;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(ctx->num_sms) * 8));
    ZI_LAUNCH(ctx, "knn_pack_all", k_pack_all, grid, 256, 0, V, s.ws, norm, lo, hi);
    uint32_t* words[2] = {lo, hi};
    std::vector<int2> passes;
    for (int b = 0; b < 4; ++b) passes.push_back(make_int2(0, 8 * b));
    for (int b = 0; b < 4; ++b) passes.push_back(make_int2(1, 8 * b));
    radix_sort_words(ctx, words, 2, n, passes, nullptr, false);
    const uint32_t cnt = static_cast<uint32_t>(std::min<uint64_t>(k, n));
    ZI_LAUNCH(ctx, "knn_gather_topk", k_gather_topk, (cnt + 255) / 256, 256, 0, lo, hi, cnt, s.ws, s.out);
    return false;
}

// rare: the selection kernel gave up (ws->overflow == 2) -> chunked merge (+ refine)
static void knn_fallback(zi_ctx* ctx, const query_scratch& s, uint32_t k, int norm, const refine_args* ra,
                         size_t rsmem) {
    ZI_LAUNCH(ctx, "knn_merge", k_knn_merge, 1, kMergeThreads, 0, s.ws, k, s.G, s.cand_cnt, s.cand, s.out);
    if (ra) ZI_LAUNCH(ctx, "refine", k_refine, 1, 1024, rsmem, ra->img, ra->w, ra->C, ra->K, s.target, s.ws, s.out, norm);
}

static void ensure_smem_attr(const zi_ctx* ctx) {
#define ZI_ATTR(PP)                                                    \
    smem_attr(ctx->device, k_seed_query<PP>, 4096 * 8);                \
    smem_attr(ctx->device, k_query_prep<PP>, 220 * 1024);
    ZI_ATTR(1) ZI_ATTR(2) ZI_ATTR(3) ZI_ATTR(4) ZI_ATTR(5) ZI_ATTR(6) ZI_ATTR(7) ZI_ATTR(8)
#undef ZI_ATTR
}

static int seed_smem_words(uint32_t k) { return std::max(seed_window(k), 2048); }

uint32_t knn_search(zi_index* idx, const uint8_t* h_query, uint32_t k, int norm, uint64_t* out) {
    zi_ctx* ctx = idx->ctx;
    k = std::max<uint32_t>(k, 1);  // knn_list capacity = max(k, 1) (proj/src/zcurve.cpp:25-31)
    if (idx->n == 0) return 0;
    ensure_smem_attr(ctx);
    views8 V;
    for (int l = 0; l < 8; ++l) V.v[l] = view_of(idx);
    const query_scratch s = carve(idx->qscratch, ctx, idx->nblk, k, 32);
    uint8_t* stage = idx->hstage.ensure(64 + ((sizeof(qws) + 63) & ~size_t(63)));
    std::memset(stage, 0, 32);
    std::memcpy(stage, h_query, idx->dims);
    ZI_CUDA(cudaMemcpyAsync(s.target, stage, 32, cudaMemcpyHostToDevice, ctx->stream));
    const int win = seed_window(k);
    const size_t seed_smem = seed_smem_words(k) * sizeof(unsigned long long);
    switch (V.v[0].P) {
#define ZI_SEED_CASE(PP) \
    case PP: ZI_LAUNCH(ctx, "knn_seed", k_seed_query<PP>, 1, 256, seed_smem, V.v[0], s.target, s.ws, k, norm, win); break;
        ZI_SEED_CASE(1) ZI_SEED_CASE(2) ZI_SEED_CASE(3) ZI_SEED_CASE(4)
        ZI_SEED_CASE(5) ZI_SEED_CASE(6) ZI_SEED_CASE(7) ZI_SEED_CASE(8)
#undef ZI_SEED_CASE
        default: throw error(ZI_E_INVALID, "dims above 32");
    }
    run_knn(ctx, V, idx->n, idx->nblk, s, k, norm);
    qws* hq = reinterpret_cast<qws*>(stage + 64);
    ZI_CUDA(cudaMemcpyAsync(hq, s.ws, sizeof(qws), cudaMemcpyDeviceToHost, ctx->stream));
    ZI_CUDA(cudaStreamSynchronize(ctx->stream));
    if (k <= kMaxScanK && hq->overflow == 2) {
        knn_fallback(ctx, s, k, norm, nullptr, 0);
        ZI_CUDA(cudaMemcpyAsync(hq, s.ws, sizeof(qws), cudaMemcpyDeviceToHost, ctx->stream));
        ZI_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    const uint32_t cnt = static_cast<uint32_t>(std::min<uint64_t>(hq->count, std::min<uint64_t>(k, idx->n)));
    if (cnt) {
        ZI_CUDA(cudaMemcpyAsync(out, s.out, cnt * sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
        ZI_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    return cnt;
}

void knn_search_batch(zi_index* idx, const uint8_t* h_queries, uint64_t nq, uint32_t k, int norm, uint64_t* out,
                      uint32_t* counts) {
    const uint32_t kk = std::max<uint32_t>(k, 1);
    if (nq == 0) return;
    if (idx->n == 0) {
        std::memset(counts, 0, nq * sizeof(uint32_t));
        return;
    }
    if (kk > kWarpMaxK) {  // large k: one multi-CTA query at a time
        for (uint64_t q = 0; q < nq; ++q) counts[q] = knn_search(idx, h_queries + q * idx->dims, kk, norm, out + q * kk);
        return;
    }
    zi_ctx* ctx = idx->ctx;
    const size_t qbytes = nq * idx->dims;
    const size_t obytes = nq * kk * sizeof(uint64_t);
    uint8_t* b = idx->qscratch.ensure(qbytes + obytes + nq * sizeof(uint32_t) + 1024);
    uint8_t* d_q = b;
    unsigned long long* d_out = reinterpret_cast<unsigned long long*>(b + ((qbytes + 255) & ~size_t(255)));
    uint32_t* d_cnt = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(d_out) + obytes);
    ZI_CUDA(cudaMemcpyAsync(d_q, h_queries, qbytes, cudaMemcpyHostToDevice, ctx->stream));
    knn_batch_device(ctx, idx, d_q, nq, kk, norm, d_out, d_cnt, nullptr);
    ZI_CUDA(cudaMemcpyAsync(out, d_out, obytes, cudaMemcpyDeviceToHost, ctx->stream));
    ZI_CUDA(cudaMemcpyAsync(counts, d_cnt, nq * sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
    ZI_CUDA(cudaStreamSynchronize(ctx->stream));
}

void knn_batch_device(zi_ctx* ctx, zi_index* idx, const uint8_t* d_queries, uint64_t nq, uint32_t k, int norm,
                      unsigned long long* d_out, uint32_t* d_counts, unsigned long long* d_stats) {
    const index_view v = view_of(idx);
    int win = 64;
    while (win < static_cast<int>(2 * k)) win <<= 1;  // window >= 2k (<= 512)
    const uint64_t per_cta = kBatchWarps;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((nq + per_cta - 1) / per_cta, 1u << 20));
    switch (v.P) {
#define ZI_BATCH_CASE(PP)                                                                                     \
    case PP:                                                                                                  \
        ZI_LAUNCH(ctx, "knn_batch", k_knn_batch<PP>, grid, 32 * kBatchWarps, 0, v, d_queries, nq, k, norm, win, \
                  d_out, d_counts, d_stats);                                                                  \
        break;
        ZI_BATCH_CASE(1) ZI_BATCH_CASE(2) ZI_BATCH_CASE(3) ZI_BATCH_CASE(4)
        ZI_BATCH_CASE(5) ZI_BATCH_CASE(6) ZI_BATCH_CASE(7) ZI_BATCH_CASE(8)
#undef ZI_BATCH_CASE
        default: throw error(ZI_E_INVALID, "dims above 32");
    }
}

static mi_view mi_view_of(zi_multi_index* mi) {
    mi_view mv;
    for (int l = 0; l < 8; ++l) mv.idx[l] = view_of(&mi->L[l].index);
    mv.local = mi->layout_local.p;
    mv.mean = mi->pca_mean.p;
    mv.comp = mi->pca_comp.p;
    mv.minmax = mi->minmax.p;
    mv.m = mi->m;
    mv.C = mi->C;
    mv.K = mi->K;
    mv.D = mi->dims;
    return mv;
}

static bool fused_query(zi_multi_index* mi, const query_scratch& s, const mi_view& mv, uint32_t k, int norm, qws* hq,
                        bool want_list) {
    zi_ctx* ctx = mi->ctx;
    const size_t KK = static_cast<size_t>(mi->K) * mi->K;
    const size_t smem = kFusedCap * sizeof(unsigned long long) + static_cast<size_t>(mi->mc) * (mi->dims + 1) * sizeof(double) +
                        KK * mi->C + 3 * KK + 64;
    static const bool enabled = std::getenv("ZI_QUERY_FUSED") != nullptr;
    if (!enabled || smem > 220 * 1024 || k > kFusedMaxK) return false;
    switch (mv.idx[0].P) {
#define ZI_FUSED_CASE(PP)                                                                                          \
    case PP: {                                                                                                     \
        smem_attr(ctx->device, k_query_fused<PP>, 220 * 1024);                                                     \
        ZI_LAUNCH(ctx, "query_fused", k_query_fused<PP>, 1, kFusedThreads, smem, mv, mi->image.p, mi->w, s.target, s.ws, \
                  k, norm, want_list ? s.out : nullptr);                                                           \
        break;                                                                                                     \
    }
        ZI_FUSED_CASE(1) ZI_FUSED_CASE(2) ZI_FUSED_CASE(3) ZI_FUSED_CASE(4)
        ZI_FUSED_CASE(5) ZI_FUSED_CASE(6) ZI_FUSED_CASE(7) ZI_FUSED_CASE(8)
#undef ZI_FUSED_CASE
        default: return false;
    }
    ZI_CUDA(cudaMemcpyAsync(hq, s.ws, sizeof(qws), cudaMemcpyDeviceToHost, ctx->stream));
    ZI_CUDA(cudaStreamSynchronize(ctx->stream));
    return hq->overflow == 0;
}

query_result query_best_patch(zi_multi_index* mi, const uint8_t* h_tv, const uint8_t* h_tk, uint32_t k, int norm,
                              uint64_t* knn_out, const std::function<void()>* while_waiting) {
    zi_ctx* ctx = mi->ctx;
    bool waited = false;  // while_waiting runs exactly once, during the device work when possible
    auto run_waiting = [&] {
        if (while_waiting && !waited) {
            waited = true;
            (*while_waiting)();
        }
    };
    struct waiting_guard {  // every other path: run it before returning
        std::function<void()> f;
        ~waiting_guard() { f(); }
    } wg{[&] { run_waiting(); }};
    k = std::max<uint32_t>(k, 1);
    ensure_smem_attr(ctx);
    const size_t KK = static_cast<size_t>(mi->K) * mi->K;
    const size_t tbytes = KK * mi->C + KK;
    const uint64_t nblk = mi->L[0].index.nblk;
    const query_scratch s = carve(mi->qscratch, ctx, nblk, k, tbytes);
    const size_t res_off = (tbytes + 255) & ~size_t(255);
    uint8_t* stage = mi->hstage.ensure(res_off + sizeof(qws));
    std::memcpy(stage, h_tv, KK * mi->C);
    std::memcpy(stage + KK * mi->C, h_tk, KK);
    bool target_on_device = false;  // the low-latency kernel takes the target in its parameters
    auto upload_target = [&] {
        if (target_on_device) return;
        ZI_CUDA(cudaMemcpyAsync(s.target, stage, tbytes, cudaMemcpyHostToDevice, ctx->stream));
        target_on_device = true;
    };
    const mi_view mv = mi_view_of(mi);
    qws* hq = reinterpret_cast<qws*>(stage + res_off);
    const size_t rsmem = ((KK * mi->C + 1) & ~size_t(1)) + (KK + 16) * sizeof(uint16_t) + kRefineSlots * sizeof(uint32_t) + 32;
    const refine_args ra{mi->image.p, mi->w, mi->C, mi->K};
    const size_t one_smem = (kOneCap + kOneMaxK + kOneBinCap) * sizeof(unsigned long long) +
                            (kOneBins + 2 + kOneCap) * sizeof(uint32_t) +
                            static_cast<size_t>(mi->mc) * (mi->dims + 1) * sizeof(double) + tbytes + 2 + KK * 2 + 16;
    bool done = false;
    static const bool force_multi = std::getenv("ZI_QUERY_MULTI") != nullptr;
    static const bool debug_query = std::getenv("ZI_DEBUG_QUERY") != nullptr;
    // mapped pinned result (fast path: no D2H copy, no stream synchronisation)
    if (!mi->hres) {
        ZI_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&mi->hres), sizeof(qres), cudaHostAllocMapped));
        std::memset(mi->hres, 0, sizeof(qres));
        ZI_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&mi->dres), mi->hres, 0));
    }
    qres* hr = reinterpret_cast<qres*>(mi->hres);
    if (s.ws != mi->qws_last) {  // new or moved workspace: contents unknown
        mi->qws_clean = false;
        mi->qws_last = s.ws;
    }
    static const bool use_one = std::getenv("ZI_QUERY_ONE") != nullptr;
    static const int lat_g = [] { const char* e = std::getenv("ZI_QLAT_G"); return e ? std::atoi(e) : 0; }();
    const size_t lat_smem = (kLatCap + kLatMaxK + kOneBinCap) * sizeof(unsigned long long) +
                            (256 + 2 + kLatCap) * sizeof(uint32_t) + static_cast<size_t>(mi->mc) * sizeof(double) +
                            tbytes + 2 + KK * 2 + 16;
    const uint64_t lat_g_max = static_cast<uint64_t>(std::min(s.G, 2 * ctx->num_sms));
    const uint64_t G2 = std::min<uint64_t>(std::max<uint64_t>(nblk, 1),
                                           lat_g > 0 ? static_cast<uint64_t>(lat_g) : lat_g_max);
    if (!use_one && !force_multi && k <= kLatMaxK && tbytes <= static_cast<size_t>(kLatMaxTarget) &&
        static_cast<size_t>(mi->mc) * mi->dims <= static_cast<size_t>(kLatCap - kLatThreads * kLatBlkRegs) &&
        lat_smem <= 112 * 1024 && nblk <= G2 * kLatThreads * kLatBlkRegs) {
        if (!mi->qws_clean) {
            ZI_CUDA(cudaMemsetAsync(&s.ws->bound, 0xff, sizeof(unsigned long long), ctx->stream));
            ZI_CUDA(cudaMemsetAsync(&s.ws->done, 0, 2 * sizeof(uint32_t), ctx->stream));  // done + gcount
        }
        const uint32_t seq = ++mi->qseq;
        qlat_params prm;
        prm.mv = mv;
        prm.img = mi->image.p;
        prm.w = mi->w;
        prm.ws = s.ws;
        prm.k = k;
        prm.norm = norm;
        prm.cand = s.cand;
        prm.ccost = s.ccost;
        prm.out = s.out;
        prm.res = reinterpret_cast<qres*>(mi->dres);
        prm.seq = seq;
        prm.want_list = knn_out != nullptr ? 1 : 0;
        prm.tbytes = static_cast<int>(tbytes);
        static dbuf<unsigned long long> dbg_buf;
        prm.dbg = debug_query ? dbg_buf.ensure(4 * G2) : nullptr;
        std::memcpy(prm.target, h_tv, KK * mi->C);
        std::memcpy(prm.target + KK * mi->C, h_tk, KK);
        switch (mv.idx[0].P) {
#define ZI_LAT_CASE(PP)                                                                                     \
    case PP:                                                                                                \
        smem_attr(ctx->device, k_query_lat<PP>, lat_smem);                                                  \
        ZI_LAUNCH(ctx, "query_one", k_query_lat<PP>, static_cast<unsigned>(G2), kLatThreads, lat_smem, prm); \
        break;
            ZI_LAT_CASE(1) ZI_LAT_CASE(2) ZI_LAT_CASE(3) ZI_LAT_CASE(4)
            ZI_LAT_CASE(5) ZI_LAT_CASE(6) ZI_LAT_CASE(7) ZI_LAT_CASE(8)
#undef ZI_LAT_CASE
            default: throw error(ZI_E_INVALID, "dims above 32");
        }
        if (debug_query || ctx->profiling) {
            ZI_CUDA(cudaMemcpyAsync(hq, s.ws, sizeof(qws), cudaMemcpyDeviceToHost, ctx->stream));
            ZI_CUDA(cudaStreamSynchronize(ctx->stream));
            if (debug_query) {  // CTA start / finish spread relative to the first start
                std::vector<unsigned long long> d(4 * G2);
                ZI_CUDA(cudaMemcpy(d.data(), prm.dbg, d.size() * 8, cudaMemcpyDeviceToHost));
                unsigned long long s0 = ~0ull, s1 = 0, f0 = ~0ull, f1 = 0, sv = 0, sc = 0, slast_v = 0, slast_c = 0;
                for (uint64_t c = 0; c < G2; ++c) {
                    s0 = std::min(s0, d[4 * c]);
                    s1 = std::max(s1, d[4 * c]);
                    f0 = std::min(f0, d[4 * c + 1]);
                    if (d[4 * c + 1] > f1) {
                        f1 = d[4 * c + 1];
                        slast_v = d[4 * c + 2];
                        slast_c = d[4 * c + 3];
                    }
                    sv = std::max(sv, d[4 * c + 2]);
                    sc = std::max(sc, d[4 * c + 3]);
                }
                std::fprintf(stderr,
                             "qlat ctas=%llu start_spread_us=%.1f finish_first_us=%.1f finish_last_us=%.1f "
                             "max_surv=%llu max_cand=%llu last_surv=%llu last_cand=%llu\n",
                             static_cast<unsigned long long>(G2), (s1 - s0) * 1e-3, (f0 - s0) * 1e-3, (f1 - s0) * 1e-3,
                             sv, sc, slast_v, slast_c);
            }
        } else {
            run_waiting();
            unsigned spins = 0;
            while (hr->seq != seq) {
                if ((++spins & 1023u) == 0) {
                    const cudaError_t e = cudaStreamQuery(ctx->stream);
                    if (e != cudaSuccess && e != cudaErrorNotReady) ZI_CUDA(e);
                    if (e == cudaSuccess && hr->seq != seq) throw error(ZI_E_RUNTIME, "query result not published");
                }
            }
            std::atomic_thread_fence(std::memory_order_acquire);
            hq->best = hr->best;
            hq->lid = hr->lid;
            hq->count = hr->count;
            hq->overflow = hr->overflow;
        }
        mi->qws_clean = hq->overflow == 0;
        if (hq->overflow == 0) done = true;  // else: the multi-launch path below answers it
    }
    if (!done) upload_target();
    if (!done && k <= kOneMaxK && one_smem <= 220 * 1024 && !force_multi) {
        const int G1 = static_cast<int>(std::min<uint64_t>(std::max<uint64_t>(nblk, 1),
                                                           std::min<uint64_t>(static_cast<uint64_t>(s.G), 2ull * ctx->num_sms)));
        if (!mi->qws_clean) {
            ZI_CUDA(cudaMemsetAsync(&s.ws->bound, 0xff, sizeof(unsigned long long), ctx->stream));
            ZI_CUDA(cudaMemsetAsync(&s.ws->done, 0, 2 * sizeof(uint32_t), ctx->stream));  // done + gcount
        }
        const uint32_t seq = ++mi->qseq;
        qres* dres = reinterpret_cast<qres*>(mi->dres);
        switch (mv.idx[0].P) {
#define ZI_ONE_CASE(PP)                                                                                              \
    case PP: {                                                                                                       \
        smem_attr(ctx->device, k_query_one<PP>, 220 * 1024);                                                         \
        ZI_LAUNCH(ctx, "query_one", k_query_one<PP>, G1, kOneThreads, one_smem, mv, mi->image.p, mi->w, s.target, s.ws, \
                  k, norm, s.cand_cnt, s.cand, s.ccost, s.out, dres, seq, knn_out != nullptr ? 1 : 0);             \
        break;                                                                                                       \
    }
            ZI_ONE_CASE(1) ZI_ONE_CASE(2) ZI_ONE_CASE(3) ZI_ONE_CASE(4)
            ZI_ONE_CASE(5) ZI_ONE_CASE(6) ZI_ONE_CASE(7) ZI_ONE_CASE(8)
#undef ZI_ONE_CASE
            default: throw error(ZI_E_INVALID, "dims above 32");
        }
        if (debug_query || ctx->profiling) {
            ZI_CUDA(cudaMemcpyAsync(hq, s.ws, sizeof(qws), cudaMemcpyDeviceToHost, ctx->stream));
            ZI_CUDA(cudaStreamSynchronize(ctx->stream));
        } else {
            // spin on the published sequence number; a fault or a finished stream without it is
            // reported instead of spinning forever
            unsigned spins = 0;
            while (hr->seq != seq) {
                if ((++spins & 1023u) == 0) {
                    const cudaError_t e = cudaStreamQuery(ctx->stream);
                    if (e != cudaSuccess && e != cudaErrorNotReady) ZI_CUDA(e);
                    if (e == cudaSuccess && hr->seq != seq) throw error(ZI_E_RUNTIME, "query result not published");
                }
            }
            std::atomic_thread_fence(std::memory_order_acquire);
            hq->best = hr->best;
            hq->lid = hr->lid;
            hq->count = hr->count;
            hq->overflow = hr->overflow;
        }
        mi->qws_clean = hq->overflow == 0;
        if (hq->overflow == 2) {  // rare: the merge did not fit -> chunked merge over the same CTA lists
            ZI_CUDA(cudaStreamSynchronize(ctx->stream));
            query_scratch s1 = s;
            s1.G = 1;
            knn_fallback(ctx, s1, k, norm, &ra, rsmem);
            ZI_CUDA(cudaMemcpyAsync(hq, s.ws, sizeof(qws), cudaMemcpyDeviceToHost, ctx->stream));
            ZI_CUDA(cudaStreamSynchronize(ctx->stream));
        }
        done = true;
    }
    if (!done) mi->qws_clean = false;  // the multi-launch paths leave the workspace as they please
    if (!done && !fused_query(mi, s, mv, k, norm, hq, knn_out != nullptr)) {
        const int win = seed_window(k);
        const size_t prep_smem = seed_smem_words(k) * sizeof(unsigned long long) +
                                 static_cast<size_t>(mi->mc) * (mi->dims + 1) * sizeof(double) + tbytes + 16;
        switch (mv.idx[0].P) {
#define ZI_PREP_CASE(PP) \
    case PP: ZI_LAUNCH(ctx, "query_prep", k_query_prep<PP>, 1, 256, prep_smem, mv, s.target, s.ws, k, norm, \
                       seed_smem_words(k)); break;
            ZI_PREP_CASE(1) ZI_PREP_CASE(2) ZI_PREP_CASE(3) ZI_PREP_CASE(4)
            ZI_PREP_CASE(5) ZI_PREP_CASE(6) ZI_PREP_CASE(7) ZI_PREP_CASE(8)
#undef ZI_PREP_CASE
            default: throw error(ZI_E_INVALID, "dims above 32");
        }
        (void)win;
        views8 V;
        for (int l = 0; l < 8; ++l) V.v[l] = mv.idx[l];
        const bool refined = run_knn(ctx, V, mi->n, nblk, s, k, norm, &ra);
        if (!refined)
            ZI_LAUNCH(ctx, "refine", k_refine, 1, 1024, rsmem, mi->image.p, mi->w, mi->C, mi->K, s.target, s.ws, s.out, norm);
        ZI_CUDA(cudaMemcpyAsync(hq, s.ws, sizeof(qws), cudaMemcpyDeviceToHost, ctx->stream));
        ZI_CUDA(cudaStreamSynchronize(ctx->stream));
        if (refined && hq->overflow == 2) {
            knn_fallback(ctx, s, k, norm, &ra, rsmem);
            ZI_CUDA(cudaMemcpyAsync(hq, s.ws, sizeof(qws), cudaMemcpyDeviceToHost, ctx->stream));
            ZI_CUDA(cudaStreamSynchronize(ctx->stream));
        }
    }
    if (debug_query) {
        std::fprintf(stderr, "query lid=%u bound_dist=%u total=%u m=%u count=%u overflow=%u phases_us:", hq->lid,
                     static_cast<unsigned>(hq->final_bound >> 32), hq->dbg_total, hq->dbg_m, hq->count, hq->overflow);
        for (int i = 1; i < 10; ++i)
            std::fprintf(stderr, " %.1f", (static_cast<double>(hq->tphase[i]) - static_cast<double>(hq->tphase[0])) * 1e-3);
        std::fprintf(stderr, "\n");
    }
    query_result r;
    r.best = hq->best;
    r.lid = hq->lid;
    r.count = static_cast<uint32_t>(std::min<uint64_t>(hq->count, std::min<uint64_t>(k, mi->n)));
    if (knn_out && r.count) {
        ZI_CUDA(cudaMemcpyAsync(knn_out, s.out, r.count * sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
        ZI_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    return r;
}

uint64_t brute_force_scan(zi_ctx* ctx, const uint8_t* d_img, int w, int C, int K, const uint32_t* d_dict, uint64_t n,
                          const uint8_t* h_tv, const uint8_t* h_tk, int norm, dbuf<uint8_t>& scratch,
                          hbuf<uint8_t>& hstage) {
    const size_t KK = static_cast<size_t>(K) * K;
    const size_t tbytes = KK * C + KK;
    const query_scratch s = carve(scratch, ctx, 1, 1, tbytes);
    const size_t res_off = (tbytes + 255) & ~size_t(255);
    uint8_t* stage = hstage.ensure(res_off + sizeof(qws));
    std::memcpy(stage, h_tv, KK * C);
    std::memcpy(stage + KK * C, h_tk, KK);
    ZI_CUDA(cudaMemcpyAsync(s.target, stage, tbytes, cudaMemcpyHostToDevice, ctx->stream));
    ZI_CUDA(cudaMemsetAsync(&s.ws->best, 0xff, sizeof(unsigned long long), ctx->stream));
    const size_t smem = ((KK * C + 3) & ~size_t(3)) + KK * C * sizeof(int) + 16;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(ctx->num_sms) * 8));
    static const bool scalar = std::getenv("ZI_BRUTE_SCALAR") != nullptr;
    static const bool quad = std::getenv("ZI_BRUTE_QUAD") != nullptr;  // A/B: the 4-entry kernel
    if (n > 0 && C == 1 && !scalar && !quad) {
        const unsigned g8 = static_cast<unsigned>(std::min<uint64_t>((n + 2047) / 2048, static_cast<uint64_t>(ctx->num_sms) * 8));
        ZI_LAUNCH(ctx, "brute_force", k_brute8, g8, 256, ((KK + 3) & ~size_t(3)) * 8 + 16, d_img, w, K, d_dict, n, s.target,
                  norm, &s.ws->best);
    } else if (n > 0 && C == 1 && !scalar) {
        const unsigned g4 = static_cast<unsigned>(std::min<uint64_t>((n + 1023) / 1024, static_cast<uint64_t>(ctx->num_sms) * 8));
        ZI_LAUNCH(ctx, "brute_force", k_brute4, g4, 256, KK * 8 + 16, d_img, w, K, d_dict, n, s.target, norm,
                  &s.ws->best);
    } else if (n > 0) {
        ZI_LAUNCH(ctx, "brute_force", k_brute, grid, 256, smem, d_img, w, C, K, d_dict, n, s.target, norm, &s.ws->best);
    }
    unsigned long long* hb = reinterpret_cast<unsigned long long*>(stage + res_off);
    ZI_CUDA(cudaMemcpyAsync(hb, &s.ws->best, 8, cudaMemcpyDeviceToHost, ctx->stream));
    ZI_CUDA(cudaStreamSynchronize(ctx->stream));
    return *hb;
}

uint64_t brute_force_best(zi_multi_index* mi, const uint8_t* h_tv, const uint8_t* h_tk, int norm) {
    return brute_force_scan(mi->ctx, mi->image.p, mi->w, mi->C, mi->K, mi->dict.p + mi->row_begin, mi->n, h_tv, h_tk,
                            norm, mi->qscratch, mi->hstage);
}

// make_query (proj/src/builder.cpp:110-127) for one layout model: unknown layout pixels take the
// mean (xc = +0.0 exactly), then the canonical fp64 fma chain per dim and the quantiser.
__global__ void __launch_bounds__(256) k_make_query(const uint8_t* __restrict__ target, int K, int C,
                                                    const int32_t* __restrict__ local, int m,
                                                    const double* __restrict__ mean, const double* __restrict__ comp,
                                                    const unsigned long long* __restrict__ minmax, int D,
                                                    uint8_t* __restrict__ out) {
    extern __shared__ double s_xc[];
    const int KK = K * K, mc = m * C;
    const uint8_t* tv = target;
    const uint8_t* tk = target + KK * C;
    for (int j = threadIdx.x; j < mc; j += blockDim.x) {
        const int l = local[j / C];
        const double mj = mean[j];
        const double x = tk[l] ? static_cast<double>(tv[l * C + j % C]) : mj;
        s_xc[j] = __dsub_rn(x, mj);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
        double y = 0.0;
        for (int j = 0; j < mc; ++j) y = __fma_rn(comp[static_cast<size_t>(j) * D + d], s_xc[j], y);
        out[d] = quantize_rn(ordered_to_double_hd(minmax[d]), ordered_to_double_hd(minmax[D + d]), y);
    }
}

void make_query(zi_ctx* ctx, const uint8_t* h_tv, const uint8_t* h_tk, int K, int C, const int32_t* d_local, int m,
                const double* d_mean, const double* d_comp, const unsigned long long* d_minmax, int D, uint8_t* h_out,
                dbuf<uint8_t>& scratch, hbuf<uint8_t>& hstage) {
    const size_t KK = static_cast<size_t>(K) * K;
    const size_t tbytes = KK * C + KK;
    const size_t out_off = (tbytes + 255) & ~size_t(255);
    uint8_t* stage = hstage.ensure(out_off + 64);
    uint8_t* dev = scratch.ensure(out_off + 64);
    std::memcpy(stage, h_tv, KK * C);
    std::memcpy(stage + KK * C, h_tk, KK);
    ZI_CUDA(cudaMemcpyAsync(dev, stage, tbytes, cudaMemcpyHostToDevice, ctx->stream));
    ZI_LAUNCH(ctx, "make_query", k_make_query, 1, 256, static_cast<size_t>(m) * C * sizeof(double), dev, K, C, d_local,
              m, d_mean, d_comp, d_minmax, D, dev + out_off);
    ZI_CUDA(cudaMemcpyAsync(stage + out_off, dev + out_off, D, cudaMemcpyDeviceToHost, ctx->stream));
    ZI_CUDA(cudaStreamSynchronize(ctx->stream));
    std::memcpy(h_out, stage + out_off, D);
}

// masked-cost refine of a caller-given candidate list (query_best_patch's refine step,
// proj/src/engine.cpp:195-212): the sharded query merges the per-shard k-NN lists on the host
// and refines the global top-k here.  Returns packed (cost<<32 | key), UINT64_MAX if empty.
uint64_t refine_candidates(zi_multi_index* mi, const uint8_t* h_tv, const uint8_t* h_tk, const uint64_t* h_cands,
                           uint32_t count, int norm) {
    zi_ctx* ctx = mi->ctx;
    if (count == 0) return ~0ull;
    const size_t KK = static_cast<size_t>(mi->K) * mi->K;
    const size_t tbytes = KK * mi->C + KK;
    const query_scratch s = carve(mi->qscratch, ctx, 1, count, tbytes);
    mi->qws_clean = false;  // the fill-loop workspace is reused below
    const size_t res_off = (tbytes + 255) & ~size_t(255);
    const size_t list_off = res_off + ((sizeof(qws) + 255) & ~size_t(255));
    uint8_t* stage = mi->hstage.ensure(list_off + count * sizeof(uint64_t));
    std::memcpy(stage, h_tv, KK * mi->C);
    std::memcpy(stage + KK * mi->C, h_tk, KK);
    std::memcpy(stage + list_off, h_cands, count * sizeof(uint64_t));
    qws* hq = reinterpret_cast<qws*>(stage + res_off);
    std::memset(hq, 0, sizeof(qws));
    hq->count = count;
    hq->best = ~0ull;
    ZI_CUDA(cudaMemcpyAsync(s.target, stage, tbytes, cudaMemcpyHostToDevice, ctx->stream));
    ZI_CUDA(cudaMemcpyAsync(s.ws, hq, sizeof(qws), cudaMemcpyHostToDevice, ctx->stream));
    ZI_CUDA(cudaMemcpyAsync(s.out, stage + list_off, count * sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream));
    const size_t rsmem = ((KK * mi->C + 1) & ~size_t(1)) + (KK + 16) * sizeof(uint16_t) + kRefineSlots * sizeof(uint32_t) + 32;
    ZI_LAUNCH(ctx, "refine", k_refine, 1, 1024, rsmem, mi->image.p, mi->w, mi->C, mi->K, s.target, s.ws, s.out, norm);
    ZI_CUDA(cudaMemcpyAsync(hq, s.ws, sizeof(qws), cudaMemcpyDeviceToHost, ctx->stream));
    ZI_CUDA(cudaStreamSynchronize(ctx->stream));
    return hq->best;
}

}  // namespace zi
