// k_ssort.cu -- K4': the Morton sort as a two-level splitter (sample) sort.  Replaces the std::sort
// of zcurve_index::from_descriptors (proj/src/zcurve.cpp:116-125).
//
// The records of G equal-sized groups (the 8 layouts of a build, group-major, or one index) are
// ordered inside each group by the composite key (Morton key words, most significant word
// first, then the payload).  The payload is unique inside a group (row id, or the packed patch
// key) and arrives ascending, so this is exactly the reference's comparator (morton_less, then
// packed key) and a stable sort on the Morton key alone gives it.
//
//   1. samples: 16 per fine bucket at regular positions, sorted (onesweep LSD); every 16th is a
//      fine splitter (B - 1 per group, buckets of ~1.5k records), every F-th fine splitter a
//      coarse one (B1 = B / F <= 256 per group);
//   2. level 1: per 32768-record tile the coarse bucket of every record (binary search over the
//      splitters in shared memory) -> per-tile histograms -> column / bucket scans -> a STABLE
//      scatter (warp-ordered ranks in 4096-record sub-tiles);
//   3. level 2: the same inside every coarse bucket with its F fine splitters (tile table built
//      on the device from the coarse sizes);
//   4. local: one CTA per fine bucket sorts it in shared memory by the Morton key with the
//      position (= payload order) as tie-break: a bitonic sort of (key suffix << 12 | position)
//      when the key bits that vary inside the bucket fit 52 bits, a stable byte-LSD otherwise.
//      Buckets above the CTA capacity (composite splitters keep buckets balanced even with heavy
//      duplicate keys; never seen) are finished by the global LSD sort on their range.
// Every scatter run is one bucket of one tile (>= ~128 records: coalesced).  HBM traffic per
// record: 5 reads + 3 writes (two count + scatter levels, one local pass) against 2 per digit
// pass of the LSD sort (8 Morton bytes + the layout digit + a histogram read at cfg4).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"

namespace zi {

// the onesweep LSD sort (k_sort.cu), for the samples and for oversized buckets
void radix_sort_words(zi_ctx* ctx, uint32_t** words, int nw, uint64_t n, const std::vector<int2>& passes,
                      const uint32_t* hist_host, bool device_bases, uint32_t** result);

namespace {

constexpr int kSsThreads = 512;
constexpr int kSsLocalThreads = 512;
constexpr int kSsLocalWarps = kSsLocalThreads / 32;
constexpr uint32_t kSsMaxOver = 1000;

template <int NW>
struct ss_words {
    uint32_t* w[NW];
};

// composite order: key words most significant first (word NW-2 is the top Morton word), then
// the payload (word NW-1)
template <int NW>
__device__ __forceinline__ bool rec_less(const uint32_t (&a)[NW], const uint32_t* b) {
#pragma unroll
    for (int k = NW - 2; k >= 0; --k)
        if (a[k] != b[k]) return a[k] < b[k];
    return a[NW - 1] < b[NW - 1];
}

// number of splitters <= rec (splitters ascending, AoS NW words each)
template <int NW>
__device__ __forceinline__ int bucket_of(const uint32_t (&rec)[NW], const uint32_t* spl, int nspl) {
    int lo = 0, hi = nspl;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (rec_less<NW>(rec, spl + mid * NW)) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

__device__ inline void block_bitonic_sort_s2(unsigned long long* a, int n) {
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

// sample j of group g: the record at row floor((j + 1/2) n / S), copied SoA
template <int NW>
__global__ void k_ss_sample(ss_words<NW> in, uint64_t n, int G, uint32_t S, ss_words<NW> out) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<uint64_t>(G) * S) return;
    const uint64_t g = i / S, j = i % S;
    const uint64_t row = (2 * j + 1) * n / (2ull * S);
#pragma unroll
    for (int k = 0; k < NW; ++k) out.w[k][i] = in.w[k][g * n + row];
}

// splitter b (1..B-1) of group g = the (b*s)-th smallest sample of g, AoS
template <int NW>
__global__ void k_ss_splitters(ss_words<NW> samp, int G, uint32_t S, int B, uint32_t* __restrict__ spl) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= G * (B - 1)) return;
    const int g = i / (B - 1), b = i % (B - 1) + 1;
    const uint64_t src = static_cast<uint64_t>(g) * S + static_cast<uint64_t>(b) * (S / B);
#pragma unroll
    for (int k = 0; k < NW; ++k) spl[static_cast<size_t>(i) * NW + k] = samp.w[k][src];
}

// ---------------------------------------------------------------------------- two-level version
// Level 1 splits every group into B1 <= 256 coarse buckets, level 2 every coarse bucket into
// F <= 256 fine buckets; both scatters are STABLE (warp-ordered ranks, per-tile offsets from a
// counting pass), so a fine bucket holds its records in payload order and the local sort only
// needs the Morton key, ties broken by position.  Every run a scatter writes is one bucket of one
// tile: with <= 256 buckets and 32768-record tiles the runs are >= 128 records long (coalesced).
constexpr int kS2Tile = 32768;
constexpr int kS2Sub = kSsThreads * 8;  // records per scatter sub-tile (8 per thread)
constexpr int kS2Samples = 16;          // samples per fine bucket

template <int NW>
__host__ __device__ constexpr int s2_cap() {
    return NW <= 4 ? 4096 : 2048;
}

// tile -> (bucket set q, first record, records): level 1 tiles are uniform per group; level 2
// tiles come from the prefix table tile_base over the coarse buckets
struct s2_tile {
    int q;
    uint64_t r0, len;
};

__device__ __forceinline__ s2_tile s2_tile_of(int level, int tile, int tpg, uint64_t n, const uint32_t* tile_base,
                                              int nq, const uint64_t* qstart, const uint32_t* qlen) {
    s2_tile t;
    if (level == 1) {
        t.q = tile / tpg;
        const uint64_t off = static_cast<uint64_t>(tile % tpg) * kS2Tile;
        t.r0 = static_cast<uint64_t>(t.q) * n + off;
        t.len = off < n ? (n - off < kS2Tile ? n - off : kS2Tile) : 0;
    } else {
        int lo = 0, hi = nq;  // last q with tile_base[q] <= tile
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (tile_base[mid] <= static_cast<uint32_t>(tile)) lo = mid;
            else hi = mid;
        }
        t.q = lo;
        const uint64_t off = static_cast<uint64_t>(tile - static_cast<int>(tile_base[lo])) * kS2Tile;
        const uint64_t L = qlen[lo];
        t.r0 = qstart[lo] + off;
        t.len = off < L ? (L - off < kS2Tile ? L - off : kS2Tile) : 0;
    }
    return t;
}

// the splitters a tile searches: level 1 = the group's B1-1 coarse splitters; level 2 = the fine
// splitters inside coarse bucket q (nf-1 of them)
template <int NW>
__device__ __forceinline__ int s2_load_splitters(int level, int q, int B, int B1, int F, const uint32_t* spl_c,
                                                 const uint32_t* spl_f, uint32_t* s_spl) {
    int cnt, g, c;
    const uint32_t* src;
    if (level == 1) {
        cnt = B1 - 1;
        src = spl_c + static_cast<size_t>(q) * (B1 - 1) * NW;
    } else {
        g = q / B1;
        c = q % B1;
        const int f0 = c * F;
        const int nf = B - f0 < F ? B - f0 : F;
        cnt = nf - 1;
        src = spl_f + (static_cast<size_t>(g) * (B - 1) + f0) * NW;
    }
    for (int i = threadIdx.x; i < cnt * NW; i += blockDim.x) s_spl[i] = src[i];
    return cnt;
}

// MODE 0: per-tile bucket histogram; MODE 1: stable scatter to the bucket cursors
template <int NW, int MODE>
__global__ void __launch_bounds__(kSsThreads) k_s2_pass(ss_words<NW> in, ss_words<NW> out, int level, uint64_t n,
                                                        int tpg, int ntiles, const uint32_t* __restrict__ tile_base,
                                                        int nq, const uint64_t* __restrict__ qstart,
                                                        const uint32_t* __restrict__ qlen, int B, int B1, int F,
                                                        const uint32_t* __restrict__ spl_c,
                                                        const uint32_t* __restrict__ spl_f, int NB,
                                                        uint32_t* __restrict__ hist,
                                                        const uint64_t* __restrict__ bstart) {
    __shared__ uint32_t s_spl[255 * 9];
    __shared__ uint32_t s_wcnt[kSsThreads / 32][256];
    __shared__ uint32_t s_cur[256], s_tot[256];
    const int tile = blockIdx.x;
    if (tile >= ntiles) return;
    const s2_tile T = s2_tile_of(level, tile, tpg, n, tile_base, nq, qstart, qlen);
    const int nspl = s2_load_splitters<NW>(level, T.q, B, B1, F, spl_c, spl_f, s_spl);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int b = tid; b < NB; b += kSsThreads) {
        if (MODE == 0) s_cur[b] = 0;
        else s_cur[b] = static_cast<uint32_t>(bstart[static_cast<size_t>(T.q) * NB + b] + hist[static_cast<size_t>(tile) * NB + b]);
    }
    __syncthreads();
    if (MODE == 0) {
        constexpr int U = 4;
        for (uint64_t r = tid; r < T.len; r += static_cast<uint64_t>(kSsThreads) * U) {
            uint32_t rec[U][NW];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint64_t i = r + static_cast<uint64_t>(u) * kSsThreads;
                if (i < T.len)
#pragma unroll
                    for (int k = 0; k < NW; ++k) rec[u][k] = in.w[k][T.r0 + i];
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (r + static_cast<uint64_t>(u) * kSsThreads < T.len) atomicAdd(&s_cur[bucket_of<NW>(rec[u], s_spl, nspl)], 1u);
        }
        __syncthreads();
        for (int b = tid; b < NB; b += kSsThreads) hist[static_cast<size_t>(tile) * NB + b] = s_cur[b];
        return;
    }
    const uint32_t lt = (1u << lane) - 1u;
    for (uint64_t s0 = 0; s0 < T.len; s0 += kS2Sub) {
        for (int i = tid; i < (kSsThreads / 32) * 256; i += kSsThreads) (&s_wcnt[0][0])[i] = 0;
        __syncthreads();
        uint32_t rec[8][NW];
        uint32_t bk[8], rk[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {  // warp w owns the 256 consecutive records [w*256, w*256+256)
            const uint64_t i = s0 + static_cast<uint64_t>(warp) * 256 + r * 32 + lane;
            const bool ok = i < T.len;
#pragma unroll
            for (int k = 0; k < NW; ++k) rec[r][k] = ok ? in.w[k][T.r0 + i] : 0u;
            bk[r] = ok ? static_cast<uint32_t>(bucket_of<NW>(rec[r], s_spl, nspl)) : 256u;
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {  // stable rank inside the warp, in record order
            const uint32_t d = bk[r];
            const uint32_t peers = __match_any_sync(0xffffffffu, d);
            uint32_t old = 0;
            if (d < 256u) old = s_wcnt[warp][d];
            __syncwarp();
            if (d < 256u && (peers >> lane) == 1u) s_wcnt[warp][d] = old + __popc(peers);
            __syncwarp();
            rk[r] = old + __popc(peers & lt);
        }
        __syncthreads();
        for (int b = tid; b < NB; b += kSsThreads) {  // warp-exclusive offsets per bucket
            uint32_t run = 0;
#pragma unroll
            for (int w = 0; w < kSsThreads / 32; ++w) {
                const uint32_t c = s_wcnt[w][b];
                s_wcnt[w][b] = run;
                run += c;
            }
            s_tot[b] = run;
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const uint32_t b = bk[r];
            if (b < 256u) {
                const uint32_t pos = s_cur[b] + s_wcnt[warp][b] + rk[r];
#pragma unroll
                for (int k = 0; k < NW; ++k) out.w[k][pos] = rec[r][k];
            }
        }
        __syncthreads();
        for (int b = tid; b < NB; b += kSsThreads) s_cur[b] += s_tot[b];
        __syncthreads();
    }
}

// per bucket set q: exclusive prefix over its tiles (in place) and the bucket totals
__global__ void k_s2_colscan(uint32_t* __restrict__ hist, int nq, int NB, int level, int tpg,
                             const uint32_t* __restrict__ tile_base, const uint32_t* __restrict__ ntile_q,
                             uint32_t* __restrict__ total) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nq * NB) return;
    const int q = i / NB, b = i % NB;
    const int t0 = level == 1 ? q * tpg : static_cast<int>(tile_base[q]);
    const int nt = level == 1 ? tpg : static_cast<int>(ntile_q[q]);
    uint32_t run = 0;
    for (int t = 0; t < nt; ++t) {
        uint32_t* p = hist + static_cast<size_t>(t0 + t) * NB + b;
        const uint32_t c = *p;
        *p = run;
        run += c;
    }
    total[i] = run;
}

// per bucket set q: bucket starts = base[q] + exclusive prefix of its totals (NB <= 256)
__global__ void __launch_bounds__(256) k_s2_bscan(const uint32_t* __restrict__ total, int NB,
                                                  const uint64_t* __restrict__ base, uint64_t n,
                                                  uint64_t* __restrict__ bstart) {
    __shared__ uint32_t s_w[8];
    const int q = blockIdx.x, b = threadIdx.x, lane = b & 31, warp = b >> 5;
    const uint32_t v = b < NB ? total[static_cast<size_t>(q) * NB + b] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    uint32_t wp = 0;
    for (int w = 0; w < warp; ++w) wp += s_w[w];
    const uint64_t b0 = base ? base[q] : static_cast<uint64_t>(q) * n;
    if (b < NB) bstart[static_cast<size_t>(q) * NB + b] = b0 + wp + x - v;
}

// level-2 tile table over the coarse buckets: ntile[q] = ceil(len / tile), tile_base = prefix
__global__ void __launch_bounds__(1024) k_s2_tiles(const uint32_t* __restrict__ qlen, int nq,
                                                   uint32_t* __restrict__ ntile, uint32_t* __restrict__ tile_base,
                                                   uint32_t* __restrict__ ntiles_total) {
    __shared__ uint32_t s_w[32];
    __shared__ uint32_t s_carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (int c0 = 0; c0 < nq; c0 += 1024) {
        const int q = c0 + tid;
        const uint32_t v = q < nq ? (qlen[q] + kS2Tile - 1) / kS2Tile : 0u;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_w[warp] = x;
        __syncthreads();
        uint32_t wp = 0;
        for (int w = 0; w < warp; ++w) wp += s_w[w];
        const uint32_t carry = s_carry;
        if (q < nq) {
            ntile[q] = v;
            tile_base[q] = carry + wp + x - v;
        }
        __syncthreads();
        if (tid == 1023) s_carry = carry + wp + x;
        __syncthreads();
    }
    if (tid == 0) *ntiles_total = s_carry;
}

// coarse splitter c (1..B1-1) of group g = the fine splitter that opens fine bucket c*F
template <int NW>
__global__ void k_s2_coarse(const uint32_t* __restrict__ spl_f, int G, int B, int B1, int F, uint32_t* __restrict__ spl_c) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= G * (B1 - 1)) return;
    const int g = i / (B1 - 1), c = i % (B1 - 1) + 1;
#pragma unroll
    for (int k = 0; k < NW; ++k)
        spl_c[static_cast<size_t>(i) * NW + k] = spl_f[(static_cast<size_t>(g) * (B - 1) + c * F - 1) * NW + k];
}

// one CTA per fine bucket (records in payload order after the stable scatters): sort by the
// Morton key with the position as tie-break.  When the key bits that vary inside the bucket fit
// 52 bits the (key suffix << 12 | position) words are bitonic-sorted; otherwise a stable LSD over
// the varying key bytes on a u16 permutation.  The bucket is rewritten in place.
template <int NW>
__global__ void __launch_bounds__(kSsLocalThreads) k_s2_local(ss_words<NW> io, const uint64_t* __restrict__ bstart,
                                                             const uint32_t* __restrict__ total,
                                                             uint64_t* __restrict__ over, uint32_t* __restrict__ nover) {
    constexpr int cap = s2_cap<NW>();
    constexpr int W = NW - 1;
    constexpr int kMaxRounds = (cap + kSsLocalWarps * 32 - 1) / (kSsLocalWarps * 32);
    extern __shared__ unsigned long long s_key[];            // cap sort words
    uint32_t* s_w = reinterpret_cast<uint32_t*>(s_key + cap);  // NW * cap (SoA)
    uint16_t* s_cur = reinterpret_cast<uint16_t*>(s_w + static_cast<size_t>(NW) * cap);
    uint16_t* s_nxt = s_cur + cap;
    __shared__ uint32_t s_hist[kSsLocalWarps][256];
    __shared__ uint32_t s_dstart[256];
    __shared__ uint32_t s_wsum[kSsLocalWarps];
    __shared__ uint32_t s_and[NW], s_or[NW];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t start = bstart[blockIdx.x];
    const int len = static_cast<int>(total[blockIdx.x]);
    if (len <= 1) return;
    if (len > cap) {
        if (tid == 0) {
            const uint32_t slot = atomicAdd(nover, 1u);
            if (slot < kSsMaxOver) {
                over[2 * slot] = start;
                over[2 * slot + 1] = static_cast<uint64_t>(len);
            }
        }
        return;
    }
    if (tid < NW) {
        s_and[tid] = 0xffffffffu;
        s_or[tid] = 0u;
    }
    __syncthreads();
    uint32_t wand[NW], wor[NW];
#pragma unroll
    for (int k = 0; k < NW; ++k) {
        wand[k] = 0xffffffffu;
        wor[k] = 0u;
    }
    for (int j = tid; j < len; j += kSsLocalThreads) {
#pragma unroll
        for (int k = 0; k < NW; ++k) {
            const uint32_t v = io.w[k][start + j];
            s_w[k * cap + j] = v;
            wand[k] &= v;
            wor[k] |= v;
        }
    }
#pragma unroll
    for (int k = 0; k < NW; ++k) {
        atomicAnd(&s_and[k], wand[k]);
        atomicOr(&s_or[k], wor[k]);
    }
    __syncthreads();
    // highest key bit that varies (bit 32k + 31 - clz of word k)
    int top = -1;
#pragma unroll
    for (int k = W - 1; k >= 0; --k) {
        const uint32_t x = s_and[k] ^ s_or[k];
        if (top < 0 && x != 0u) top = 32 * k + 31 - __clz(x);
    }
    if (top < 0) return;  // one key: already in payload order
    if (top < 52) {
        const unsigned long long mask = (1ull << (top + 1)) - 1ull;
        int sz = 32;
        while (sz < len) sz <<= 1;
        for (int j = tid; j < sz; j += kSsLocalThreads) {
            unsigned long long key = ~0ull;
            if (j < len) {
                const unsigned long long lo = s_w[j];
                const unsigned long long hi = W > 1 ? s_w[cap + j] : 0u;
                key = ((((hi << 32) | lo) & mask) << 12) | static_cast<unsigned long long>(j);
            }
            s_key[j] = key;
        }
        __syncthreads();
        block_bitonic_sort_s2(s_key, sz);
        for (int j = tid; j < len; j += kSsLocalThreads) {
            const int src = static_cast<int>(s_key[j] & 0xfffull);
#pragma unroll
            for (int k = 0; k < NW; ++k) io.w[k][start + j] = s_w[k * cap + src];
        }
        return;
    }
    // wide keys: stable LSD over the varying key bytes (the payload order is already right)
    for (int j = tid; j < len; j += kSsLocalThreads) s_cur[j] = static_cast<uint16_t>(j);
    __syncthreads();
    const int CH = ((len + kSsLocalWarps - 1) / kSsLocalWarps + 31) & ~31;
    const int nround = CH / 32;
    const uint32_t lt = (1u << lane) - 1u;
    for (int q = 0; q < 4 * W; ++q) {
        const int wk = q >> 2;
        const int sh = (q & 3) * 8;
        if ((((s_and[wk] ^ s_or[wk]) >> sh) & 0xffu) == 0u) continue;
        for (int i = tid; i < kSsLocalWarps * 256; i += kSsLocalThreads) (&s_hist[0][0])[i] = 0;
        __syncthreads();
        uint32_t dg[kMaxRounds], rk[kMaxRounds];
#pragma unroll
        for (int r = 0; r < kMaxRounds; ++r) {
            if (r < nround) {
                const int i = warp * CH + r * 32 + lane;
                uint32_t d = 256u;
                if (i < len) d = (s_w[wk * cap + s_cur[i]] >> sh) & 0xffu;
                const uint32_t peers = __match_any_sync(0xffffffffu, d);
                uint32_t old = 0;
                if (d < 256u) old = s_hist[warp][d];
                __syncwarp();
                if (d < 256u && (peers >> lane) == 1u) s_hist[warp][d] = old + __popc(peers);
                __syncwarp();
                dg[r] = d;
                rk[r] = old + __popc(peers & lt);
            }
        }
        __syncthreads();
        if (tid < 256) {
            const int d = tid;
            uint32_t run = 0;
#pragma unroll
            for (int w = 0; w < kSsLocalWarps; ++w) {
                const uint32_t c = s_hist[w][d];
                s_hist[w][d] = run;
                run += c;
            }
            uint32_t x = run;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) s_wsum[warp] = x;
            s_dstart[d] = x - run;
        }
        __syncthreads();
        if (tid < 256) {
            uint32_t wp = 0;
            for (int w = 0; w < (tid >> 5); ++w) wp += s_wsum[w];
            s_dstart[tid] += wp;
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < kMaxRounds; ++r) {
            if (r < nround) {
                const int i = warp * CH + r * 32 + lane;
                if (dg[r] < 256u) s_nxt[s_dstart[dg[r]] + s_hist[warp][dg[r]] + rk[r]] = s_cur[i];
            }
        }
        __syncthreads();
        uint16_t* tmp = s_cur;
        s_cur = s_nxt;
        s_nxt = tmp;
    }
    for (int j = tid; j < len; j += kSsLocalThreads) {
        const int src = s_cur[j];
#pragma unroll
        for (int k = 0; k < NW; ++k) io.w[k][start + j] = s_w[k * cap + src];
    }
}

template <int NW>
void sample_sort_t(zi_ctx* ctx, uint32_t* const* words, uint64_t n, int G, int D, bool group_in_payload,
                   uint32_t** out) {
    const uint64_t N = static_cast<uint64_t>(G) * n;
    constexpr int cap = s2_cap<NW>();
    static const int tgt_env = [] { const char* e = std::getenv("ZI_SSORT_TARGET"); return e ? std::atoi(e) : 0; }();
    const uint64_t target = tgt_env > 0 ? static_cast<uint64_t>(tgt_env) : static_cast<uint64_t>(cap) * 3 / 8;
    const int B = static_cast<int>(std::max<uint64_t>(1, (n + target - 1) / target));
    const int F = std::max(1, std::min(256, (B + 255) / 256 > 64 ? (B + 255) / 256 : 64));
    const int B1 = (B + F - 1) / F;
    if (B1 > 256) throw error(ZI_E_INVALID, "sample sort: group too large");
    const uint32_t S = static_cast<uint32_t>(B) * kS2Samples;
    const int tpg = static_cast<int>((n + kS2Tile - 1) / kS2Tile);
    const int nq2 = G * B1;                                        // coarse buckets
    const int tiles1 = G * tpg;
    const int tiles2_max = static_cast<int>(N / kS2Tile) + nq2 + 1;
    ss_words<NW> A{}, Bw{};
    for (int k = 0; k < NW; ++k) A.w[k] = words[k];
    // scratch (ctx->ss_buf): alt records | samples | fine + coarse splitters | hist1 | hist2 |
    // totals / starts | tile table | overflow list
    const size_t n_alt = static_cast<size_t>(NW) * N;
    const size_t n_samp = static_cast<size_t>(NW) * G * S;
    const size_t n_splf = static_cast<size_t>(G) * (B - 1 > 0 ? B - 1 : 1) * NW;
    const size_t n_splc = static_cast<size_t>(G) * (B1 - 1 > 0 ? B1 - 1 : 1) * NW;
    const size_t n_h1 = static_cast<size_t>(tiles1) * B1;
    const size_t n_h2 = static_cast<size_t>(tiles2_max) * F;
    const size_t n_t1 = static_cast<size_t>(nq2), n_t2 = static_cast<size_t>(nq2) * F;
    size_t words_total = n_alt + n_samp + n_splf + n_splc + n_h1 + n_h2 + n_t1 + n_t2 + 2 * nq2 + 64;
    words_total += 2 * (n_t1 + n_t2) + 8;  // u64 starts
    words_total += 2 * 2 * 1024 + 64;      // overflow list
    uint32_t* p = ctx->ss_buf.ensure(words_total);
    auto take32 = [&](size_t cnt) { uint32_t* r = p; p += cnt; return r; };
    auto take64 = [&](size_t cnt) {
        p = reinterpret_cast<uint32_t*>((reinterpret_cast<uintptr_t>(p) + 7) & ~uintptr_t(7));
        uint64_t* r = reinterpret_cast<uint64_t*>(p);
        p += 2 * cnt;
        return r;
    };
    uint32_t* alt = take32(n_alt);
    for (int k = 0; k < NW; ++k) Bw.w[k] = alt + static_cast<size_t>(k) * N;
    uint32_t* samp = take32(n_samp);
    uint32_t* spl_f = take32(n_splf);
    uint32_t* spl_c = take32(n_splc);
    uint32_t* hist1 = take32(n_h1);
    uint32_t* hist2 = take32(n_h2);
    uint32_t* tot1 = take32(n_t1);
    uint32_t* tot2 = take32(n_t2);
    uint32_t* ntile2 = take32(nq2);
    uint32_t* tbase2 = take32(nq2 + 8);
    uint32_t* ntot2 = tbase2 + nq2;
    uint64_t* cstart = take64(n_t1);
    uint64_t* fstart = take64(n_t2);
    uint64_t* over = take64(2 * 1024);
    uint32_t* nover = reinterpret_cast<uint32_t*>(over + 2 * kSsMaxOver + 2);
    ZI_CUDA(cudaMemsetAsync(nover, 0, sizeof(uint32_t), ctx->stream));

    ss_words<NW> fin = A;  // where the fine buckets end up
    if (B > 1) {
        ss_words<NW> sw{};
        for (int k = 0; k < NW; ++k) sw.w[k] = samp + static_cast<size_t>(k) * G * S;
        const uint64_t ns = static_cast<uint64_t>(G) * S;
        ZI_LAUNCH(ctx, "ssort_sample", k_ss_sample<NW>, static_cast<unsigned>((ns + 255) / 256), 256, 0, A, n, G, S, sw);
        std::vector<int2> passes;
        for (int q = 0; q < D; ++q) passes.push_back(make_int2(q >> 2, (q & 3) * 8));
        if (G > 1 && group_in_payload) passes.push_back(make_int2(NW - 1, 29));
        uint32_t* sp[kSortMaxWords];
        uint32_t* sres[kSortMaxWords];
        for (int k = 0; k < NW; ++k) sp[k] = sw.w[k];
        radix_sort_words(ctx, sp, NW, ns, passes, nullptr, true, sres);
        ss_words<NW> ss{};
        for (int k = 0; k < NW; ++k) ss.w[k] = sres[k];
        ZI_LAUNCH(ctx, "ssort_splitters", k_ss_splitters<NW>, static_cast<unsigned>((G * (B - 1) + 255) / 256), 256, 0,
                  ss, G, S, B, spl_f);
        // level 1: G groups -> B1 coarse buckets each
        ss_words<NW> src = A, dst = Bw;
        if (B1 > 1) {
            ZI_LAUNCH(ctx, "ssort_splitters", k_s2_coarse<NW>, static_cast<unsigned>((G * (B1 - 1) + 255) / 256), 256, 0,
                      spl_f, G, B, B1, F, spl_c);
            ZI_LAUNCH(ctx, "ssort_count", (k_s2_pass<NW, 0>), static_cast<unsigned>(tiles1), kSsThreads, 0, A, Bw, 1, n,
                      tpg, tiles1, tbase2, G, cstart, tot1, B, B1, F, spl_c, spl_f, B1, hist1, cstart);
            ZI_LAUNCH(ctx, "ssort_colscan", k_s2_colscan, static_cast<unsigned>((G * B1 + 255) / 256), 256, 0, hist1, G,
                      B1, 1, tpg, tbase2, ntile2, tot1);
            ZI_LAUNCH(ctx, "ssort_bscan", k_s2_bscan, static_cast<unsigned>(G), 256, 0, tot1, B1,
                      static_cast<const uint64_t*>(nullptr), n, cstart);
            ZI_LAUNCH(ctx, "ssort_scatter", (k_s2_pass<NW, 1>), static_cast<unsigned>(tiles1), kSsThreads, 0, A, Bw, 1,
                      n, tpg, tiles1, tbase2, G, cstart, tot1, B, B1, F, spl_c, spl_f, B1, hist1, cstart);
            src = Bw;
            dst = A;
        } else {  // one coarse bucket per group: the whole group
            std::vector<uint64_t> hs(G);
            std::vector<uint32_t> ht(G);
            for (int g = 0; g < G; ++g) {
                hs[g] = static_cast<uint64_t>(g) * n;
                ht[g] = static_cast<uint32_t>(n);
            }
            ZI_CUDA(cudaMemcpyAsync(cstart, hs.data(), G * sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream));
            ZI_CUDA(cudaMemcpyAsync(tot1, ht.data(), G * sizeof(uint32_t), cudaMemcpyHostToDevice, ctx->stream));
            ZI_CUDA(cudaStreamSynchronize(ctx->stream));  // pageable sources
        }
        // level 2: every coarse bucket -> <= F fine buckets (tile table from the coarse sizes)
        ZI_LAUNCH(ctx, "ssort_tiles", k_s2_tiles, 1, 1024, 0, tot1, nq2, ntile2, tbase2, ntot2);
        ZI_LAUNCH(ctx, "ssort_count", (k_s2_pass<NW, 0>), static_cast<unsigned>(tiles2_max), kSsThreads, 0, src, dst, 2,
                  n, tpg, tiles2_max, tbase2, nq2, cstart, tot1, B, B1, F, spl_c, spl_f, F, hist2, fstart);
        ZI_LAUNCH(ctx, "ssort_colscan", k_s2_colscan, static_cast<unsigned>((nq2 * F + 255) / 256), 256, 0, hist2, nq2, F,
                  2, tpg, tbase2, ntile2, tot2);
        ZI_LAUNCH(ctx, "ssort_bscan", k_s2_bscan, static_cast<unsigned>(nq2), 256, 0, tot2, F,
                  static_cast<const uint64_t*>(cstart), n, fstart);
        ZI_LAUNCH(ctx, "ssort_scatter", (k_s2_pass<NW, 1>), static_cast<unsigned>(tiles2_max), kSsThreads, 0, src, dst, 2,
                  n, tpg, tiles2_max, tbase2, nq2, cstart, tot1, B, B1, F, spl_c, spl_f, F, hist2, fstart);
        fin = dst;
    } else {
        std::vector<uint64_t> hs(G);
        std::vector<uint32_t> ht(G);
        for (int g = 0; g < G; ++g) {
            hs[g] = static_cast<uint64_t>(g) * n;
            ht[g] = static_cast<uint32_t>(n);
        }
        ZI_CUDA(cudaMemcpyAsync(fstart, hs.data(), G * sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream));
        ZI_CUDA(cudaMemcpyAsync(tot2, ht.data(), G * sizeof(uint32_t), cudaMemcpyHostToDevice, ctx->stream));
        ZI_CUDA(cudaStreamSynchronize(ctx->stream));  // pageable sources
    }
    // fine buckets: nq2*F entries (the empty slots of a short last coarse bucket have 0 records)
    const unsigned nfine = B > 1 ? static_cast<unsigned>(nq2) * F : static_cast<unsigned>(G);
    const size_t lsmem = static_cast<size_t>(cap) * 8 + static_cast<size_t>(NW) * cap * 4 + static_cast<size_t>(cap) * 4;
    smem_attr(ctx->device, k_s2_local<NW>, lsmem);
    ZI_LAUNCH(ctx, "ssort_local", k_s2_local<NW>, nfine, kSsLocalThreads, lsmem, fin, fstart, tot2, over, nover);
    for (int k = 0; k < NW; ++k) out[k] = fin.w[k];
    uint32_t hn = 0;
    ZI_CUDA(cudaMemcpyAsync(&hn, nover, sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
    ZI_CUDA(cudaStreamSynchronize(ctx->stream));
    if (hn == 0) return;
    if (hn > kSsMaxOver) throw error(ZI_E_RUNTIME, "sample sort: too many oversized buckets");
    std::vector<uint64_t> ho(2 * hn);
    ZI_CUDA(cudaMemcpyAsync(ho.data(), over, ho.size() * sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
    ZI_CUDA(cudaStreamSynchronize(ctx->stream));
    // stable LSD over the key bytes (the bucket is in payload order)
    std::vector<int2> full;
    for (int q = 0; q < D; ++q) full.push_back(make_int2(q >> 2, (q & 3) * 8));
    static const bool debug = std::getenv("ZI_DEBUG_SORT") != nullptr;
    for (uint32_t i = 0; i < hn; ++i) {
        if (debug)
            std::fprintf(stderr, "sample sort: oversized bucket at %llu (%llu records)\n",
                         static_cast<unsigned long long>(ho[2 * i]), static_cast<unsigned long long>(ho[2 * i + 1]));
        uint32_t* sub[kSortMaxWords];
        for (int k = 0; k < NW; ++k) sub[k] = fin.w[k] + ho[2 * i];
        radix_sort_words(ctx, sub, NW, ho[2 * i + 1], full, nullptr, false, nullptr);
    }
}

}  // namespace

void sample_sort_groups(zi_ctx* ctx, uint32_t* const* words, int nw, uint64_t n, int G, int D, bool group_in_payload,
                        uint32_t** out) {
    if (G > 1 && !group_in_payload) throw error(ZI_E_INVALID, "sample sort: groups need the group id in the payload");
    if (n == 0) {
        for (int k = 0; k < nw; ++k) out[k] = words[k];
        return;
    }
    if (static_cast<uint64_t>(G) * n >= (1ull << 30)) throw error(ZI_E_INVALID, "sample sort: more than 2^30 records");
    switch (nw) {
        case 2: sample_sort_t<2>(ctx, words, n, G, D, group_in_payload, out); break;
        case 3: sample_sort_t<3>(ctx, words, n, G, D, group_in_payload, out); break;
        case 4: sample_sort_t<4>(ctx, words, n, G, D, group_in_payload, out); break;
        case 5: sample_sort_t<5>(ctx, words, n, G, D, group_in_payload, out); break;
        case 6: sample_sort_t<6>(ctx, words, n, G, D, group_in_payload, out); break;
        case 7: sample_sort_t<7>(ctx, words, n, G, D, group_in_payload, out); break;
        case 8: sample_sort_t<8>(ctx, words, n, G, D, group_in_payload, out); break;
        case 9: sample_sort_t<9>(ctx, words, n, G, D, group_in_payload, out); break;
        default: throw error(ZI_E_INVALID, "sample sort: unsupported record width");
    }
}

}  // namespace zi
