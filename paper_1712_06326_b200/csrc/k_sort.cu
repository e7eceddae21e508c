// k_sort.cu -- K4: stable LSD radix sort ("onesweep": one read + one write per 8-bit digit
// pass, chained decoupled look-back for the cross-tile digit prefixes) of (Morton key words,
// payload) records.  Replaces the std::sort of zcurve_index::from_descriptors
// (proj/src/zcurve.cpp:116-125).  Because the reference's comparator is (morton_less, then
// packed key) and every build path feeds keys in ascending packed order, a STABLE sort on
// the Morton key alone reproduces its permutation exactly; when the input
// keys are not ascending, 4 leading passes on the payload establish that order first.
//
// Records are SoA: word k of every record is contiguous (coalesced loads per word).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace zi {

#ifndef ZI_OS_THREADS
#define ZI_OS_THREADS 256
#endif
constexpr int kSortThreads = ZI_OS_THREADS;  // the first 256 threads double as the digits' threads
constexpr int kSortWarps = kSortThreads / 32;
constexpr uint32_t kFlagAgg = 1u << 30, kFlagInc = 2u << 30, kValMask = (1u << 30) - 1;
constexpr int kMaxWords = 9;  // up to 8 Morton key words (D <= 32) + payload

struct sort_words {
    const uint32_t* in[kMaxWords];
    uint32_t* out[kMaxWords];
};

// Histograms of every pass in one read: hist[(q*G + g)*256 + digit] for records in groups of gn
// (group g = records [g*gn, (g+1)*gn)).  Each CTA reads a contiguous chunk (at most a few group
// changes, flushed as they come) with four records per thread in flight.
__global__ void __launch_bounds__(256) k_sort_hist(sort_words io, int npass, const int2* __restrict__ passes,
                                                   uint64_t n, uint64_t gn, int G, uint32_t* __restrict__ hist) {
    extern __shared__ uint32_t s_hist[];  // npass*256
    __shared__ int2 s_pass[40];
    const int nb = npass * 256;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) s_hist[i] = 0;
    if (threadIdx.x < npass) s_pass[threadIdx.x] = passes[threadIdx.x];
    __syncthreads();
    const uint64_t chunk = (n + gridDim.x - 1) / gridDim.x;
    const uint64_t c0 = static_cast<uint64_t>(blockIdx.x) * chunk;
    const uint64_t c1 = c0 + chunk < n ? c0 + chunk : n;
    uint64_t seg = c0;
    while (seg < c1) {  // the part of the chunk inside one group
        const int g = G > 1 ? static_cast<int>(seg / gn) : 0;
        const uint64_t gend = G > 1 ? (static_cast<uint64_t>(g) + 1) * gn : n;
        const uint64_t e = gend < c1 ? gend : c1;
        constexpr int U = 4;
        for (uint64_t b = seg + threadIdx.x; b < e; b += static_cast<uint64_t>(blockDim.x) * U) {
            for (int q = 0; q < npass; ++q) {
                const uint32_t* wq = io.in[s_pass[q].x];
                const int sh = s_pass[q].y;
                uint32_t v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint64_t i = b + static_cast<uint64_t>(u) * blockDim.x;
                    v[u] = i < e ? __ldg(wq + i) : 0u;
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (b + static_cast<uint64_t>(u) * blockDim.x < e) atomicAdd(&s_hist[q * 256 + ((v[u] >> sh) & 0xffu)], 1u);
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < nb; i += blockDim.x) {
            const uint32_t v = s_hist[i];
            if (v) {
                atomicAdd(&hist[(static_cast<size_t>(i >> 8) * G + g) * 256 + (i & 255)], v);
                s_hist[i] = 0;
            }
        }
        __syncthreads();
        seg = e;
    }
}

// exclusive scans of the digit histograms (one block per (pass, group)): the onesweep bases, on
// the device, when the host does not need to see the histograms
__global__ void __launch_bounds__(256) k_sort_bases(const uint32_t* __restrict__ hist, uint32_t* __restrict__ bases) {
    __shared__ uint32_t s_w[8];
    const int q = blockIdx.x, d = threadIdx.x, lane = d & 31, warp = d >> 5;
    const uint32_t c = hist[q * 256 + d];
    uint32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    uint32_t wp = 0;
    for (int w = 0; w < warp; ++w) wp += s_w[w];
    bases[q * 256 + d] = wp + x - c;
}

__device__ __forceinline__ uint32_t os_load(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void os_store(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Decoupled look-back for digit d (one thread per digit, status words tile-major: st[tile*256 + d]).
// The statuses of kLbWin predecessors are loaded together (independent loads, one round trip),
// then summed up to the first inclusive one; an unpublished predecessor is re-read from there.
// A one-at-a-time walk pays one dependent L2 round trip per predecessor, and the number of
// predecessors still holding only their aggregate grows with the tiles in flight.
constexpr int kLbWin = 4;
__device__ __forceinline__ uint32_t lookback(const uint32_t* st, uint32_t tile, uint32_t gfirst, int d) {
    uint32_t prefix = 0;
    int j = static_cast<int>(tile) - 1;
    while (true) {
        uint32_t v[kLbWin];
#pragma unroll
        for (int u = 0; u < kLbWin; ++u)
            v[u] = j - u >= static_cast<int>(gfirst) ? os_load(st + static_cast<size_t>(j - u) * 256 + d) : kFlagInc;
        int used = 0;
        bool done = false;
#pragma unroll
        for (int u = 0; u < kLbWin; ++u) {
            if (used == u && !done) {
                const uint32_t flag = v[u] & ~kValMask;
                if (flag != 0u) {
                    prefix += v[u] & kValMask;
                    ++used;
                    done = flag == kFlagInc;
                }
            }
        }
        if (done) return prefix;
        j -= used;
    }
}

// Build-time knobs of the pass (defaults = the measured best at cfg4, n = 8 x 14.9 M records of
// 3 words; the alternatives are kept for A/B):
//   ZI_OS_RANK  2: KC per-warp histogram chains advanced together (default); 1: one shared atomic
//               per digit group (MIO-bound when the digit is random); 0: one chain, a shared-memory
//               round trip per record slot
//   ZI_OS_KC    chains of ZI_OS_RANK 2 (2; 3 and 4 need more shared memory than four CTAs per SM leave)
//   ZI_OS_MATCH 0: __match_any_sync (default); 1: eight ballots (slower with two chains)
//   ZI_OS_CTAS  CTAs per SM for records of <= 36 words per thread (4); ZI_OS_IT3: records per thread
//               of 3-word records (12); ZI_OS_THREADS: CTA size (256; 512 measured 7 % slower)
#ifndef ZI_OS_MATCH
#define ZI_OS_MATCH 0
#endif
// lanes of the warp holding the same 9-bit value (bit 8 = "no record"): MATCH.ANY is throttled
// in the MIO pipe when the warp holds many distinct values (a random digit: ~30 per warp), eight
// ballots and their mask updates issue on the ALU side
__device__ __forceinline__ uint32_t digit_peers(uint32_t d) {
#if ZI_OS_MATCH == 0
    return __match_any_sync(0xffffffffu, d);
#else
    uint32_t peers = __ballot_sync(0xffffffffu, d < 256u);
    if (d >= 256u) peers = ~peers;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const bool bit = (d >> b) & 1u;
        const uint32_t bal = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? bal : ~bal;
    }
    return peers;
#endif
}

#ifndef ZI_OS_IT3
#define ZI_OS_IT3 12
#endif
#ifndef ZI_OS_KC
#define ZI_OS_KC 2
#endif
#ifndef ZI_OS_HT
#define ZI_OS_HT uint32_t
#endif
#ifndef ZI_OS_CTAS
#define ZI_OS_CTAS 4
#endif
#ifndef ZI_OS_RANK
#define ZI_OS_RANK 2
#endif
// One stable digit pass over a tile of TILE = kSortThreads * IT records.  Records come in groups of gn
// (group-major; G = 1: one group); a group is tiled on its own (tpg tiles) and sorted on its own.
// Where the records of a digit go:
//   MODE 1 (default): offs[tile][d] = global position of the tile's first record of digit d,
//          precomputed by k_lsd_count + the chunk scans (reduce-then-scan: no inter-tile waits);
//   MODE 0: digit_base[g][d] + decoupled look-back over the previous tiles of the group (status).
// All record indices are 32-bit (N < 2^30); the word pointers are offset once per tile.  A
// thread keeps IT records in registers plus one (digit << 16 | warp rank) word per record; the
// records are staged in shared memory in tile-sorted order, then written as runs per digit.
// MODE 1 with DF > 0 (the sort's last pass over the 8-layout records, D = DF): the records are not
// written back but straight into the layout indices -- dim planes (de-interleaved Morton key) and
// the dictionary key of the payload row -- at their final positions (finalize without its read).
template <int NW, int IT, int MODE, int DF = 0>
__global__ void __launch_bounds__(kSortThreads, (NW * IT <= 36 ? ZI_OS_CTAS : 2) * 256 / kSortThreads)
    k_onesweep(sort_words io, int dw, int ds, const uint32_t* __restrict__ digit_base, uint32_t* __restrict__ status,
               uint32_t* __restrict__ tile_ctr, const uint32_t* __restrict__ offs, uint32_t gn, uint32_t tpg,
               const __grid_constant__ final_sink sink) {
    constexpr int TILE = kSortThreads * IT;
    extern __shared__ uint32_t s_stage[];  // NW * TILE
#if ZI_OS_RANK == 2
    // KC independent ranking chains: record slot i of a warp counts into histogram i / (IT / KC)
    constexpr int KC = IT % ZI_OS_KC == 0 ? ZI_OS_KC : 1;
    constexpr int SPC = IT / KC;  // slots per chain
    typedef ZI_OS_HT hist_t;
    __shared__ hist_t s_hist[kSortWarps][KC][256];
#else
    constexpr int KC = 1;
    __shared__ uint32_t s_hist[kSortWarps][256];
#endif
    __shared__ uint32_t s_start[256];
    __shared__ uint32_t s_delta[256];  // global position of the digit's first record, minus its tile start
    __shared__ uint32_t s_warp[8];
    __shared__ uint32_t s_tile;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#if ZI_OS_RANK == 2
    for (int i = tid; i < kSortWarps * KC * 256 * static_cast<int>(sizeof(hist_t)) / 4; i += kSortThreads)
        reinterpret_cast<uint32_t*>(&s_hist[0][0][0])[i] = 0;
#else
    for (int i = tid; i < kSortWarps * 256; i += kSortThreads) (&s_hist[0][0])[i] = 0;
#endif
    if (MODE == 0) {
        if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
        __syncthreads();
    }
    const uint32_t tile = MODE == 0 ? s_tile : blockIdx.x;
    const uint32_t grp = tile / tpg, tig = tile - grp * tpg;  // group, tile inside the group
    const uint32_t t0 = tig * static_cast<uint32_t>(TILE);
    const uint32_t cnt = gn - t0 < static_cast<uint32_t>(TILE) ? gn - t0 : static_cast<uint32_t>(TILE);
    const uint32_t tb = grp * gn + t0;  // global index of the tile's first record
    uint32_t goff = 0;
    if (MODE == 1 && tid < 256) goff = __ldg(offs + static_cast<size_t>(tile) * 256 + tid);  // in flight with the records

    // every word of the tile's records is loaded up front (maximum loads in flight)
    uint32_t rec[IT][NW];
    uint32_t dr[IT];
    const uint32_t w0 = static_cast<uint32_t>(warp * (IT * 32) + lane);
    {
        const uint32_t* src[NW];
#pragma unroll
        for (int k = 0; k < NW; ++k) src[k] = io.in[k] + tb;
#pragma unroll
        for (int i = 0; i < IT; ++i) {
            const uint32_t j = w0 + static_cast<uint32_t>(i * 32);
            const bool ok = j < cnt;
#pragma unroll
            for (int k = 0; k < NW; ++k) rec[i][k] = ok ? __ldg(src[k] + j) : 0u;
        }
    }
    if (MODE == 1) __syncthreads();  // s_hist zeroed
    const uint32_t lt_mask = (1u << lane) - 1u;
    // the digit word through masks (a select chain on rec[i][k] becomes an indexed local-memory
    // load of rec[] after the compiler's select-to-index rewrite)
    uint32_t wmask[NW];
#pragma unroll
    for (int k = 0; k < NW; ++k) wmask[k] = dw == k ? 0xffffffffu : 0u;
#if ZI_OS_RANK == 2
    // Ranking: per record slot the lanes read their digit's running count in the warp's
    // histogram and the highest lane of each digit group adds the group's size.  That read ->
    // write -> next read chain costs a shared-memory round trip per slot; the slots are split over
    // KC histograms (slot i -> chain i / SPC, which keeps the record order: warp, chain, slot)
    // and one step advances all KC chains, so the round trips of KC slots overlap.
#pragma unroll
    for (int s = 0; s < SPC; ++s) {
        uint32_t dd[KC], pp[KC], oo[KC];
#pragma unroll
        for (int c = 0; c < KC; ++c) {
            const int i = c * SPC + s;
            uint32_t x = 0;
#pragma unroll
            for (int k = 0; k < NW; ++k) x |= rec[i][k] & wmask[k];
            dd[c] = w0 + static_cast<uint32_t>(i * 32) < cnt ? (x >> ds) & 0xffu : 0x100u;
            pp[c] = digit_peers(dd[c]);
        }
#pragma unroll
        for (int c = 0; c < KC; ++c) oo[c] = dd[c] < 256u ? s_hist[warp][c][dd[c]] : 0u;
        __syncwarp();
#pragma unroll
        for (int c = 0; c < KC; ++c)
            if (dd[c] < 256u && (pp[c] >> lane) == 1u) s_hist[warp][c][dd[c]] = static_cast<hist_t>(oo[c] + __popc(pp[c]));
        __syncwarp();
#pragma unroll
        for (int c = 0; c < KC; ++c) dr[c * SPC + s] = (dd[c] << 16) | (oo[c] + __popc(pp[c] & lt_mask));
    }
#elif ZI_OS_RANK == 1
    // Ranking without a dependent shared-memory round trip per record: the highest peer lane of
    // each digit group adds the group's size to the warp's histogram with one shared atomic per
    // record slot -- issued back to back (nothing waits on the result; a warp's shared-memory
    // instructions are performed in issue order, so slot i's groups precede slot i + 1's) -- and
    // the returned bases are handed to the peers by shuffles at the end.
    uint32_t old[IT];
#pragma unroll
    for (int i = 0; i < IT; ++i) {
        uint32_t x = 0;
#pragma unroll
        for (int k = 0; k < NW; ++k) x |= rec[i][k] & wmask[k];
        const uint32_t d = w0 + static_cast<uint32_t>(i * 32) < cnt ? (x >> ds) & 0xffu : 0x100u;
        const uint32_t peers = digit_peers(d);
        old[i] = 0;
        if (d < 256u && (peers >> lane) == 1u) old[i] = atomicAdd(&s_hist[warp][d], static_cast<uint32_t>(__popc(peers)));
        // digit | leader lane | rank among the peers
        dr[i] = (d << 16) | (static_cast<uint32_t>(31 - __clz(peers)) << 8) | static_cast<uint32_t>(__popc(peers & lt_mask));
    }
#pragma unroll
    for (int i = 0; i < IT; ++i) {
        const uint32_t base = __shfl_sync(0xffffffffu, old[i], (dr[i] >> 8) & 31u);
        dr[i] = (dr[i] & 0xffff0000u) | (base + (dr[i] & 0xffu));
    }
#else
#pragma unroll
    for (int i = 0; i < IT; ++i) {
        uint32_t x = 0;
#pragma unroll
        for (int k = 0; k < NW; ++k) x |= rec[i][k] & wmask[k];
        const uint32_t d = w0 + static_cast<uint32_t>(i * 32) < cnt ? (x >> ds) & 0xffu : 0x100u;
        const uint32_t peers = digit_peers(d);
        uint32_t old = 0;
        if (d < 256u) old = s_hist[warp][d];
        __syncwarp();
        if (d < 256u && (peers >> lane) == 1u) s_hist[warp][d] = old + __popc(peers);
        __syncwarp();
        dr[i] = (d << 16) | (old + __popc(peers & lt_mask));
    }
#endif
    __syncthreads();

    // per-digit: warp exclusive offsets + tile count
    const int d = tid & 255;
    const bool dthr = tid < 256;  // digit thread
    uint32_t run = 0;
    if (dthr) {
#if ZI_OS_RANK == 2
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w)
#pragma unroll
            for (int c = 0; c < KC; ++c) {
                const uint32_t t = s_hist[w][c][d];
                s_hist[w][c][d] = static_cast<hist_t>(run);
                run += t;
            }
#else
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) {
            const uint32_t t = s_hist[w][d];
            s_hist[w][d] = run;
            run += t;
        }
#endif
    }
    const uint32_t tile_cnt = run;
    if (MODE == 0 && dthr) os_store(status + static_cast<size_t>(tile) * 256 + d, (tig == 0 ? kFlagInc : kFlagAgg) | tile_cnt);

    // tile-local exclusive scan over digits
    uint32_t start;
    {
        uint32_t x = tile_cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31 && dthr) s_warp[warp] = x;
        __syncthreads();
        uint32_t wp = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) wp += w < warp ? s_warp[w] : 0u;
        start = wp + x - tile_cnt;
        if (dthr) s_start[d] = start;
    }
    if (MODE == 0 && dthr) {
        uint32_t prefix = 0;
        if (tig > 0) {
            prefix = lookback(status, tile, tile - tig, d);
            os_store(status + static_cast<size_t>(tile) * 256 + d, kFlagInc | (prefix + tile_cnt));
        }
        goff = grp * gn + digit_base[grp * 256 + d] + prefix;
    }
    if (dthr) s_delta[d] = goff - start;
    __syncthreads();

    // stage records in tile-sorted order
#pragma unroll
    for (int i = 0; i < IT; ++i) {
        const uint32_t dg = dr[i] >> 16;
        if (dg < 256u) {
#if ZI_OS_RANK == 2
            const uint32_t pos = s_start[dg] + s_hist[warp][i / SPC][dg] + (dr[i] & 0xffffu);
#else
            const uint32_t pos = s_start[dg] + s_hist[warp][dg] + (dr[i] & 0xffffu);
#endif
#pragma unroll
            for (int k = 0; k < NW; ++k) s_stage[k * TILE + pos] = rec[i][k];
        }
    }
    __syncthreads();
    const uint32_t* sdig = s_stage + dw * TILE;
    if constexpr (DF > 0) {
        constexpr int W = NW - 1;
        static_assert((DF + 3) / 4 == W, "final pass: record width and dims disagree");
        uint32_t* pl = sink.planes[grp];
        uint32_t* ky = sink.keys[grp];
        const uint32_t g0 = grp * gn;
#pragma unroll 4
        for (int i = 0; i < IT; ++i) {
            const uint32_t j = static_cast<uint32_t>(tid + i * kSortThreads);
            if (j < cnt) {
                const uint32_t loc = s_delta[(sdig[j] >> ds) & 0xffu] + j - g0;
                uint32_t kw[W], pw[W];
#pragma unroll
                for (int k = 0; k < W; ++k) kw[k] = s_stage[k * TILE + j];
                morton_deinterleave8<DF>(kw, pw);
#pragma unroll
                for (int p = 0; p < W; ++p) pl[static_cast<size_t>(p) * gn + loc] = pw[p];
                const uint32_t pay = s_stage[W * TILE + j];
                ky[loc] = sink.dict ? __ldg(sink.dict + (pay & ((1u << 29) - 1u))) : pay;  // null dict: payload = key
            }
        }
    } else {
        uint32_t* dst[NW];
#pragma unroll
        for (int k = 0; k < NW; ++k) dst[k] = io.out[k];
#pragma unroll
        for (int i = 0; i < IT; ++i) {
            const uint32_t j = static_cast<uint32_t>(tid + i * kSortThreads);
            if (j < cnt) {
                const uint32_t o = s_delta[(sdig[j] >> ds) & 0xffu] + j;
#pragma unroll
                for (int k = 0; k < NW; ++k) dst[k][o] = s_stage[k * TILE + j];
            }
        }
    }
}

// per-256-entry bounding boxes of the layout indices' dim planes (the fused last pass leaves them
// out): one warp per (layout, block), every plane's eight loads per lane in flight together
struct bbox_job {
    const uint32_t* planes[8];
    uint32_t* bmin[8];
    uint32_t* bmax[8];
};
template <int P>
__global__ void __launch_bounds__(256) k_index_bbox(const __grid_constant__ bbox_job J, uint64_t n, uint64_t nblk,
                                                    int nidx) {
    const int lane = threadIdx.x & 31;
    const uint64_t wid = static_cast<uint64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
    // a warp takes kBB consecutive blocks of one layout; full blocks of 16-byte-aligned planes are
    // read as two 16-byte vectors per lane and plane, all of the warp's loads in flight together
    constexpr int kBB = P <= 2 ? 4 : 2;
    const uint64_t wpl = (nblk + kBB - 1) / kBB;  // warps per layout
    if (wid >= wpl * static_cast<uint64_t>(nidx)) return;
    const int l = static_cast<int>(wid / wpl);
    const uint64_t blk0 = (wid - static_cast<uint64_t>(l) * wpl) * kBB;
    const uint32_t* pl = J.planes[l];
    const bool vec = (n & 3u) == 0 && (reinterpret_cast<uintptr_t>(pl) & 15u) == 0 && (blk0 + kBB) * 256 <= n;
    if (vec) {
        uint4 v[kBB][P][2];
#pragma unroll
        for (int b = 0; b < kBB; ++b)
#pragma unroll
            for (int p = 0; p < P; ++p)
#pragma unroll
                for (int e = 0; e < 2; ++e)
                    v[b][p][e] = __ldg(reinterpret_cast<const uint4*>(pl + static_cast<size_t>(p) * n + (blk0 + b) * 256 + e * 128) + lane);
#pragma unroll
        for (int b = 0; b < kBB; ++b)
#pragma unroll
            for (int p = 0; p < P; ++p) {
                uint32_t mn = 0xffffffffu, mx = 0u;
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const uint4 x = v[b][p][e];
                    mn = __vminu4(__vminu4(mn, __vminu4(x.x, x.y)), __vminu4(x.z, x.w));
                    mx = __vmaxu4(__vmaxu4(mx, __vmaxu4(x.x, x.y)), __vmaxu4(x.z, x.w));
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    mn = __vminu4(mn, __shfl_xor_sync(0xffffffffu, mn, o));
                    mx = __vmaxu4(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                }
                if (lane == 0) {
                    J.bmin[l][static_cast<size_t>(p) * nblk + blk0 + b] = mn;
                    J.bmax[l][static_cast<size_t>(p) * nblk + blk0 + b] = mx;
                }
            }
        return;
    }
    for (uint64_t blk = blk0; blk < blk0 + kBB && blk < nblk; ++blk) {
        uint32_t v[P][8];
#pragma unroll
        for (int p = 0; p < P; ++p)
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const uint64_t i = blk * 256 + e * 32 + lane;
                v[p][e] = i < n ? __ldg(pl + static_cast<size_t>(p) * n + i) : 0u;
            }
#pragma unroll
        for (int p = 0; p < P; ++p) {
            uint32_t mn = 0xffffffffu, mx = 0u;
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if (blk * 256 + e * 32 + lane < n) {
                    mn = __vminu4(mn, v[p][e]);
                    mx = __vmaxu4(mx, v[p][e]);
                }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                mn = __vminu4(mn, __shfl_xor_sync(0xffffffffu, mn, o));
                mx = __vmaxu4(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            }
            if (lane == 0) {
                J.bmin[l][static_cast<size_t>(p) * nblk + blk] = mn;
                J.bmax[l][static_cast<size_t>(p) * nblk + blk] = mx;
            }
        }
    }
}

// ---- reduce-then-scan offsets of one pass (MODE 1).  Tiles are grouped in chunks of kLsdChunk
// consecutive tiles of one group: counts[tile][d] -> chunk sums -> per group an exclusive scan over
// its chunks plus the group's digit bases -> per chunk a running sum over its tiles, in place:
// counts[tile][d] becomes the global position of the tile's first record of digit d.
constexpr int kLsdChunk = 32;

template <int IT>
__global__ void __launch_bounds__(kSortThreads) k_lsd_count(const uint32_t* __restrict__ word, int ds, uint32_t gn,
                                                            uint32_t tpg, uint32_t* __restrict__ counts) {
    constexpr int TILE = kSortThreads * IT;
    __shared__ uint32_t s_h[kSortWarps][256];  // per-warp counts: contention only inside a warp
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t tile = blockIdx.x, grp = tile / tpg, tig = tile - grp * tpg;
    const uint32_t t0 = tig * static_cast<uint32_t>(TILE);
    const uint32_t cnt = gn - t0 < static_cast<uint32_t>(TILE) ? gn - t0 : static_cast<uint32_t>(TILE);
    const uint32_t* src = word + grp * gn + t0;
    for (int i = tid; i < kSortWarps * 256; i += kSortThreads) (&s_h[0][0])[i] = 0;
    uint32_t x[IT];
#pragma unroll
    for (int i = 0; i < IT; ++i) {
        const uint32_t j = static_cast<uint32_t>(tid + i * kSortThreads);
        x[i] = j < cnt ? __ldg(src + j) : 0u;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < IT; ++i) {
        const uint32_t j = static_cast<uint32_t>(tid + i * kSortThreads);
        if (j < cnt) atomicAdd(&s_h[warp][(x[i] >> ds) & 0xffu], 1u);
    }
    __syncthreads();
    if (tid < 256) {
        uint32_t c = 0;
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) c += s_h[w][tid];
        counts[static_cast<size_t>(tile) * 256 + tid] = c;
    }
}

__global__ void __launch_bounds__(256) k_lsd_chunk_sum(const uint32_t* __restrict__ counts, uint32_t tpg, uint32_t cpg,
                                                       uint32_t* __restrict__ csum) {
    const uint32_t c = blockIdx.x, g = c / cpg, k = c - g * cpg, d = threadIdx.x;
    const uint32_t t0 = g * tpg + k * kLsdChunk, t1 = min(t0 + kLsdChunk, (g + 1) * tpg);
    uint32_t s = 0;
#pragma unroll 8
    for (uint32_t t = t0; t < t1; ++t) s += __ldg(counts + static_cast<size_t>(t) * 256 + d);
    csum[static_cast<size_t>(c) * 256 + d] = s;
}

// one block per group, kScanParts x 256 threads: thread (part q, digit d) owns a contiguous part of
// the group's chunks (the walk over the chunks is a chain of L2 round trips; the parts run side by
// side): part totals -> exclusive prefix over the parts -> the running sums, in place
constexpr int kScanParts = 4;
__global__ void __launch_bounds__(256 * kScanParts) k_lsd_chunk_scan(uint32_t* __restrict__ csum, uint32_t cpg, uint32_t gn,
                                                                     uint32_t* __restrict__ gbase) {
    __shared__ uint32_t s_w[8];
    __shared__ uint32_t s_part[kScanParts][256];
    const uint32_t g = blockIdx.x;
    const int d = threadIdx.x & 255, q = threadIdx.x >> 8, lane = d & 31, warp = d >> 5;
    uint32_t* cs = csum + static_cast<size_t>(g) * cpg * 256 + d;
    const uint32_t plen = (cpg + kScanParts - 1) / kScanParts;
    const uint32_t k0 = min(cpg, static_cast<uint32_t>(q) * plen), k1 = min(cpg, k0 + plen);
    constexpr uint32_t U = 8;  // chunk sums loaded together
    uint32_t tot = 0;
    for (uint32_t k = k0; k < k1; k += U) {
        uint32_t v[U];
#pragma unroll
        for (uint32_t u = 0; u < U; ++u) v[u] = k + u < k1 ? cs[static_cast<size_t>(k + u) * 256] : 0u;
#pragma unroll
        for (uint32_t u = 0; u < U; ++u) tot += v[u];
    }
    s_part[q][d] = tot;
    __syncthreads();
    uint32_t run = 0, all = 0;
#pragma unroll
    for (int p = 0; p < kScanParts; ++p) {
        const uint32_t t = s_part[p][d];
        run += p < q ? t : 0u;
        all += t;
    }
    for (uint32_t k = k0; k < k1; k += U) {
        uint32_t v[U];
#pragma unroll
        for (uint32_t u = 0; u < U; ++u) v[u] = k + u < k1 ? cs[static_cast<size_t>(k + u) * 256] : 0u;
#pragma unroll
        for (uint32_t u = 0; u < U; ++u) {
            if (k + u < k1) cs[static_cast<size_t>(k + u) * 256] = run;
            run += v[u];
        }
    }
    // the group's digit bases: exclusive scan of the totals over the digits (added by k_lsd_offsets)
    uint32_t x = all;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (q == 0 && lane == 31) s_w[warp] = x;
    __syncthreads();
    if (q == 0) {
        uint32_t wp = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) wp += w < warp ? s_w[w] : 0u;
        gbase[g * 256 + d] = g * gn + wp + x - all;
    }
}

__global__ void __launch_bounds__(256) k_lsd_offsets(uint32_t* __restrict__ counts, const uint32_t* __restrict__ csum,
                                                     const uint32_t* __restrict__ gbase, uint32_t tpg, uint32_t cpg) {
    const uint32_t c = blockIdx.x, g = c / cpg, k = c - g * cpg, d = threadIdx.x;
    const uint32_t t0 = g * tpg + k * kLsdChunk, t1 = min(t0 + kLsdChunk, (g + 1) * tpg);
    uint32_t run = csum[static_cast<size_t>(c) * 256 + d] + gbase[g * 256 + d];
    uint32_t v[kLsdChunk];  // the chunk's counts, all loads in flight before the running sum
#pragma unroll
    for (int u = 0; u < kLsdChunk; ++u) v[u] = t0 + u < t1 ? counts[static_cast<size_t>(t0 + u) * 256 + d] : 0u;
#pragma unroll
    for (int u = 0; u < kLsdChunk; ++u) {
        if (t0 + u < t1) counts[static_cast<size_t>(t0 + u) * 256 + d] = run;
        run += v[u];
    }
}

// records per thread: the largest count whose registers fit without spills at the kernel's
// occupancy (NW * IT <= 36: three CTAs per SM, else two)
template <int NW>
constexpr int os_items() {
    return NW == 2 ? 12 : NW == 3 ? ZI_OS_IT3 : NW == 4 ? 16 : NW == 5 ? 12 : 8;
}

static int onesweep_items(int nw) {
    switch (nw) {
        case 2: return os_items<2>();
        case 3: return os_items<3>();
        case 4: return os_items<4>();
        case 5: return os_items<5>();
        case 6: return os_items<6>();
        case 7: return os_items<7>();
        case 8: return os_items<8>();
        default: return os_items<9>();
    }
}

static bool lookback_mode() {  // ZI_SORT_LOOKBACK=1: the decoupled look-back pass (A/B)
    static const bool v = std::getenv("ZI_SORT_LOOKBACK") != nullptr;
    return v;
}

struct pass_plan {
    uint64_t gn;
    unsigned tpg, ntiles, cpg;
    const uint32_t* digit_base;  // MODE 0
    uint32_t* status;            // MODE 0
    uint32_t* ctr;               // MODE 0
    uint32_t* counts;            // MODE 1: [ntiles][256]
    uint32_t* csum;              // MODE 1: [G * cpg][256]
    uint32_t* gbase;             // MODE 1: [G][256] first position of every (group, digit)
};

template <int NW>
static void launch_pass(zi_ctx* ctx, const sort_words& io, int dw, int ds, const pass_plan& pp, int G,
                        const final_sink* sink = nullptr) {
    constexpr int IT = os_items<NW>();
    const size_t smem = static_cast<size_t>(NW) * kSortThreads * IT * sizeof(uint32_t);
    if (lookback_mode()) {
        smem_attr(ctx->device, k_onesweep<NW, IT, 0>, smem);
        ZI_LAUNCH(ctx, "radix_onesweep", (k_onesweep<NW, IT, 0>), pp.ntiles, kSortThreads, smem, io, dw, ds, pp.digit_base,
                  pp.status, pp.ctr, static_cast<const uint32_t*>(nullptr), static_cast<uint32_t>(pp.gn), pp.tpg,
                  final_sink{});
        return;
    }
    const uint32_t gn = static_cast<uint32_t>(pp.gn);
    ZI_LAUNCH(ctx, "radix_count", k_lsd_count<IT>, pp.ntiles, kSortThreads, 0, io.in[dw], ds, gn, pp.tpg, pp.counts);
    const unsigned nch = pp.cpg * static_cast<unsigned>(G);
    ZI_LAUNCH(ctx, "radix_scan", k_lsd_chunk_sum, nch, 256, 0, pp.counts, pp.tpg, pp.cpg, pp.csum);
    ZI_LAUNCH(ctx, "radix_scan", k_lsd_chunk_scan, static_cast<unsigned>(G), 256 * kScanParts, 0, pp.csum, pp.cpg, gn, pp.gbase);
    ZI_LAUNCH(ctx, "radix_scan", k_lsd_offsets, nch, 256, 0, pp.counts, pp.csum, pp.gbase, pp.tpg, pp.cpg);
    if (sink) {  // the last pass of the 8-layout sort: straight into the indices
        constexpr int DF = NW == 2 ? 4 : NW == 3 ? 8 : NW == 4 ? 12 : 16;
        if constexpr (NW >= 2 && NW <= 5) {
            smem_attr(ctx->device, k_onesweep<NW, IT, 1, DF>, smem);
            ZI_LAUNCH(ctx, "radix_onesweep", (k_onesweep<NW, IT, 1, DF>), pp.ntiles, kSortThreads, smem, io, dw, ds,
                      static_cast<const uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                      static_cast<uint32_t*>(nullptr), static_cast<const uint32_t*>(pp.counts), gn, pp.tpg, *sink);
            return;
        }
    }
    smem_attr(ctx->device, k_onesweep<NW, IT, 1>, smem);
    ZI_LAUNCH(ctx, "radix_onesweep", (k_onesweep<NW, IT, 1>), pp.ntiles, kSortThreads, smem, io, dw, ds,
              static_cast<const uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
              static_cast<const uint32_t*>(pp.counts), gn, pp.tpg, final_sink{});
}

// Generic stable LSD sort of NW-word SoA records; passes are (word, shift) digits from the
// least significant.  Trivial passes (every group's records share the digit) are skipped when the
// histograms are on the host.  G groups of n/G records (group-major) are sorted each on its own
// (no pass on a group digit).
// digit histograms of every pass (host copy, [pass][group][256]), one read of the records
std::vector<uint32_t> pass_histograms(zi_ctx* ctx, uint32_t* const* words, int nw, uint64_t n,
                                      const std::vector<int2>& passes, int G) {
    const int npass = static_cast<int>(passes.size());
    const size_t hist_words = static_cast<size_t>(npass) * G * 256;
    uint32_t* h = ctx->counter.ensure(hist_words + 4 * npass + 64);
    int2* d_passes = reinterpret_cast<int2*>(h + hist_words + 8);
    d_passes = reinterpret_cast<int2*>((reinterpret_cast<uintptr_t>(d_passes) + 15) & ~uintptr_t(15));
    ZI_CUDA(cudaMemsetAsync(h, 0, hist_words * sizeof(uint32_t), ctx->stream));
    ZI_CUDA(cudaMemcpyAsync(d_passes, passes.data(), passes.size() * sizeof(int2), cudaMemcpyHostToDevice, ctx->stream));
    sort_words io{};
    for (int k = 0; k < nw; ++k) io.in[k] = words[k];
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(ctx->num_sms) * 4));
    smem_attr(ctx->device, k_sort_hist, static_cast<size_t>(npass) * 256 * sizeof(uint32_t));
    ZI_LAUNCH(ctx, "radix_hist", k_sort_hist, grid, 256, static_cast<size_t>(npass) * 256 * sizeof(uint32_t), io, npass,
              d_passes, n, n / G, G, h);
    std::vector<uint32_t> out(hist_words);
    ZI_CUDA(cudaMemcpyAsync(out.data(), h, hist_words * sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
    ZI_CUDA(cudaStreamSynchronize(ctx->stream));
    return out;
}

// groups G > 1: at most 40 passes, digit bases per (pass, group) in the scratch
static bool groups_fit(int npass, int G) { return npass <= 40 && G <= 8; }

// result (optional): receives the buffers holding the sorted words -- the scratch copy after an
// odd number of passes -- instead of copying them back into `words`.  device_bases: every pass
// runs, nothing goes through the host (the histograms are only needed to skip trivial passes).
void radix_sort_words(zi_ctx* ctx, uint32_t** words, int nw, uint64_t n, const std::vector<int2>& passes,
                      const uint32_t* hist_host, bool device_bases, uint32_t** result, int G,
                      const final_sink* sink = nullptr) {
    if (result)
        for (int k = 0; k < nw; ++k) result[k] = words[k];
    if (n <= 1 || passes.empty()) return;
    if (n > kValMask) throw error(ZI_E_INVALID, "radix sort: more than 2^30 records");
    if (nw < 2 || nw > kMaxWords) throw error(ZI_E_INVALID, "radix sort: unsupported record width");
    if (G < 1 || n % G != 0) throw error(ZI_E_INVALID, "radix sort: records do not split into equal groups");
    const int npass = static_cast<int>(passes.size());
    const bool lb = lookback_mode();
    pass_plan pp{};
    pp.gn = n / G;
    const uint64_t tile = static_cast<uint64_t>(kSortThreads) * onesweep_items(nw);
    pp.tpg = static_cast<unsigned>((pp.gn + tile - 1) / tile);
    pp.ntiles = pp.tpg * static_cast<unsigned>(G);
    pp.cpg = (pp.tpg + kLsdChunk - 1) / kLsdChunk;
    // scratch: alt words (nw*n) | hist (npass*G*256) | bases (same) | MODE 1: counts (ntiles*256),
    // chunk sums (G*cpg*256) / MODE 0: status (npass*ntiles*256), counters | pass table
    const size_t alt_words = static_cast<size_t>(nw) * n;
    const size_t hist_words = static_cast<size_t>(npass) * G * 256;
    const size_t work_words = lb ? static_cast<size_t>(npass) * pp.ntiles * 256 + npass + 8
                                 : static_cast<size_t>(pp.ntiles) * 256 + static_cast<size_t>(G) * (pp.cpg + 1) * 256;
    uint32_t* scr = reinterpret_cast<uint32_t*>(
        ctx->scratch.ensure((alt_words + 2 * hist_words + work_words + 4 * npass + 64) * sizeof(uint32_t)));
    uint32_t* alt = scr;
    uint32_t* hist = alt + alt_words;
    uint32_t* bases = hist + hist_words;
    uint32_t* work = bases + hist_words;
    int2* d_passes = reinterpret_cast<int2*>(work + work_words + 8);  // tiny
    d_passes = reinterpret_cast<int2*>((reinterpret_cast<uintptr_t>(d_passes) + 15) & ~uintptr_t(15));
    if (lb) {
        pp.status = work;
        pp.ctr = work + static_cast<size_t>(npass) * pp.ntiles * 256;
    } else {
        pp.counts = work;
        pp.csum = work + static_cast<size_t>(pp.ntiles) * 256;
        pp.gbase = pp.csum + static_cast<size_t>(G) * pp.cpg * 256;
    }

    sort_words io{};
    for (int k = 0; k < nw; ++k) {
        io.in[k] = words[k];
        io.out[k] = alt + static_cast<size_t>(k) * n;
    }
    std::vector<int> active;
    std::vector<uint32_t> h_hist(hist_words);
    auto run_hist = [&] {
        ZI_CUDA(cudaMemsetAsync(hist, 0, hist_words * sizeof(uint32_t), ctx->stream));
        ZI_CUDA(cudaMemcpyAsync(d_passes, passes.data(), passes.size() * sizeof(int2), cudaMemcpyHostToDevice, ctx->stream));
        const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(ctx->num_sms) * 4));
        const size_t hsm = static_cast<size_t>(npass) * 256 * sizeof(uint32_t);
        smem_attr(ctx->device, k_sort_hist, hsm);
        ZI_LAUNCH(ctx, "radix_hist", k_sort_hist, grid, 256, hsm, io, npass, d_passes, n, pp.gn, G, hist);
    };
    if (device_bases) {  // no host round trip: every pass runs (trivial ones are a copy)
        if (lb) {  // the look-back pass needs the global digit bases up front
            run_hist();
            ZI_LAUNCH(ctx, "radix_bases", k_sort_bases, static_cast<unsigned>(npass * G), 256, 0, hist, bases);
        }
        for (int q = 0; q < npass; ++q) active.push_back(q);
    } else {
        if (hist_host) {
            std::copy(hist_host, hist_host + hist_words, h_hist.begin());
        } else {
            run_hist();
            ZI_CUDA(cudaMemcpyAsync(h_hist.data(), hist, hist_words * sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
            ZI_CUDA(cudaStreamSynchronize(ctx->stream));
        }
        std::vector<uint32_t> h_bases(hist_words, 0);
        for (int q = 0; q < npass; ++q) {
            bool trivial = true;
            for (int g = 0; g < G; ++g) {
                bool gt = false;
                uint32_t r = 0;
                for (int dgt = 0; dgt < 256; ++dgt) {
                    const size_t at = (static_cast<size_t>(q) * G + g) * 256 + dgt;
                    const uint32_t c = h_hist[at];
                    if (c == pp.gn) gt = true;
                    h_bases[at] = r;
                    r += c;
                }
                trivial = trivial && gt;
            }
            if (!trivial) active.push_back(q);
        }
        if (!active.empty() && lb)
            ZI_CUDA(cudaMemcpyAsync(bases, h_bases.data(), hist_words * sizeof(uint32_t), cudaMemcpyHostToDevice, ctx->stream));
    }
    if (active.empty()) return;
    if (lb) {
        ZI_CUDA(cudaMemsetAsync(pp.status, 0, static_cast<size_t>(npass) * pp.ntiles * 256 * sizeof(uint32_t), ctx->stream));
        ZI_CUDA(cudaMemsetAsync(pp.ctr, 0, npass * sizeof(uint32_t), ctx->stream));
    }
    uint32_t* cur[kMaxWords];
    uint32_t* oth[kMaxWords];
    for (int k = 0; k < nw; ++k) {
        cur[k] = words[k];
        oth[k] = alt + static_cast<size_t>(k) * n;
    }
    for (size_t a = 0; a < active.size(); ++a) {
        const int q = active[a];
        for (int k = 0; k < nw; ++k) {
            io.in[k] = cur[k];
            io.out[k] = oth[k];
        }
        pass_plan pq = pp;
        if (lb) {
            pq.status = pp.status + static_cast<size_t>(q) * pp.ntiles * 256;
            pq.ctr = pp.ctr + q;
            pq.digit_base = bases + static_cast<size_t>(q) * G * 256;
        }
        const int dw = passes[q].x, ds = passes[q].y;
        const final_sink* sk = a + 1 == active.size() ? sink : nullptr;  // (the look-back mode takes no sink)
        switch (nw) {
            case 2: launch_pass<2>(ctx, io, dw, ds, pq, G, sk); break;
            case 3: launch_pass<3>(ctx, io, dw, ds, pq, G, sk); break;
            case 4: launch_pass<4>(ctx, io, dw, ds, pq, G, sk); break;
            case 5: launch_pass<5>(ctx, io, dw, ds, pq, G, sk); break;
            case 6: launch_pass<6>(ctx, io, dw, ds, pq, G); break;
            case 7: launch_pass<7>(ctx, io, dw, ds, pq, G); break;
            case 8: launch_pass<8>(ctx, io, dw, ds, pq, G); break;
            default: launch_pass<9>(ctx, io, dw, ds, pq, G); break;
        }
        for (int k = 0; k < nw; ++k) std::swap(cur[k], oth[k]);
    }
    if (result) {
        for (int k = 0; k < nw; ++k) result[k] = cur[k];
    } else if (active.size() % 2 == 1) {
        for (int k = 0; k < nw; ++k)
            ZI_CUDA(cudaMemcpyAsync(words[k], cur[k], n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, ctx->stream));
    }
}

void radix_sort_words(zi_ctx* ctx, uint32_t** words, int nw, uint64_t n, const std::vector<int2>& passes,
                      const uint32_t* hist_host, bool device_bases, uint32_t** result) {
    radix_sort_words(ctx, words, nw, n, passes, hist_host, device_bases, result, 1);
}

void radix_sort_words(zi_ctx* ctx, uint32_t** words, int nw, uint64_t n, const std::vector<int2>& passes,
                      const uint32_t* hist_host, bool device_bases) {
    radix_sort_words(ctx, words, nw, n, passes, hist_host, device_bases, nullptr, 1);
}

// ---------------------------------------------------------------------------- hybrid sort
// MSD split + local sort.  A few onesweep passes order the records by the top Morton bytes
// (and, for the 8-layout build, the layout bits of the payload) -- segments of equal top bits
// are then contiguous.  k_segsort finishes each segment in shared memory with the full
// comparator (Morton key, payload).  The payload is unique, so this order is the unique stable
// order whatever order the segment arrives in; the result is bit-identical to the all-LSD sort
// at roughly a third of its HBM passes.
static int msd_bytes_forced() {  // ZI_SORT_MSD overrides the histogram-driven MSD depth
    static const int v = [] {
        const char* e = std::getenv("ZI_SORT_MSD");
        return e ? std::atoi(e) : 0;
    }();
    return v;
}
static bool verify_on() {
    static const bool v = std::getenv("ZI_SORT_VERIFY") != nullptr;
    return v;
}
constexpr int kSegThreads = 256;
constexpr uint32_t kMaxBig = 64;  // oversized segments finished one by one; more -> full LSD

// segmask[k]: the bits of record word k that form the segment key (the top nb Morton bytes, and
// the payload's layout bits); cmpmask[k] (k < 3): the bits of key word k below the segment key.
// When the remaining bytes fit (D - nb <= 12) a record's order inside its segment is the 128-bit
// compare key ((w2 & m2):(w1 & m1), (w0 & m0):payload).
template <int NW>
struct seg_ctx {
    uint32_t* w[kMaxWords];
    uint64_t N;
    uint32_t segmask[kMaxWords];
    uint32_t cmpmask[3];
    bool can_count;
};

template <int NW>
__device__ inline bool seg_differs(const seg_ctx<NW>& c, uint64_t i, uint64_t j) {
    uint32_t d = 0;
#pragma unroll
    for (int k = 0; k < NW; ++k) d |= (c.w[k][i] ^ c.w[k][j]) & c.segmask[k];
    return d != 0;
}

// first segment head in [from, limit) (limit if none); one warp
template <int NW>
__device__ inline uint64_t find_head(const seg_ctx<NW>& c, uint64_t from, uint64_t limit) {
    const int lane = threadIdx.x & 31;
    if (from == 0) return 0;
    if (limit > c.N) limit = c.N;
    for (uint64_t b = from; b < limit; b += 32) {
        const uint64_t i = b + lane;
        const bool h = i < limit && seg_differs(c, i, i - 1);
        const unsigned m = __ballot_sync(0xffffffffu, h);
        if (m) return b + __ffs(m) - 1;
    }
    return limit;
}

// Shared-memory record layout of the window sort: array-of-records, P words per record (16-byte
// aligned for NW > 2) so a whole record is one or two vector loads.
template <int NW>
struct seg_rec {
    static constexpr int P = NW <= 2 ? 2 : (NW + 3) & ~3;
    __device__ static inline void load(const uint32_t* p, uint32_t (&r)[NW]) {
        if constexpr (P == 2) {
            const uint2 v = *reinterpret_cast<const uint2*>(p);
            r[0] = v.x;
            if constexpr (NW > 1) r[NW - 1] = v.y;
        } else {
#pragma unroll
            for (int q = 0; q < P / 4; ++q) {
                const uint4 v = *reinterpret_cast<const uint4*>(p + 4 * q);
                if (4 * q + 0 < NW) r[(4 * q + 0) % NW] = v.x;
                if (4 * q + 1 < NW) r[(4 * q + 1) % NW] = v.y;
                if (4 * q + 2 < NW) r[(4 * q + 2) % NW] = v.z;
                if (4 * q + 3 < NW) r[(4 * q + 3) % NW] = v.w;
            }
        }
    }
};

// One CTA sorts one window: the records of the segments that start in [w*T, (w+1)*T) (so the
// window is a union of whole segments), loaded into shared memory and written back in place.
// Segments never change the segment key at any position, so neighbours reading a boundary
// while this CTA writes see the same keys.  Two ways to order a window:
//  * rank by counting (short segments, the common case): record j of segment [ss, se) goes to
//    ss + #{k in [ss, se) : rec_k < rec_j} under the full comparator -- sum of L^2 compares,
//    no passes; segment bounds come from a head bitmask (last head <= j, first head > j);
//  * all passes of the global LSD sort replayed on a u16 permutation (long segments).
// The record-weighted mean segment length (sum L^2 / len) picks the way per window.
constexpr int kSegCountMean = 24;

template <int NW>
__global__ void __launch_bounds__(kSegThreads) k_segsort(seg_ctx<NW> c, int T, int cap, int npass,
                                                         const int2* __restrict__ passes,
                                                         unsigned long long* __restrict__ big,
                                                         uint32_t* __restrict__ nbig, int count_mean,
                                                         unsigned long long* __restrict__ sumL) {
    using R = seg_rec<NW>;
    extern __shared__ uint32_t s_w[];  // cap records of R::P words, cur / nxt (u16 cap each), head bits
    uint16_t* s_cur = reinterpret_cast<uint16_t*>(s_w + static_cast<size_t>(R::P) * cap);
    uint16_t* s_nxt = s_cur + cap;
    uint32_t* s_head = reinterpret_cast<uint32_t*>(s_nxt + cap);  // (cap + kSegThreads + 32) / 32 words
    constexpr int kWarps = kSegThreads / 32;
    __shared__ uint32_t s_hist[kWarps][256];
    __shared__ uint32_t s_dstart[256];
    __shared__ uint32_t s_wsum[kWarps];
    __shared__ uint64_t s_range[2];
    __shared__ int2 s_pass[40];
    __shared__ unsigned long long s_sumL;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t w0 = static_cast<uint64_t>(blockIdx.x) * T;
    const uint64_t w1 = w0 + T < c.N ? w0 + T : c.N;
    // the segments starting in [w0, w1): start = first head, end = first head at or after w1;
    // searches stop once the range cannot fit (no quadratic scans inside long segments)
    if (warp == 0) {
        const uint64_t st = find_head(c, w0, w1);
        uint64_t en = st;
        if (st < w1) en = w1 >= c.N ? c.N : find_head(c, w1, st + cap + 1);
        if (lane == 0) {
            s_range[0] = st;
            s_range[1] = en;
        }
    }
    if (tid < npass) s_pass[tid] = passes[tid];
    if (tid == 0) s_sumL = 0;
    __syncthreads();
    const uint64_t start = s_range[0];
    uint64_t end = s_range[1];
    if (start >= w1) return;  // no segment starts in this window
    if (end - start > static_cast<uint64_t>(cap)) {  // longer than shared memory: global fallback
        if (warp == 0) {
            const uint64_t e2 = end >= c.N ? c.N : find_head(c, end, c.N);  // its real end (once per segment)
            if (lane == 0) s_range[1] = e2;
        }
        __syncthreads();
        end = s_range[1];
        if (tid == 0) {
            const uint32_t slot = atomicAdd(nbig, 1u);
            if (slot < kMaxBig) {
                big[2 * slot] = start;
                big[2 * slot + 1] = end;
            }
            atomicAdd(nbig + 1, static_cast<uint32_t>(end - start < 0xffffffffull ? end - start : 0xffffffffull));
        }
        return;
    }
    const int len = static_cast<int>(end - start);
    if (len <= 1) return;
    __shared__ uint32_t s_and[NW], s_or[NW];
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
    // batches of kLoadRounds rounds: all of a batch's global loads are in flight together
    constexpr int kLoadRounds = 4;
    for (int j0 = 0; j0 < len; j0 += kSegThreads * kLoadRounds) {
        uint32_t v[kLoadRounds][NW];
#pragma unroll
        for (int r = 0; r < kLoadRounds; ++r) {
            const int j = j0 + r * kSegThreads + tid;
            if (j < len)
#pragma unroll
                for (int k = 0; k < NW; ++k) v[r][k] = c.w[k][start + j];
        }
#pragma unroll
        for (int r = 0; r < kLoadRounds; ++r) {
            const int j = j0 + r * kSegThreads + tid;
            if (j < len) {
#pragma unroll
                for (int k = 0; k < NW; ++k) {
                    s_w[j * R::P + k] = v[r][k];
                    wand[k] &= v[r][k];
                    wor[k] |= v[r][k];
                }
                s_cur[j] = static_cast<uint16_t>(j);
            }
        }
    }
#pragma unroll
    for (int k = 0; k < NW; ++k) {  // digits equal over the whole window need no pass
        atomicAnd(&s_and[k], wand[k]);
        atomicOr(&s_or[k], wor[k]);
    }
    __syncthreads();  // records and the constant-digit masks are complete
    // segment heads; bit len is a sentinel head
    for (int b = 0; b <= len; b += kSegThreads) {
        const int j = b + tid;
        bool h = j == len;
        if (j < len) {
            if (j == 0) {
                h = true;
            } else {
                uint32_t a[NW], p[NW], d = 0;
                R::load(s_w + j * R::P, a);
                R::load(s_w + (j - 1) * R::P, p);
#pragma unroll
                for (int k = 0; k < NW; ++k) d |= (a[k] ^ p[k]) & c.segmask[k];
                h = d != 0;
            }
        }
        const unsigned m = __ballot_sync(0xffffffffu, h);
        if (lane == 0) s_head[j >> 5] = m;
    }
    __syncthreads();
    auto seg_start = [&](int j) {
        int wi = j >> 5;
        unsigned m = s_head[wi] & (0xffffffffu >> (31 - (j & 31)));
        while (m == 0) m = s_head[--wi];
        return (wi << 5) + 31 - __clz(m);
    };
    auto seg_end = [&](int j) {
        int wi = j >> 5;
        unsigned m = (j & 31) == 31 ? 0u : s_head[wi] & (0xfffffffeu << (j & 31));
        while (m == 0) m = s_head[++wi];
        return (wi << 5) + __ffs(m) - 1;
    };
    {
        unsigned long long sl = 0;
        for (int j = tid; j < len; j += kSegThreads) sl += static_cast<unsigned>(seg_end(j) - seg_start(j));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sl += __shfl_xor_sync(0xffffffffu, sl, o);
        if (lane == 0) atomicAdd(&s_sumL, sl);
    }
    __syncthreads();
    if (tid == 0) atomicAdd(sumL, s_sumL);
    if (c.can_count && s_sumL <= static_cast<unsigned long long>(count_mean) * static_cast<unsigned long long>(len)) {
        ulonglong2* s_ck = reinterpret_cast<ulonglong2*>(
            (reinterpret_cast<uintptr_t>(s_head + (cap + kSegThreads + 32) / 32) + 15) & ~static_cast<uintptr_t>(15));
        for (int j = tid; j < len; j += kSegThreads) {
            uint32_t r[NW];
            R::load(s_w + j * R::P, r);
            const uint32_t w1 = NW > 2 ? r[NW > 2 ? 1 : 0] & c.cmpmask[1] : 0u;
            const uint32_t w2 = NW > 3 ? r[NW > 3 ? 2 : 0] & c.cmpmask[2] : 0u;
            s_ck[j] = make_ulonglong2((static_cast<unsigned long long>(r[0] & c.cmpmask[0]) << 32) | r[NW - 1],
                                      (static_cast<unsigned long long>(w2) << 32) | w1);
        }
        __syncthreads();
        for (int j = tid; j < len; j += kSegThreads) {
            const int ss = seg_start(j), se = seg_end(j);
            const ulonglong2 me = s_ck[j];
            int rank = 0;
            for (int k = ss; k < se; ++k) {
                const ulonglong2 o = s_ck[k];
                rank += (o.y < me.y || (o.y == me.y && o.x < me.x)) ? 1 : 0;
            }
            s_nxt[ss + rank] = static_cast<uint16_t>(j);
        }
        __syncthreads();
        for (int j = tid; j < len; j += kSegThreads) {
            const int src = s_nxt[j];
#pragma unroll
            for (int k = 0; k < NW; ++k) c.w[k][start + j] = s_w[src * R::P + k];
        }
        return;
    }
    // warp w ranks the contiguous chunk [w*CH, (w+1)*CH) in rounds of 32 (stable order)
    const int CH = ((len + kWarps - 1) / kWarps + 31) & ~31;
    const int nround = CH / 32;
    const uint32_t lt = (1u << lane) - 1u;
    constexpr int kMaxRounds = 16;  // cap <= 4096 -> CH <= 512
    for (int q = 0; q < npass; ++q) {
        const int wk = s_pass[q].x, sh = s_pass[q].y;
        if ((((s_and[wk] ^ s_or[wk]) >> sh) & 0xffu) == 0u) continue;  // uniform: constant digit
        for (int i = tid; i < kWarps * 256; i += kSegThreads) (&s_hist[0][0])[i] = 0;
        __syncthreads();
        uint32_t dg[kMaxRounds], rk[kMaxRounds];
#pragma unroll
        for (int r = 0; r < kMaxRounds; ++r) {
            if (r < nround) {
                const int i = warp * CH + r * 32 + lane;
                uint32_t d = 256u;
                if (i < len) d = (s_w[s_cur[i] * R::P + wk] >> sh) & 0xffu;
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
        // digit-major exclusive offsets: warp w's run of digit d starts at dstart[d] + off[w][d]
        {
            const int d = tid;  // kSegThreads == 256 digits
            uint32_t run = 0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                const uint32_t t = s_hist[w][d];
                s_hist[w][d] = run;
                run += t;
            }
            uint32_t x = run;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) s_wsum[warp] = x;
            __syncthreads();
            uint32_t wp = 0;
            for (int w = 0; w < warp; ++w) wp += s_wsum[w];
            s_dstart[d] = wp + x - run;
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
        uint16_t* t = s_cur;
        s_cur = s_nxt;
        s_nxt = t;
    }
    for (int j = tid; j < len; j += kSegThreads) {
        const int src = s_cur[j];
#pragma unroll
        for (int k = 0; k < NW; ++k) c.w[k][start + j] = s_w[src * R::P + k];
    }
}

template <int NW>
static void launch_segsort(zi_ctx* ctx, uint32_t* const* words, uint64_t N, int D, int nb, bool layouts,
                           const std::vector<int2>& passes, int2* d_passes, unsigned long long* big, uint32_t* nbig,
                           unsigned long long* sumL) {
    seg_ctx<NW> c{};
    for (int k = 0; k < NW; ++k) c.w[k] = words[k];
    c.N = N;
    for (int p = std::max(D - nb, 0); p < D; ++p) c.segmask[p >> 2] |= 0xffu << ((p & 3) * 8);
    if (layouts) c.segmask[NW - 1] = 0xe0000000u;
    for (int p = 0; p < D - nb && p < 12; ++p) c.cmpmask[p >> 2] |= 0xffu << ((p & 3) * 8);
    c.can_count = D - nb <= 12;
    static const int cap0 = [] { const char* e = std::getenv("ZI_SORT_CAP"); return e ? std::atoi(e) : 4096; }();
    static const int count_mean = [] { const char* e = std::getenv("ZI_SORT_COUNT"); return e ? std::atoi(e) : kSegCountMean; }();
    constexpr int P = seg_rec<NW>::P;
    // records | cur, nxt | head bits | 16-byte compare keys
    auto bytes = [](int cp) {
        return static_cast<size_t>(cp) * (P * 4 + 4) + static_cast<size_t>(cp + kSegThreads + 32) / 32 * 4 + 16 +
               static_cast<size_t>(cp) * 16;
    };
    int cap = cap0;
    while (cap > 1024 && bytes(cap) > 112 * 1024) cap >>= 1;
    const int T = cap / 2;
    const size_t smem = bytes(cap);
    smem_attr(ctx->device, k_segsort<NW>, smem);
    ZI_CUDA(cudaMemcpyAsync(d_passes, passes.data(), passes.size() * sizeof(int2), cudaMemcpyHostToDevice, ctx->stream));
    const unsigned grid = static_cast<unsigned>((N + T - 1) / T);
    ZI_LAUNCH(ctx, "segment_sort", k_segsort<NW>, grid, kSegThreads, smem, c, T, cap, static_cast<int>(passes.size()),
              d_passes, big, nbig, count_mean, sumL);
}

// window sort + oversized-segment handling after the MSD passes
// all: the passes of the full (grouped, G > 1: no layout digit) LSD sort; all_full: every pass,
// layout digit included (the window replay and sub-range sorts, which can straddle two layouts)
static void finish_hybrid(zi_ctx* ctx, uint32_t** words, uint32_t** orig, int W, uint64_t N, int D, int nb,
                          bool layouts, const std::vector<int2>& all, const std::vector<int2>& all_full, int G,
                          int& learnt) {
    const int nw = W + 1;
    static const bool debug = std::getenv("ZI_DEBUG_SORT") != nullptr;
    // counters | big-segment list | pass table, in the context counter buffer
    uint32_t* cnt = ctx->counter.ensure(16 + 4 * kMaxBig + 2 * 64);
    unsigned long long* big = reinterpret_cast<unsigned long long*>(cnt + 16);
    int2* d_passes = reinterpret_cast<int2*>(cnt + 16 + 4 * kMaxBig);
    unsigned long long* sumL = reinterpret_cast<unsigned long long*>(cnt + 2);  // sum of L^2 over segments
    ZI_CUDA(cudaMemsetAsync(cnt, 0, 4 * sizeof(uint32_t), ctx->stream));
    switch (nw) {
        case 2: launch_segsort<2>(ctx, words, N, D, nb, layouts, all_full, d_passes, big, cnt, sumL); break;
        case 3: launch_segsort<3>(ctx, words, N, D, nb, layouts, all_full, d_passes, big, cnt, sumL); break;
        case 4: launch_segsort<4>(ctx, words, N, D, nb, layouts, all_full, d_passes, big, cnt, sumL); break;
        case 5: launch_segsort<5>(ctx, words, N, D, nb, layouts, all_full, d_passes, big, cnt, sumL); break;
        case 6: launch_segsort<6>(ctx, words, N, D, nb, layouts, all_full, d_passes, big, cnt, sumL); break;
        case 7: launch_segsort<7>(ctx, words, N, D, nb, layouts, all_full, d_passes, big, cnt, sumL); break;
        case 8: launch_segsort<8>(ctx, words, N, D, nb, layouts, all_full, d_passes, big, cnt, sumL); break;
        case 9: launch_segsort<9>(ctx, words, N, D, nb, layouts, all_full, d_passes, big, cnt, sumL); break;
        default: throw error(ZI_E_INVALID, "radix sort: unsupported record width");
    }
    uint32_t hc[4] = {0, 0, 0, 0};
    ZI_CUDA(cudaMemcpyAsync(hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, ctx->stream));
    ZI_CUDA(cudaStreamSynchronize(ctx->stream));
    const uint32_t nbig = hc[0];
    const double mean_len = static_cast<double>((static_cast<uint64_t>(hc[3]) << 32) | hc[2]) / static_cast<double>(N);
    if (debug)
        std::fprintf(stderr, "hybrid sort N=%llu nb=%d: oversized segments %u (%u records), record-weighted mean segment %.1f\n",
                     static_cast<unsigned long long>(N), nb, nbig, hc[1], mean_len);
    // windows rank by counting while segments are short; long ones replay the LSD passes at
    // several times the cost -- later builds with these dims split one byte deeper
    if (nbig == 0 && mean_len > kSegCountMean && msd_bytes_forced() <= 0 && learnt >= 0 && nb + 1 <= D - 3 &&
        D - (nb + 1) <= 12)
        learnt = nb + 1;
    if (nbig == 0) return;
    if (words[0] != orig[0]) {  // the nested sorts below use the scratch buffer the records sit in
        for (int k = 0; k < nw; ++k) {
            ZI_CUDA(cudaMemcpyAsync(orig[k], words[k], N * sizeof(uint32_t), cudaMemcpyDeviceToDevice, ctx->stream));
            words[k] = orig[k];
        }
    }
    if (nbig > kMaxBig || static_cast<uint64_t>(hc[1]) * 8 > N) {
        // top bytes too clustered for the split (smooth images, or few high-variance PCA dims):
        // finish with the full LSD sort.  Equal keys are already in payload order everywhere, so
        // the stable passes from the current order give the reference permutation.  Later builds
        // with these dims go straight to LSD (one byte deeper rarely splits a clustered top: cfg4
        // still leaves 10 % / 6 % of the records in oversized segments at 4 / 5 MSD bytes).
        learnt = -1;
        radix_sort_words(ctx, words, nw, N, all, nullptr, true, nullptr, G);
        return;
    }
    std::vector<unsigned long long> h(2 * nbig);
    ZI_CUDA(cudaMemcpyAsync(h.data(), big, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
    ZI_CUDA(cudaStreamSynchronize(ctx->stream));
    // oversized ranges (whole segments, the last one running past shared memory): the global
    // LSD sort on that range with every pass (stable, so the payload order of ties stays; the
    // range can hold several segments, so the top bytes take part too)
    for (uint32_t q = 0; q < nbig; ++q) {
        uint32_t* sub[kMaxWords];
        for (int k = 0; k < nw; ++k) sub[k] = words[k] + h[2 * q];
        radix_sort_words(ctx, sub, nw, h[2 * q + 1] - h[2 * q], all_full, nullptr, false);
    }
}

// ZI_SORT_VERIFY: check the (layout, Morton key, payload) order of the finished records on the host
static void verify_sorted(zi_ctx* ctx, uint32_t* const* words, int W, uint64_t N, int D, int nb, bool layouts) {
    const int nw = W + 1;
    std::vector<std::vector<uint32_t>> h(nw, std::vector<uint32_t>(N));
    for (int k = 0; k < nw; ++k)
        ZI_CUDA(cudaMemcpyAsync(h[k].data(), words[k], N * sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
    ZI_CUDA(cudaStreamSynchronize(ctx->stream));
    auto less = [&](uint64_t a, uint64_t b) {
        if (layouts && (h[W][a] >> 29) != (h[W][b] >> 29)) return (h[W][a] >> 29) < (h[W][b] >> 29);
        for (int k = W - 1; k >= 0; --k)
            if (h[k][a] != h[k][b]) return h[k][a] < h[k][b];
        return h[W][a] < h[W][b];
    };
    for (uint64_t i = 1; i < N; ++i)
        if (!less(i - 1, i)) {
            std::fprintf(stderr, "ZI_SORT_VERIFY: order broken at %llu of %llu (D=%d nb=%d layouts=%d)\n",
                         static_cast<unsigned long long>(i), static_cast<unsigned long long>(N), D, nb, layouts ? 1 : 0);
            for (uint64_t j = i > 3 ? i - 3 : 0; j < std::min<uint64_t>(N, i + 3); ++j) {
                std::fprintf(stderr, "  [%llu]", static_cast<unsigned long long>(j));
                for (int k = nw - 1; k >= 0; --k) std::fprintf(stderr, " %08x", h[k][j]);
                std::fprintf(stderr, "\n");
            }
            throw error(ZI_E_CUDA, "hybrid sort order broken");
        }
}

// Sort (key words, payload) records by (Morton key, payload); `layouts`: the payload's top 3
// bits are a layout id that orders first.
// result (optional, see radix_sort_words): the buffers holding the sorted records
// G > 1 (layouts): the records are G equal layout groups, group-major -- every global pass sorts
// the groups on their own, so no pass on the layout digit is needed
static bool fusable_dims(int D) { return D % 4 == 0 && D <= 16 && !lookback_mode(); }

// true when the 8-layout build sort of these dims goes straight to device LSD passes (an earlier
// build found its top bytes too clustered for the MSD split): its last pass can take a sink
bool layouts_sort_fuses(zi_ctx* ctx, int D) {
    return ctx->sort_depth[D][1] < 0 && msd_bytes_forced() <= 0 && fusable_dims(D);
}

static bool morton_sort_hybrid(zi_ctx* ctx, uint32_t** words, int W, uint64_t N, int D, bool layouts,
                               uint32_t** result = nullptr, int G = 1, const final_sink* sink = nullptr) {
    const int nw = W + 1;
    uint32_t* cur[kMaxWords];
    auto done = [&] {  // hand the final buffers to the caller, or move them into `words`
        if (result) {
            for (int k = 0; k < nw; ++k) result[k] = cur[k];
        } else if (cur[0] != words[0]) {
            for (int k = 0; k < nw; ++k)
                ZI_CUDA(cudaMemcpyAsync(words[k], cur[k], N * sizeof(uint32_t), cudaMemcpyDeviceToDevice, ctx->stream));
        }
    };
    if (G > 1 && (!layouts || N % G != 0 || !groups_fit(D, G))) G = 1;
    std::vector<int2> all, all_full;
    for (int p = 0; p < D; ++p) all.push_back(make_int2(p >> 2, (p & 3) * 8));
    all_full = all;
    if (layouts) all_full.push_back(make_int2(W, 29));
    if (G == 1) all = all_full;
    int& learnt = ctx->sort_depth[D][layouts ? 1 : 0];
    if (learnt > 0 && msd_bytes_forced() <= 0 && learnt <= D - 3) {
        // depth known from an earlier build: MSD passes with device-side digit bases, no
        // histogram round trip to the host
        const int nb = learnt;
        std::vector<int2> msd;
        for (int p = D - nb; p < D; ++p) msd.push_back(make_int2(p >> 2, (p & 3) * 8));
        if (layouts && G == 1) msd.push_back(make_int2(W, 29));
        radix_sort_words(ctx, words, nw, N, msd, nullptr, true, cur, G);
        finish_hybrid(ctx, cur, words, W, N, D, nb, layouts, all, all_full, G, learnt);
        if (verify_on()) verify_sorted(ctx, cur, W, N, D, nb, layouts);
        done();
        return false;
    }
    if (learnt < 0 && msd_bytes_forced() <= 0) {
        // an earlier build with these dims found the top bytes too clustered for the MSD split:
        // the plain LSD sort, every pass on the device (no histogram round trip); with a sink the
        // last pass writes the layout indices themselves
        const bool fused = sink && G == 8 && fusable_dims(D);
        radix_sort_words(ctx, words, nw, N, all, nullptr, true, cur, G, fused ? sink : nullptr);
        if (fused) return true;
        done();
        return false;
    }
    const std::vector<uint32_t> hist = pass_histograms(ctx, words, nw, N, all, G);  // [pass][group][256]
    // MSD depth: the fewest top bytes whose (marginal) entropies predict segments of <= 16
    // records per layout; a clustered top (smooth images) pushes it up, and when the split
    // would leave little for the windows the plain LSD sort is used.
    auto entropy = [&](int q) {
        double e = 0.0;
        for (int b = 0; b < 256; ++b) {
            uint64_t c = 0;
            for (int g = 0; g < G; ++g) c += hist[(static_cast<size_t>(q) * G + g) * 256 + b];
            const double pr = static_cast<double>(c) / static_cast<double>(N);
            if (pr > 0) e -= pr * std::log2(pr);
        }
        return e;
    };
    const double per_layout = static_cast<double>(N) / (layouts ? 8.0 : 1.0);
    int nb = msd_bytes_forced();
    if (nb <= 0 && learnt != 0) nb = learnt < 0 ? D : learnt;
    if (nb <= 0) {
        double bits = 0.0;
        nb = 0;
        while (nb < D && std::exp2(bits) * 16.0 < per_layout) {
            bits += entropy(D - 1 - nb);
            ++nb;
        }
        nb = std::max(nb, 2);
    }
    nb = std::min(nb, D);
    static const bool debug = std::getenv("ZI_DEBUG_SORT") != nullptr;
    if (nb > D - 3) {  // little left for the windows: all-LSD with the histograms already taken
        if (debug) std::fprintf(stderr, "hybrid sort N=%llu: MSD depth %d of %d -> LSD\n", static_cast<unsigned long long>(N), nb, D);
        radix_sort_words(ctx, words, nw, N, all, hist.data(), false, cur, G);
        done();
        return false;
    }
    std::vector<int2> msd;
    std::vector<uint32_t> msd_hist;
    const size_t qw = static_cast<size_t>(G) * 256;  // histogram words per pass
    for (int p = D - nb; p < D; ++p) {
        msd.push_back(make_int2(p >> 2, (p & 3) * 8));
        msd_hist.insert(msd_hist.end(), hist.begin() + static_cast<size_t>(p) * qw, hist.begin() + static_cast<size_t>(p + 1) * qw);
    }
    if (layouts && G == 1) {
        msd.push_back(make_int2(W, 29));
        msd_hist.insert(msd_hist.end(), hist.begin() + static_cast<size_t>(D) * qw, hist.end());
    }
    radix_sort_words(ctx, words, nw, N, msd, msd_hist.data(), false, cur, G);
    if (learnt == 0) learnt = nb;  // remembered: later builds skip the histogram round trip
    finish_hybrid(ctx, cur, words, W, N, D, nb, layouts, all, all_full, G, learnt);
    if (verify_on()) verify_sorted(ctx, cur, W, N, D, nb, layouts);
    done();
    return false;
}

void morton_sort(zi_ctx* ctx, uint32_t* d_keyw, uint32_t* d_val, uint64_t n, int D, bool payload_first) {
    const int W = (D + 3) / 4;
    uint32_t* words[kMaxWords];
    for (int k = 0; k < W; ++k) words[k] = d_keyw + static_cast<size_t>(k) * n;
    words[W] = d_val;
    std::vector<int2> passes;
    if (payload_first)
        for (int b = 0; b < 4; ++b) passes.push_back(make_int2(W, 8 * b));
    for (int p = 0; p < D; ++p) passes.push_back(make_int2(p >> 2, (p & 3) * 8));
    radix_sort_words(ctx, words, W + 1, n, passes, nullptr, false);
}

void morton_sort_rows(zi_ctx* ctx, uint32_t* d_keyw, uint32_t* d_val, uint64_t n, int D) {
    const int W = (D + 3) / 4;
    uint32_t* words[kMaxWords];
    for (int k = 0; k < W; ++k) words[k] = d_keyw + static_cast<size_t>(k) * n;
    words[W] = d_val;
    morton_sort_hybrid(ctx, words, W, n, D, false);
}

bool morton_sort_records(zi_ctx* ctx, uint32_t* d_keyw, uint32_t* d_val, uint64_t n, int G, int D,
                         bool group_in_payload, uint32_t** out, bool payload_ascending, const final_sink* sink) {
    const int W = (D + 3) / 4;
    const uint64_t N = static_cast<uint64_t>(G) * n;
    static const bool splitter = [] {
        const char* e = std::getenv("ZI_SORT");
        return e != nullptr && std::strcmp(e, "splitter") == 0;
    }();
    if (splitter && payload_ascending) {  // experimental: k_ssort.cu
        uint32_t* words[kMaxWords];
        for (int k = 0; k < W; ++k) words[k] = d_keyw + static_cast<size_t>(k) * N;
        words[W] = d_val;
        sample_sort_groups(ctx, words, W + 1, n, G, D, group_in_payload, out);
        return false;
    }
    if (G > 1) {  // layout groups sorted on their own: no layout-digit pass
        uint32_t* words[kMaxWords];
        for (int k = 0; k < W; ++k) words[k] = d_keyw + static_cast<size_t>(k) * N;
        words[W] = d_val;
        return morton_sort_hybrid(ctx, words, W, N, D, group_in_payload, out, G, sink);
    }
    if (payload_ascending) {  // hybrid MSD + window sort, stable: payload order ties
        uint32_t* words[kMaxWords];
        for (int k = 0; k < W; ++k) words[k] = d_keyw + static_cast<size_t>(k) * n;
        words[W] = d_val;
        morton_sort_hybrid(ctx, words, W, n, D, false, out);
        return false;
    }
    morton_sort(ctx, d_keyw, d_val, n, D, true);  // payload passes first: any input order
    for (int k = 0; k < W; ++k) out[k] = d_keyw + static_cast<size_t>(k) * n;
    out[W] = d_val;
    return false;
}

void finalize_index_bboxes(zi_ctx* ctx, zi_index* const* idx, int nidx) {
    if (nidx <= 0 || idx[0]->n == 0) return;
    bbox_job J{};
    for (int l = 0; l < nidx; ++l) {
        J.planes[l] = idx[l]->planes.p;
        J.bmin[l] = idx[l]->bbox_min.p;
        J.bmax[l] = idx[l]->bbox_max.p;
    }
    const uint64_t nblk = idx[0]->nblk;
    const uint64_t kbb = idx[0]->planes_n <= 2 ? 4 : 2;  // blocks per warp (k_index_bbox)
    const unsigned grid = static_cast<unsigned>((((nblk + kbb - 1) / kbb) * nidx + 7) / 8);
    switch (idx[0]->planes_n) {
#define ZI_BBOX_CASE(PP)                                                                                        \
    case PP:                                                                                                    \
        ZI_LAUNCH(ctx, "index_bbox", k_index_bbox<PP>, grid, 256, 0, J, idx[0]->n, nblk, nidx);                 \
        break;
        ZI_BBOX_CASE(1) ZI_BBOX_CASE(2) ZI_BBOX_CASE(3) ZI_BBOX_CASE(4)
#undef ZI_BBOX_CASE
        default: throw error(ZI_E_INVALID, "index bboxes: more than 16 dims");
    }
}

void morton_sort_layouts(zi_ctx* ctx, uint32_t* d_keyw, uint32_t* d_val, uint64_t N, int D, uint32_t** out) {
    const int W = (D + 3) / 4;
    uint32_t* words[kMaxWords];
    for (int k = 0; k < W; ++k) words[k] = d_keyw + static_cast<size_t>(k) * N;
    words[W] = d_val;
    morton_sort_hybrid(ctx, words, W, N, D, true, out);
}

}  // namespace zi
