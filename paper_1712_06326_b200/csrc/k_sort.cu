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
#include <vector>

#include "common.cuh"

namespace zi {

constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;
constexpr int kSortTile = kSortThreads * kSortItems;  // 4096
constexpr int kSortWarps = kSortThreads / 32;
constexpr uint32_t kFlagAgg = 1u << 30, kFlagInc = 2u << 30, kValMask = (1u << 30) - 1;
constexpr int kMaxWords = 9;  // up to 8 Morton key words (D <= 32) + payload

struct sort_words {
    const uint32_t* in[kMaxWords];
    uint32_t* out[kMaxWords];
};

// Histograms of every pass in one read: hist[q*256 + digit]
__global__ void __launch_bounds__(256) k_sort_hist(sort_words io, int npass, const int2* __restrict__ passes,
                                                   uint64_t n, uint32_t* __restrict__ hist) {
    extern __shared__ uint32_t s_hist[];  // npass*256
    __shared__ int2 s_pass[40];
    for (int i = threadIdx.x; i < npass * 256; i += blockDim.x) s_hist[i] = 0;
    if (threadIdx.x < npass) s_pass[threadIdx.x] = passes[threadIdx.x];
    __syncthreads();
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        for (int q = 0; q < npass; ++q) {
            const uint32_t d = (io.in[s_pass[q].x][i] >> s_pass[q].y) & 0xffu;
            atomicAdd(&s_hist[q * 256 + d], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < npass * 256; i += blockDim.x)
        if (s_hist[i]) atomicAdd(&hist[i], s_hist[i]);
}

template <int NW>
__global__ void __launch_bounds__(kSortThreads) k_onesweep(sort_words io, int dw, int ds,
                                                           const uint32_t* __restrict__ digit_base,
                                                           uint32_t* __restrict__ status,
                                                           uint32_t* __restrict__ tile_ctr, uint64_t n) {
    extern __shared__ uint32_t s_stage[];  // NW * kSortTile
    __shared__ uint32_t s_hist[kSortWarps][256];
    __shared__ uint32_t s_start[256];
    __shared__ uint32_t s_gofs[256];
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_tile;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < kSortWarps * 256; i += kSortThreads) (&s_hist[0][0])[i] = 0;
    if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint64_t tbase = static_cast<uint64_t>(tile) * kSortTile;
    const uint64_t wbase = tbase + warp * (kSortItems * 32);

    // every word of the tile's records is loaded up front (maximum loads in flight)
    uint32_t rec[kSortItems][NW];
    uint32_t dig[kSortItems];
    uint32_t rank[kSortItems];
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
        const uint64_t idx = wbase + i * 32 + lane;
        const bool ok = idx < n;
#pragma unroll
        for (int k = 0; k < NW; ++k) rec[i][k] = ok ? io.in[k][idx] : 0u;
        // (a second, L1-hitting load of the digit word: selecting it from rec[] by the runtime
        // dw makes the compiler spill rec[] to local memory)
        dig[i] = ok ? (__ldg(io.in[dw] + idx) >> ds) & 0xffu : 0x100u;
    }
    const uint32_t lt_mask = (1u << lane) - 1u;
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
        const uint32_t d = dig[i];
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        uint32_t old = 0;
        if (d < 256u) old = s_hist[warp][d];
        __syncwarp();
        if (d < 256u && (peers >> lane) == 1u) s_hist[warp][d] = old + __popc(peers);
        __syncwarp();
        rank[i] = old + __popc(peers & lt_mask);
    }
    __syncthreads();

    // per-digit: warp exclusive offsets + tile count
    const int d = tid;
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
        const uint32_t t = s_hist[w][d];
        s_hist[w][d] = run;
        run += t;
    }
    const uint32_t tile_cnt = run;
    volatile uint32_t* vstatus = status;
    if (tile == 0) vstatus[d] = kFlagInc | tile_cnt;
    else vstatus[static_cast<size_t>(tile) * 256 + d] = kFlagAgg | tile_cnt;

    // tile-local exclusive scan over digits
    {
        uint32_t x = tile_cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_warp[warp] = x;
        __syncthreads();
        uint32_t wp = 0;
        for (int w = 0; w < warp; ++w) wp += s_warp[w];
        s_start[d] = wp + x - tile_cnt;
    }

    // decoupled look-back for the prefix of digit d over the previous tiles
    uint32_t prefix = 0;
    if (tile > 0) {
        int64_t j = static_cast<int64_t>(tile) - 1;
        while (true) {
            const uint32_t v = vstatus[static_cast<size_t>(j) * 256 + d];
            const uint32_t flag = v & ~kValMask;
            if (flag == 0) continue;  // predecessor not yet published
            prefix += v & kValMask;
            if (flag == kFlagInc) break;
            --j;
        }
        vstatus[static_cast<size_t>(tile) * 256 + d] = kFlagInc | (prefix + tile_cnt);
    }
    s_gofs[d] = digit_base[d] + prefix;
    __syncthreads();

    // stage records in tile-sorted order
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
        if (dig[i] < 256u) {
            const uint32_t pos = s_start[dig[i]] + s_hist[warp][dig[i]] + rank[i];
#pragma unroll
            for (int k = 0; k < NW; ++k) s_stage[k * kSortTile + pos] = rec[i][k];
        }
    }
    __syncthreads();
    const uint32_t cnt = static_cast<uint32_t>(n - tbase < static_cast<uint64_t>(kSortTile) ? n - tbase : kSortTile);
    for (uint32_t j = tid; j < cnt; j += kSortThreads) {
        const uint32_t dd = (s_stage[dw * kSortTile + j] >> ds) & 0xffu;
        const uint64_t o = static_cast<uint64_t>(s_gofs[dd]) + (j - s_start[dd]);
#pragma unroll
        for (int k = 0; k < NW; ++k) io.out[k][o] = s_stage[k * kSortTile + j];
    }
}

template <int NW>
static void launch_onesweep(zi_ctx* ctx, const sort_words& io, int dw, int ds, const uint32_t* base, uint32_t* status,
                            uint32_t* ctr, uint64_t n, unsigned ntiles) {
    const size_t smem = static_cast<size_t>(NW) * kSortTile * sizeof(uint32_t);
    static bool attr = false;
    if (!attr) {
        ZI_CUDA(cudaFuncSetAttribute(k_onesweep<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(kMaxWords * kSortTile * sizeof(uint32_t))));
        attr = true;
    }
    ZI_LAUNCH(ctx, "radix_onesweep", k_onesweep<NW>, ntiles, kSortThreads, smem, io, dw, ds, base, status, ctr, n);
}

// Generic stable LSD sort of NW-word SoA records; passes are (word, shift) digits from the
// least significant.  Trivial passes (all records share the digit) are skipped.
void radix_sort_words(zi_ctx* ctx, uint32_t** words, int nw, uint64_t n, const std::vector<int2>& passes) {
    if (n <= 1 || passes.empty()) return;
    if (n > kValMask) throw error(ZI_E_INVALID, "radix sort: more than 2^30 records");
    if (nw > kMaxWords) throw error(ZI_E_INVALID, "radix sort: too many words");
    const int npass = static_cast<int>(passes.size());
    const unsigned ntiles = static_cast<unsigned>((n + kSortTile - 1) / kSortTile);
    // scratch layout: alt words (nw*n) | hist (npass*256) | bases (npass*256) | status (npass*ntiles*256) | ctr
    const size_t alt_words = static_cast<size_t>(nw) * n;
    const size_t hist_words = static_cast<size_t>(npass) * 256;
    const size_t status_words = static_cast<size_t>(npass) * ntiles * 256;
    uint32_t* scr = reinterpret_cast<uint32_t*>(
        ctx->scratch.ensure((alt_words + 2 * hist_words + status_words + 4 * npass + 64) * sizeof(uint32_t)));
    uint32_t* alt = scr;
    uint32_t* hist = alt + alt_words;
    uint32_t* bases = hist + hist_words;
    uint32_t* status = bases + hist_words;
    uint32_t* ctr = status + status_words;
    int2* d_passes = reinterpret_cast<int2*>(ctr + npass + 8);  // tiny
    d_passes = reinterpret_cast<int2*>((reinterpret_cast<uintptr_t>(d_passes) + 15) & ~uintptr_t(15));

    ZI_CUDA(cudaMemsetAsync(hist, 0, hist_words * sizeof(uint32_t), ctx->stream));
    ZI_CUDA(cudaMemcpyAsync(d_passes, passes.data(), passes.size() * sizeof(int2), cudaMemcpyHostToDevice, ctx->stream));
    sort_words io{};
    for (int k = 0; k < nw; ++k) {
        io.in[k] = words[k];
        io.out[k] = alt + static_cast<size_t>(k) * n;
    }
    {
        const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(ctx->num_sms) * 4));
        ZI_LAUNCH(ctx, "radix_hist", k_sort_hist, grid, 256, hist_words * sizeof(uint32_t), io, npass, d_passes, n, hist);
    }
    std::vector<uint32_t> h_hist(hist_words);
    ZI_CUDA(cudaMemcpyAsync(h_hist.data(), hist, hist_words * sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
    ZI_CUDA(cudaStreamSynchronize(ctx->stream));
    std::vector<int> active;
    std::vector<uint32_t> h_bases(hist_words, 0);
    for (int q = 0; q < npass; ++q) {
        bool trivial = false;
        uint32_t run = 0;
        for (int dgt = 0; dgt < 256; ++dgt) {
            const uint32_t c = h_hist[q * 256 + dgt];
            if (c == n) trivial = true;
            h_bases[q * 256 + dgt] = run;
            run += c;
        }
        if (!trivial) active.push_back(q);
    }
    if (active.empty()) return;
    ZI_CUDA(cudaMemcpyAsync(bases, h_bases.data(), hist_words * sizeof(uint32_t), cudaMemcpyHostToDevice, ctx->stream));
    ZI_CUDA(cudaMemsetAsync(status, 0, status_words * sizeof(uint32_t), ctx->stream));
    ZI_CUDA(cudaMemsetAsync(ctr, 0, npass * sizeof(uint32_t), ctx->stream));
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
        uint32_t* st = status + static_cast<size_t>(q) * ntiles * 256;
        switch (nw) {
            case 2: launch_onesweep<2>(ctx, io, passes[q].x, passes[q].y, bases + q * 256, st, ctr + q, n, ntiles); break;
            case 3: launch_onesweep<3>(ctx, io, passes[q].x, passes[q].y, bases + q * 256, st, ctr + q, n, ntiles); break;
            case 4: launch_onesweep<4>(ctx, io, passes[q].x, passes[q].y, bases + q * 256, st, ctr + q, n, ntiles); break;
            case 5: launch_onesweep<5>(ctx, io, passes[q].x, passes[q].y, bases + q * 256, st, ctr + q, n, ntiles); break;
            case 6: launch_onesweep<6>(ctx, io, passes[q].x, passes[q].y, bases + q * 256, st, ctr + q, n, ntiles); break;
            case 7: launch_onesweep<7>(ctx, io, passes[q].x, passes[q].y, bases + q * 256, st, ctr + q, n, ntiles); break;
            case 8: launch_onesweep<8>(ctx, io, passes[q].x, passes[q].y, bases + q * 256, st, ctr + q, n, ntiles); break;
            case 9: launch_onesweep<9>(ctx, io, passes[q].x, passes[q].y, bases + q * 256, st, ctr + q, n, ntiles); break;
            default: throw error(ZI_E_INVALID, "radix sort: unsupported record width");
        }
        for (int k = 0; k < nw; ++k) std::swap(cur[k], oth[k]);
    }
    if (active.size() % 2 == 1)
        for (int k = 0; k < nw; ++k)
            ZI_CUDA(cudaMemcpyAsync(words[k], cur[k], n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, ctx->stream));
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
    radix_sort_words(ctx, words, W + 1, n, passes);
}

void morton_sort_layouts(zi_ctx* ctx, uint32_t* d_keyw, uint32_t* d_val, uint64_t N, int D) {
    const int W = (D + 3) / 4;
    uint32_t* words[kMaxWords];
    for (int k = 0; k < W; ++k) words[k] = d_keyw + static_cast<size_t>(k) * N;
    words[W] = d_val;
    std::vector<int2> passes;
    for (int p = 0; p < D; ++p) passes.push_back(make_int2(p >> 2, (p & 3) * 8));
    passes.push_back(make_int2(W, 29));  // layout id (3 bits)
    radix_sort_words(ctx, words, W + 1, N, passes);
}

}  // namespace zi
