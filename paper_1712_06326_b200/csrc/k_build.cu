// k_build.cu -- index-construction kernels (sm_100a):
//   K1 collect_dictionary   proj/src/builder.cpp:74-108
//   K2 patch_moments        proj/src/pca.cpp:20-37 (exact integer restatement)
//   K3 project / quantize   proj/src/builder.cpp:159-187, :55-61
//   K5 finalize_index       proj/src/zcurve.cpp:127-137 (+ per-block bounding boxes)
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "common.cuh"

namespace zi {

// ============================================================== K1: dictionary collection
// colflag[y][x] = 1 iff any unknown pixel in column x, rows y..y+K-1
__global__ void k_colflag(const uint8_t* __restrict__ known, int w, int h, int K,
                          uint8_t* __restrict__ colflag) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    if (x >= w) return;
    uint8_t any = 0;
    for (int r = 0; r < K; ++r) any |= known[static_cast<size_t>(y + r) * w + x] == 0;
    colflag[static_cast<size_t>(y) * w + x] = any;
}

// valid[y][x] (x < w-K+1) = no flagged column among x..x+K-1
__global__ void k_validflag(const uint8_t* __restrict__ colflag, int w, int K, int wo,
                            uint8_t* __restrict__ valid) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    if (x >= wo) return;
    uint8_t any = 0;
    const uint8_t* row = colflag + static_cast<size_t>(y) * w + x;
    for (int c = 0; c < K; ++c) any |= row[c];
    valid[static_cast<size_t>(y) * wo + x] = any ? 0 : 1;
}

// Both window flags in one pass for word-aligned rows (w % 4 == 0, K <= KMAX): a thread makes the
// valid flags x .. x+3 of R consecutive rows from the (R + K - 1) x (K + 3) mask bytes above them,
// read once as aligned words: f = byte-wise (known == 0); the column flags of an output row are
// the OR of its K rows of f, the valid flag of byte j the OR of the column bytes j .. j+K-1 (funnel
// shifts of the flag words).  No colflag array, word loads, every mask word loaded once per thread.
template <int KMAX, int R>
__global__ void __launch_bounds__(256) k_validfused(const uint8_t* __restrict__ known, int w, int K, int wo, int ho,
                                                    uint8_t* __restrict__ valid) {
    constexpr int NW = (KMAX + 6) / 4;  // words covering K + 3 bytes
    constexpr int NR = R + KMAX - 1;
    const int x = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
    const int y0 = blockIdx.y * R;
    if (x >= wo) return;
    const int nw = (K + 6) >> 2;
    uint32_t f[NR][NW];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        const bool rok = r < R + K - 1 && y0 + r < ho + K - 1;
        const uint32_t* row = reinterpret_cast<const uint32_t*>(known + static_cast<size_t>(y0 + r) * w + x);
#pragma unroll
        for (int i = 0; i < NW; ++i) f[r][i] = (rok && i < nw && x + 4 * i < w) ? __vcmpeq4(__ldg(row + i), 0u) : 0u;
    }
#pragma unroll
    for (int j = 0; j < R; ++j) {
        if (y0 + j >= ho) break;
        uint32_t c[NW + 1];
#pragma unroll
        for (int i = 0; i < NW; ++i) {
            uint32_t v = 0u;
#pragma unroll
            for (int r = 0; r < KMAX; ++r)
                if (r < K) v |= f[j + r][i];
            c[i] = v;
        }
        c[NW] = 0u;
        uint32_t any = 0u;
#pragma unroll
        for (int k = 0; k < KMAX; ++k)
            if (k < K) any |= (k & 3) ? __funnelshift_r(c[k >> 2], c[(k >> 2) + 1], 8 * (k & 3)) : c[k >> 2];
        const uint32_t ok = ~any & 0x01010101u;  // __vcmpeq4 gives 0xff per equal byte
        const size_t o = static_cast<size_t>(y0 + j) * wo + x;
        if (x + 3 < wo && (o & 3) == 0) {
            *reinterpret_cast<uint32_t*>(valid + o) = ok;
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (x + q < wo) valid[o + q] = static_cast<uint8_t>((ok >> (8 * q)) & 1u);
        }
    }
}

constexpr int kCompactThreads = 256;
constexpr int kCompactPer = 16;
constexpr int kCompactTile = kCompactThreads * kCompactPer;  // 4096 flags per block

__device__ inline uint32_t block_exclusive_scan(uint32_t v, uint32_t* s_warp, uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        uint32_t t = lane < nw ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        if (lane < nw) s_warp[lane] = t;  // inclusive per-warp totals
    }
    __syncthreads();
    const uint32_t warp_prefix = warp ? s_warp[warp - 1] : 0;
    if (total) *total = s_warp[(blockDim.x >> 5) - 1];
    const uint32_t r = warp_prefix + x - v;
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kCompactThreads) k_count_flags(const uint8_t* __restrict__ flags, uint64_t n,
                                                                 uint32_t* __restrict__ counts) {
    __shared__ uint32_t s_warp[32];
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kCompactTile + threadIdx.x * kCompactPer;
    uint32_t c = 0;
    for (int i = 0; i < kCompactPer; ++i) c += (base + i < n) ? flags[base + i] : 0;
    uint32_t total;
    block_exclusive_scan(c, s_warp, &total);
    if (threadIdx.x == 0) counts[blockIdx.x] = total;
}

// single-CTA exclusive scan of nb block counts (in place); total -> counts[nb]
__global__ void __launch_bounds__(1024) k_scan_counts(uint32_t* counts, uint64_t nb) {
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (uint64_t b = 0; b < nb; b += 1024) {
        const uint64_t i = b + threadIdx.x;
        const uint32_t v = i < nb ? counts[i] : 0;
        uint32_t total;
        const uint32_t ex = block_exclusive_scan(v, s_warp, &total);
        if (i < nb) counts[i] = s_carry + ex;
        __syncthreads();
        if (threadIdx.x == 0) s_carry += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) counts[nb] = s_carry;
}

__global__ void __launch_bounds__(kCompactThreads) k_write_keys(const uint8_t* __restrict__ flags, uint64_t n,
                                                                int wo, const uint32_t* __restrict__ offsets,
                                                                uint32_t* __restrict__ keys) {
    __shared__ uint32_t s_warp[32];
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kCompactTile + threadIdx.x * kCompactPer;
    static_assert(kCompactPer == 16, "one 16-byte vector of flags per thread");
    uint8_t f[kCompactPer];
    uint32_t c = 0;
    if (base + kCompactPer <= n && (reinterpret_cast<uintptr_t>(flags + base) & 15) == 0) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(flags + base));
        const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < kCompactPer; ++i) {
            f[i] = static_cast<uint8_t>((wv[i >> 2] >> (8 * (i & 3))) & 0xffu);
            c += f[i];
        }
    } else {
        for (int i = 0; i < kCompactPer; ++i) {
            f[i] = (base + i < n) ? flags[base + i] : 0;
            c += f[i];
        }
    }
    // the block's keys are collected in shared memory and written as one contiguous run
    __shared__ uint32_t s_keys[kCompactTile];
    uint32_t total;
    uint32_t pos = block_exclusive_scan(c, s_warp, &total);
    // (row, column) of the thread's first flag by one division, then stepped
    uint32_t y = static_cast<uint32_t>(base / wo), x = static_cast<uint32_t>(base - static_cast<uint64_t>(y) * wo);
#pragma unroll
    for (int i = 0; i < kCompactPer; ++i) {
        if (f[i]) s_keys[pos++] = (y << 16) | x;
        if (++x == static_cast<uint32_t>(wo)) {
            x = 0;
            ++y;
        }
    }
    __syncthreads();
    uint32_t* dst = keys + offsets[blockIdx.x];
    for (uint32_t i = threadIdx.x; i < total; i += kCompactThreads) dst[i] = s_keys[i];
}

uint64_t collect_dictionary(zi_ctx* ctx, const uint8_t* d_known, int w, int h, int K,
                            dbuf<uint32_t>& keys_out) {
    if (w < K || h < K) return 0;
    const int ho = h - K + 1, wo = w - K + 1;
    const uint64_t n_orig = static_cast<uint64_t>(ho) * wo;
    const uint64_t nb = (n_orig + kCompactTile - 1) / kCompactTile;
    // scratch: colflag (ho*w) + valid (n_orig) + counts (nb+1)
    const size_t sz_col = static_cast<size_t>(ho) * w, sz_valid = n_orig;
    uint8_t* base = ctx->scratch.ensure(sz_col + sz_valid + 16 + (nb + 1) * sizeof(uint32_t) + 16);
    uint8_t* colflag = base;
    uint8_t* valid = base + sz_col;
    uint32_t* counts = reinterpret_cast<uint32_t*>(base + ((sz_col + sz_valid + 15) & ~size_t(15)));
    if ((w & 3) == 0 && K <= 17 && (reinterpret_cast<uintptr_t>(d_known) & 3) == 0 && (reinterpret_cast<uintptr_t>(valid) & 3) == 0) {
        const unsigned gx = static_cast<unsigned>(((wo + 3) / 4 + 255) / 256);
        if (K <= 9)
            ZI_LAUNCH(ctx, "collect_validflag", (k_validfused<9, 8>), dim3(gx, (ho + 7) / 8), 256, 0, d_known, w, K, wo, ho, valid);
        else
            ZI_LAUNCH(ctx, "collect_validflag", (k_validfused<17, 2>), dim3(gx, (ho + 1) / 2), 256, 0, d_known, w, K, wo, ho, valid);
    } else {
        ZI_LAUNCH(ctx, "collect_colflag", k_colflag, dim3((w + 255) / 256, ho), 256, 0, d_known, w, h, K, colflag);
        ZI_LAUNCH(ctx, "collect_validflag", k_validflag, dim3((wo + 255) / 256, ho), 256, 0, colflag, w, K, wo, valid);
    }
    ZI_LAUNCH(ctx, "collect_count", k_count_flags, dim3(static_cast<unsigned>(nb)), kCompactThreads, 0, valid,
              n_orig, counts);
    ZI_LAUNCH(ctx, "collect_scan", k_scan_counts, 1, 1024, 0, counts, nb);
    uint32_t total = 0;
    ZI_CUDA(cudaMemcpyAsync(&total, counts + nb, sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
    ZI_CUDA(cudaStreamSynchronize(ctx->stream));
    keys_out.ensure(total ? total : 1);
    if (total)
        ZI_LAUNCH(ctx, "collect_write", k_write_keys, dim3(static_cast<unsigned>(nb)), kCompactThreads, 0, valid,
                  n_orig, wo, counts, keys_out.p);
    return total;
}

// ============================================================== K2: exact patch moments
// S = sum_p x_p x_p^T and s = sum_p x_p over the full K*K*C patch vectors (u8), exact.
// Two kernels:
//   k_patch_matrix  the feature-major patch matrix XT[f][p] (Fpad x npad u8, zero padded) in HBM:
//                   one warp writes one feature x 128 consecutive patches (one coalesced 128 B
//                   store), reading adjacent pixels of the image (L1/L2 resident).
//   k_moments       X^T X on the tensor cores (mma.sync m16n8k32 u8 x u8 -> s32): one CTA = one
//                   128x128 feature tile pair (ti <= tj) x one patch chunk; 128-patch stages
//                   stream in with cp.async (3-stage ring, 144 B pitch -> conflict-free ldmatrix).
//                   Chunks hold <= 65536 patches so the s32 accumulators, read as u32, are exact
//                   (65536 * 255^2 < 2^32); chunk partials go into int64 with atomics
//                   (order-free -> deterministic).
constexpr int kMomTile = 128;
constexpr int kMomStage = 128;              // patches per stage (four k32 MMA steps)
constexpr int kMomStages = 3;
constexpr int kMomPitch = kMomStage + 16;   // 144 B rows: 36 words -> conflict-free 8x16B reads
constexpr uint64_t kMomMaxChunk = 65536;

__device__ inline void mma_u8_16832(int (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

__device__ inline void ldmatrix_x4(uint32_t (&r)[4], const void* p) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(a));
}

__device__ inline void cp_async16(void* dst, const void* src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ inline void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ inline void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__global__ void __launch_bounds__(256) k_patch_matrix(const uint8_t* __restrict__ img, int w, int C, int K, int F,
                                                      const uint32_t* __restrict__ keys, uint64_t n, uint64_t npad,
                                                      int Fpad, uint8_t* __restrict__ XT) {
    extern __shared__ int s_off[];  // Fpad byte offsets (-1: zero row, -2: the ones row F)
    __shared__ int s_base[128];
    const int tid = threadIdx.x;
    const uint64_t p0 = static_cast<uint64_t>(blockIdx.x) * 128;
    if (tid < 128) {
        const uint64_t p = p0 + tid;
        if (p < n) {
            const uint32_t key = keys[p];
            s_base[tid] = static_cast<int>(((key >> 16) * static_cast<uint32_t>(w) + (key & 0xffffu)) * C);
        } else {
            s_base[tid] = -1;
        }
    }
    for (int f = tid; f < Fpad; f += 256)
        s_off[f] = f < F ? (((f / C) / K) * w + (f / C) % K) * C + f % C : (f == F ? -2 : -1);
    __syncthreads();
    // one warp per feature row, lane l = patches 4l..4l+3: the warp's loads of one feature cover
    // 128 adjacent pixels (a few 128-byte lines per instruction) and it stores 128 contiguous bytes
    const int lane = tid & 31, warp = tid >> 5;
    int bs[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) bs[j] = s_base[4 * lane + j];
    for (int f = warp; f < Fpad; f += 8) {
        const int of = s_off[f];
        uint32_t wv = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint32_t v = 0;
            if (bs[j] >= 0) v = of >= 0 ? static_cast<uint32_t>(__ldg(img + bs[j] + of)) : (of == -2 ? 1u : 0u);
            wv |= v << (8 * j);
        }
        *reinterpret_cast<uint32_t*>(XT + static_cast<size_t>(f) * npad + p0 + 4 * lane) = wv;
    }
}

__global__ void __launch_bounds__(256) k_moments(const uint8_t* __restrict__ XT, uint64_t npad, int F, int ntile,
                                                 uint64_t chunk, unsigned long long* __restrict__ out) {
    extern __shared__ __align__(16) uint8_t sm_mom[];
    int pr = blockIdx.x, ti = 0;
    while (pr >= ntile - ti) {
        pr -= ntile - ti;
        ++ti;
    }
    const int tj = ti + pr;
    const bool diag = ti == tj;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp >> 2, wn = warp & 3;  // warp tile: rows wm*64..+64, cols wn*32..+32
    const uint64_t c0 = static_cast<uint64_t>(blockIdx.y) * chunk;
    const uint64_t c1 = c0 + chunk < npad ? c0 + chunk : npad;
    const int nst = static_cast<int>((c1 - c0) / kMomStage);
    constexpr int kTileBytes = kMomTile * kMomPitch;
    const uint8_t* srcA = XT + static_cast<size_t>(ti) * kMomTile * npad + c0;
    const uint8_t* srcB = XT + static_cast<size_t>(tj) * kMomTile * npad + c0;
    auto load_stage = [&](int st) {
        uint8_t* dA = sm_mom + (st % kMomStages) * 2 * kTileBytes;
        uint8_t* dB = dA + kTileBytes;
        const size_t so = static_cast<size_t>(st) * kMomStage;
#pragma unroll
        for (int e = tid; e < kMomTile * (kMomStage / 16); e += 256) {
            const int r = e >> 3, c16 = (e & 7) * 16;
            cp_async16(dA + r * kMomPitch + c16, srcA + static_cast<size_t>(r) * npad + so + c16);
            if (!diag) cp_async16(dB + r * kMomPitch + c16, srcB + static_cast<size_t>(r) * npad + so + c16);
        }
    };
#pragma unroll
    for (int st = 0; st < kMomStages - 1; ++st) {
        if (st < nst) load_stage(st);
        cp_async_commit();
    }
    int acc[4][4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[a][b][c] = 0;
    uint32_t rs = 0;  // row sum of row `tid` (diagonal CTAs, tid < 128)
    // ldmatrix lane roles: matrix i = lane / 8, row lane % 8
    const int mi = lane >> 3, mr = lane & 7;
    for (int st = 0; st < nst; ++st) {
        cp_async_wait<kMomStages - 2>();
        __syncthreads();  // stage st landed; stage st-1's buffer is free
        if (st + kMomStages - 1 < nst) load_stage(st + kMomStages - 1);
        cp_async_commit();
        const uint8_t* A = sm_mom + (st % kMomStages) * 2 * kTileBytes;
        const uint8_t* B = diag ? A : A + kTileBytes;
#pragma unroll
        for (int kk = 0; kk < kMomStage; kk += 32) {
            uint32_t af[4][4], bq[2][4];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
                ldmatrix_x4(af[mt], A + (wm * 64 + mt * 16 + (mi & 1) * 8 + mr) * kMomPitch + kk + (mi >> 1) * 16);
#pragma unroll
            for (int np = 0; np < 2; ++np)
                ldmatrix_x4(bq[np], B + (wn * 32 + np * 16 + (mi >> 1) * 8 + mr) * kMomPitch + kk + (mi & 1) * 16);
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) {
                    const uint32_t bf[2] = {bq[nt >> 1][(nt & 1) * 2], bq[nt >> 1][(nt & 1) * 2 + 1]};
                    mma_u8_16832(acc[mt][nt], af[mt], bf);
                }
        }
        if (diag && tid < kMomTile) {
            const uint8_t* row = A + tid * kMomPitch;
#pragma unroll
            for (int q = 0; q < kMomStage; q += 16) {
                const uint4 v = *reinterpret_cast<const uint4*>(row + q);
                rs = __dp4a(v.x, 0x01010101u, rs);
                rs = __dp4a(v.y, 0x01010101u, rs);
                rs = __dp4a(v.z, 0x01010101u, rs);
                rs = __dp4a(v.w, 0x01010101u, rs);
            }
        }
    }
    cp_async_wait<0>();
    // flush: D fragment (row g / g+8, cols 2t, 2t+1) of every 16x8 tile
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int fi = ti * kMomTile + wm * 64 + mt * 16 + g + (c >> 1) * 8;
                const int fj = tj * kMomTile + wn * 32 + nt * 8 + 2 * t + (c & 1);
                const unsigned v = static_cast<unsigned>(acc[mt][nt][c]);
                if (fi < F && fj < F && v) atomicAdd(out + F + static_cast<size_t>(fi) * F + fj, static_cast<unsigned long long>(v));
            }
    if (diag && tid < kMomTile && rs) {
        const int fi = ti * kMomTile + tid;
        if (fi < F) atomicAdd(out + fi, static_cast<unsigned long long>(rs));
    }
}

void patch_moments(zi_ctx* ctx, const uint8_t* d_img, int w, int C, int K, const uint32_t* d_keys,
                   uint64_t n, unsigned long long* d_out) {
    const int F = K * K * C;
    ZI_CUDA(cudaMemsetAsync(d_out, 0, (static_cast<size_t>(F) + static_cast<size_t>(F) * F) * sizeof(unsigned long long),
                            ctx->stream));
    if (n == 0) return;
    // the fused tensor-core path (k_proj_tc.cu): no patch matrix in HBM
    if (patch_moments_fused(ctx, d_img, w, C, K, d_keys, n, d_out, ctx->gm_wtab)) return;
    // Fpad > F: row F of XT is all ones over the real patches (G[f][F] = first moments)
    const int ntile = (F + 1 + kMomTile - 1) / kMomTile;
    const int Fpad = ntile * kMomTile;
    const uint64_t npad = (n + kMomStage - 1) / kMomStage * kMomStage;
    uint8_t* XT = ctx->scratch.ensure(static_cast<size_t>(Fpad) * npad);
    ZI_LAUNCH(ctx, "patch_matrix", k_patch_matrix, static_cast<unsigned>(npad / 128), 256, Fpad * sizeof(int), d_img, w,
              C, K, F, d_keys, n, npad, Fpad, XT);
    static const bool use_mma = std::getenv("ZI_MOMENTS_MMA") != nullptr;  // legacy mma.sync path (A/B checks)
    if (!use_mma) {
        gram_u8_tc(ctx, XT, F, Fpad, npad, d_out);
        return;
    }
    const int npairs = ntile * (ntile + 1) / 2;
    // about two CTAs per SM in one wave; stage-aligned chunks of <= 65536 patches
    const uint64_t want = std::max<uint64_t>(1, (2ull * ctx->num_sms + npairs - 1) / npairs);
    uint64_t chunk = (npad + want - 1) / want;
    chunk = std::min<uint64_t>(kMomMaxChunk, (chunk + kMomStage - 1) / kMomStage * kMomStage);
    const uint64_t nchunk = (npad + chunk - 1) / chunk;
    const size_t smem = static_cast<size_t>(kMomStages) * 2 * kMomTile * kMomPitch;
    smem_attr(ctx->device, k_moments, smem);
    ZI_LAUNCH(ctx, "patch_moments", k_moments, dim3(npairs, static_cast<unsigned>(nchunk)), 256, smem, XT, npad, F,
              ntile, chunk, d_out);
}

// ============================================================== K3: projection
// Y[d*n + i] = sum_j fma(comp[j][d], x_ij - mean_j) in the canonical order (j ascending,
// starting from +0.0) -- bit-identical to the oracle's restatement of
// proj/src/builder.cpp:166-167/180-181 (fill_chunk gather order :20-34).
// Projection on the FP64 tensor cores.  mma.sync.m8n8k4.f64 accumulates its four k-products
// into C as four sequential round-to-nearest FMAs in k order -- bit-identical to the canonical
// y = fma(comp[j][d], x_j - mean_j, y), j ascending (checked on B200 with random operands,
// 4M elements, 0 differences; a single-rounding 4-term sum differs in ~40%).  So the canonical
// order runs as Y(8 patches x 8 dims) += Xc(8 x 4 columns) * Comp(4 x 8), k-steps in column
// order; columns past m*C are zero-padded in Comp (fma(x, 0, y) == y since y is never -0).
// A warp owns kProjGroups groups of 8 consecutive dictionary patches (independent accumulator
// chains); lane (r, c) = (lane/4, lane%4) gathers byte x[patch r][column 4*ks + c].
constexpr int kProjThreads = 256;
constexpr int kProjGroups = 4;  // 8-patch groups per warp
constexpr int kProjPF = 3;      // gather prefetch distance (k-steps)

__device__ inline void dmma_8x8x4(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// One warp's G groups of 8 patches starting at dictionary row `base`.
template <int D, int G>
__device__ __forceinline__ void project_groups(const uint8_t* __restrict__ img, int w, int C,
                                               const uint32_t* __restrict__ keys, uint64_t n, uint64_t base, int KS,
                                               const double* s_B, const double* s_mean, const int* s_joff,
                                               double* __restrict__ Y, unsigned long long (*s_mm)[D]) {
    constexpr int NT = (D + 7) / 8;
    const int lane = threadIdx.x & 31, r = lane >> 2, c = lane & 3;
    const uint8_t* pb[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const uint64_t i = base + 8 * g + r;
        const uint32_t key = keys[i < n ? i : n - 1];
        pb[g] = img + static_cast<size_t>((key >> 16) * static_cast<uint32_t>(w) + (key & 0xffffu)) * C;
    }
    double acc[G][NT][2];
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
        for (int t = 0; t < NT; ++t) acc[g][t][0] = acc[g][t][1] = 0.0;
    uint32_t xr[kProjPF][G];
#pragma unroll
    for (int s = 0; s < kProjPF; ++s)
        if (s < KS) {
            const int o = s_joff[s * 4 + c];
#pragma unroll
            for (int g = 0; g < G; ++g) xr[s][g] = __ldg(pb[g] + o);
        }
    for (int ks0 = 0; ks0 < KS; ks0 += kProjPF) {
#pragma unroll
        for (int s = 0; s < kProjPF; ++s) {
            const int ks = ks0 + s;
            if (ks < KS) {
                uint32_t xcur[G];
#pragma unroll
                for (int g = 0; g < G; ++g) xcur[g] = xr[s][g];
                if (ks + kProjPF < KS) {
                    const int o = s_joff[(ks + kProjPF) * 4 + c];
#pragma unroll
                    for (int g = 0; g < G; ++g) xr[s][g] = __ldg(pb[g] + o);
                }
                const double mj = s_mean[ks * 4 + c];
                double bf[NT];
#pragma unroll
                for (int t = 0; t < NT; ++t) bf[t] = s_B[(ks * NT + t) * 32 + lane];
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const double a = __dsub_rn(static_cast<double>(xcur[g]), mj);
#pragma unroll
                    for (int t = 0; t < NT; ++t) dmma_8x8x4(acc[g][t][0], acc[g][t][1], a, bf[t]);
                }
            }
        }
    }
    // lane holds y[patch base + 8g + r][dim 8t + 2c + e]
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

template <int D>
__global__ void __launch_bounds__(kProjThreads) k_project(const uint8_t* __restrict__ img, int w, int C,
                                                          const uint32_t* __restrict__ keys, uint64_t n,
                                                          const int32_t* __restrict__ off, int m,
                                                          const double* __restrict__ mean,
                                                          const double* __restrict__ comp, double* __restrict__ Y,
                                                          unsigned long long* __restrict__ minmax) {
    constexpr int NT = (D + 7) / 8;  // 8-dim tiles
    extern __shared__ double sm[];
    const int mc = m * C, KS = (mc + 3) / 4;
    double* s_B = sm;                                          // [KS][NT][32] B fragments (Comp, zero padded)
    double* s_mean = s_B + static_cast<size_t>(KS) * NT * 32;  // [KS*4]
    int* s_joff = reinterpret_cast<int*>(s_mean + KS * 4);     // [KS*4] byte offset of column j
    for (int idx = threadIdx.x; idx < KS * NT * 32; idx += kProjThreads) {
        const int ks = idx / (NT * 32), t = (idx / 32) % NT, ln = idx % 32;
        const int j = ks * 4 + ln % 4, d = t * 8 + ln / 4;
        s_B[idx] = (j < mc && d < D) ? comp[j * D + d] : 0.0;
    }
    for (int j = threadIdx.x; j < KS * 4; j += kProjThreads) {
        s_mean[j] = j < mc ? mean[j] : 0.0;
        s_joff[j] = j < mc ? off[j / C] + j % C : 0;
    }
    // the quantiser's lo / hi: block-level ordered-u64 min / max in shared memory, folded in
    // with shared atomics as each 8-patch group is stored (no running registers)
    __shared__ unsigned long long s_mm[2][D];
    if (threadIdx.x < 2 * D) s_mm[threadIdx.x / D][threadIdx.x % D] = threadIdx.x < D ? ~0ull : 0ull;
    __syncthreads();
    const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (kProjThreads / 32);
    for (uint64_t base = (static_cast<uint64_t>(blockIdx.x) * (kProjThreads / 32) + (threadIdx.x >> 5)) * (8 * kProjGroups);
         base < n; base += warps * 8 * kProjGroups)
        project_groups<D, kProjGroups>(img, w, C, keys, n, base, KS, s_B, s_mean, s_joff, Y, s_mm);
    __syncthreads();
    if (threadIdx.x < D) {
        atomicMin(minmax + threadIdx.x, s_mm[0][threadIdx.x]);
        atomicMax(minmax + D + threadIdx.x, s_mm[1][threadIdx.x]);
    }
}

// quantise (proj/src/builder.cpp:55-61) and interleave to the 8*D-bit Morton key
// (proj/include/zinpaint/morton.hpp:14-29): bit L of dim d -> key bit L*D + D-1-d.
// Records of all 8 layouts share one array of N = 8n entries (layout-major); word k of entry
// e lives at keyw[k*N + e]; the payload is (layout << 29) | dictionary row.
template <int D>
__global__ void __launch_bounds__(256) k_quantize(const double* __restrict__ Y,
                                                  const unsigned long long* __restrict__ minmax, uint64_t n,
                                                  uint64_t N, uint32_t layout, uint32_t row_base,
                                                  uint32_t* __restrict__ keyw, uint32_t* __restrict__ val) {
    constexpr int W = (D + 3) / 4;
    __shared__ double s_lo[D], s_hi[D], s_rcp[D];
    // spread table: bit L of q -> bit L*D (W words); dim d's contribution is spread(q) << (D-1-d)
    __shared__ uint32_t s_spread[256][W];
    {
        const uint32_t q = threadIdx.x;  // blockDim.x == 256
        uint32_t sp[W];
#pragma unroll
        for (int k = 0; k < W; ++k) sp[k] = 0;
#pragma unroll
        for (int L = 0; L < 8; ++L) sp[(L * D) >> 5] |= ((q >> L) & 1u) << ((L * D) & 31);
#pragma unroll
        for (int k = 0; k < W; ++k) s_spread[q][k] = sp[k];
    }
    if (threadIdx.x < D) {
        const double l = ordered_to_double_hd(minmax[threadIdx.x]);
        const double h = ordered_to_double_hd(minmax[D + threadIdx.x]);
        s_lo[threadIdx.x] = l;
        s_hi[threadIdx.x] = h;
        s_rcp[threadIdx.x] = h > l ? __ddiv_rn(1.0, __dsub_rn(h, l)) : 0.0;
    }
    __syncthreads();
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        double y[D];
#pragma unroll
        for (int d = 0; d < D; ++d) y[d] = Y[static_cast<size_t>(d) * n + i];
        uint32_t kw[W];
#pragma unroll
        for (int k = 0; k < W; ++k) kw[k] = 0;
#pragma unroll
        for (int d = 0; d < D; ++d) {
            const uint32_t q = quantize_fast(s_lo[d], s_hi[d], s_rcp[d], y[d]);
            const int sh = D - 1 - d;  // = morton_bit(0, d, D)
            uint32_t prev = 0;
#pragma unroll
            for (int k = 0; k < W; ++k) {
                const uint32_t cur = s_spread[q][k];
                kw[k] |= sh ? __funnelshift_l(prev, cur, sh) : cur;
                prev = cur;
            }
        }
        const uint64_t e = static_cast<uint64_t>(layout) * n + i;
#pragma unroll
        for (int k = 0; k < W; ++k) keyw[static_cast<size_t>(k) * N + e] = kw[k];
        val[e] = (layout << 29) | (row_base + static_cast<uint32_t>(i));
    }
}

// row-major coords (zcurve_index::from_descriptors input) -> Morton key words
__global__ void __launch_bounds__(256) k_interleave(const uint8_t* __restrict__ coords,
                                                    const uint32_t* __restrict__ keys_in, uint64_t n, int D,
                                                    uint32_t* __restrict__ keyw, uint32_t* __restrict__ val) {
    const int W = (D + 3) / 4;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        uint32_t kw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int d = 0; d < D; ++d) {
            const uint32_t q = coords[i * D + d];
            for (int L = 0; L < 8; ++L) {
                const int u = morton_bit(L, d, D);
                kw[u >> 5] |= ((q >> L) & 1u) << (u & 31);
            }
        }
        for (int k = 0; k < W; ++k) keyw[static_cast<size_t>(k) * n + i] = kw[k];
        val[i] = keys_in[i];
    }
}

// ============================================================== K5: finalize
// Sorted Morton words -> dim planes (4 dims per u32), keys, and per-256-entry bboxes.
// Entries [off, off+n) of a record array with word stride N; when dict != nullptr the payload
// is a dictionary row (low 29 bits) and the key is gathered from dict (L2-resident).
// One warp per 256-entry bbox block, 8 entries per lane (coalesced, all loads and the dictionary
// gathers in flight together); the bbox is a warp reduction (no block barrier).
constexpr int kFinWarps = 8;
template <int D>
__device__ __forceinline__ void finalize_block(const uint32_t* __restrict__ keyw, const uint32_t* __restrict__ val,
                                               uint64_t N, uint64_t off, uint64_t n,
                                               const uint32_t* __restrict__ dict, uint32_t* __restrict__ planes,
                                               uint32_t* __restrict__ keys, uint32_t* __restrict__ bmin,
                                               uint32_t* __restrict__ bmax, uint64_t nblk) {
    constexpr int W = (D + 3) / 4, P = W, E = 8;
    const int lane = threadIdx.x & 31;
    const uint64_t blk = static_cast<uint64_t>(blockIdx.x) * kFinWarps + (threadIdx.x >> 5);
    if (blk >= nblk) return;
    const uint64_t b0 = blk * 256;
    uint32_t kw[E][W], v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const uint64_t i = b0 + e * 32 + lane;
        const bool ok = i < n;
#pragma unroll
        for (int k = 0; k < W; ++k) kw[e][k] = ok ? __ldg(keyw + static_cast<size_t>(k) * N + off + i) : 0u;
        v[e] = ok ? __ldg(val + off + i) : 0u;
    }
    if (dict) {
#pragma unroll
        for (int e = 0; e < E; ++e)
            if (b0 + e * 32 + lane < n) v[e] = __ldg(dict + (v[e] & ((1u << 29) - 1u)));
    }
    uint32_t mn[P], mx[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
        mn[p] = 0xffffffffu;
        mx[p] = 0u;
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const uint64_t i = b0 + e * 32 + lane;
        if (i < n) {
            uint32_t pw[P];
            morton_deinterleave8<D>(kw[e], pw);
            keys[i] = v[e];
#pragma unroll
            for (int p = 0; p < P; ++p) {
                planes[static_cast<size_t>(p) * n + i] = pw[p];
                mn[p] = __vminu4(mn[p], pw[p]);
                mx[p] = __vmaxu4(mx[p], pw[p]);
            }
        }
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mn[p] = __vminu4(mn[p], __shfl_xor_sync(0xffffffffu, mn[p], o));
            mx[p] = __vmaxu4(mx[p], __shfl_xor_sync(0xffffffffu, mx[p], o));
        }
        // padding bytes (dims >= D) are zero in both coords and queries
        if (lane == p) {
            bmin[static_cast<size_t>(p) * nblk + blk] = mn[p];
            bmax[static_cast<size_t>(p) * nblk + blk] = mx[p];
        }
    }
}

template <int D>
__global__ void __launch_bounds__(kFinWarps * 32) k_finalize(const uint32_t* __restrict__ keyw, const uint32_t* __restrict__ val,
                                                           uint64_t N, uint64_t off, uint64_t n,
                                                           const uint32_t* __restrict__ dict, uint32_t* __restrict__ planes,
                                                           uint32_t* __restrict__ keys, uint32_t* __restrict__ bmin,
                                                           uint32_t* __restrict__ bmax, uint64_t nblk) {
    finalize_block<D>(keyw, val, N, off, n, dict, planes, keys, bmin, bmax, nblk);
}

// the 8 layout indices of a build in one launch (blockIdx.y = layout; layout l's records start at l n)
struct fin_job {
    uint32_t* planes[8];
    uint32_t* keys[8];
    uint32_t* bmin[8];
    uint32_t* bmax[8];
};
template <int D>
__global__ void __launch_bounds__(kFinWarps * 32) k_finalize_layouts(const uint32_t* __restrict__ keyw,
                                                                   const uint32_t* __restrict__ val, uint64_t N, uint64_t n,
                                                                   const uint32_t* __restrict__ dict,
                                                                   const __grid_constant__ fin_job J, uint64_t nblk) {
    const int l = blockIdx.y;
    finalize_block<D>(keyw, val, N, static_cast<uint64_t>(l) * n, n, dict, J.planes[l], J.keys[l], J.bmin[l], J.bmax[l], nblk);
}

// ============================================================== host launchers
template <int D>
static void launch_project_t(zi_ctx* ctx, const uint8_t* img, int w, int C, const uint32_t* keys, uint64_t n,
                             const int32_t* off, int m, const double* mean, const double* comp, double* Y,
                             unsigned long long* minmax) {
    constexpr int NT = (D + 7) / 8;
    const int KS = (m * C + 3) / 4;
    const size_t smem = static_cast<size_t>(KS) * NT * 32 * sizeof(double) + static_cast<size_t>(KS) * 4 * sizeof(double) +
                        static_cast<size_t>(KS) * 4 * sizeof(int);
    smem_attr(ctx->device, k_project<D>, smem);
    const uint64_t warps = (n + 8 * kProjGroups - 1) / (8 * kProjGroups);
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((warps + kProjThreads / 32 - 1) / (kProjThreads / 32),
                                                                   static_cast<uint64_t>(ctx->num_sms) * 8));
    ZI_LAUNCH(ctx, "project", k_project<D>, grid, kProjThreads, smem, img, w, C, keys, n, off, m, mean, comp, Y,
              minmax);
}

template <int D>
static void launch_quantize_t(zi_ctx* ctx, const double* Y, const unsigned long long* mm, uint64_t n, uint64_t N,
                              uint32_t layout, uint32_t row_base, uint32_t* keyw, uint32_t* val) {
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(ctx->num_sms) * 16));
    ZI_LAUNCH(ctx, "quantize_interleave", k_quantize<D>, grid, 256, 0, Y, mm, n, N, layout, row_base, keyw, val);
}

#define ZI_DIMS_SWITCH(D, FN, ...)                                                        \
    switch (D) {                                                                          \
        case 1: FN<1>(__VA_ARGS__); break;   case 2: FN<2>(__VA_ARGS__); break;          \
        case 3: FN<3>(__VA_ARGS__); break;   case 4: FN<4>(__VA_ARGS__); break;          \
        case 5: FN<5>(__VA_ARGS__); break;   case 6: FN<6>(__VA_ARGS__); break;          \
        case 7: FN<7>(__VA_ARGS__); break;   case 8: FN<8>(__VA_ARGS__); break;          \
        case 9: FN<9>(__VA_ARGS__); break;   case 10: FN<10>(__VA_ARGS__); break;        \
        case 11: FN<11>(__VA_ARGS__); break; case 12: FN<12>(__VA_ARGS__); break;        \
        case 13: FN<13>(__VA_ARGS__); break; case 14: FN<14>(__VA_ARGS__); break;        \
        case 15: FN<15>(__VA_ARGS__); break; case 16: FN<16>(__VA_ARGS__); break;        \
        case 17: FN<17>(__VA_ARGS__); break; case 18: FN<18>(__VA_ARGS__); break;        \
        case 19: FN<19>(__VA_ARGS__); break; case 20: FN<20>(__VA_ARGS__); break;        \
        case 21: FN<21>(__VA_ARGS__); break; case 22: FN<22>(__VA_ARGS__); break;        \
        case 23: FN<23>(__VA_ARGS__); break; case 24: FN<24>(__VA_ARGS__); break;        \
        case 25: FN<25>(__VA_ARGS__); break; case 26: FN<26>(__VA_ARGS__); break;        \
        case 27: FN<27>(__VA_ARGS__); break; case 28: FN<28>(__VA_ARGS__); break;        \
        case 29: FN<29>(__VA_ARGS__); break; case 30: FN<30>(__VA_ARGS__); break;        \
        case 31: FN<31>(__VA_ARGS__); break; case 32: FN<32>(__VA_ARGS__); break;        \
        default: throw error(ZI_E_INVALID, "dims must be in [1, 32]");                   \
    }

template <int D>
static void launch_finalize_t(zi_ctx* ctx, const uint32_t* keyw, const uint32_t* val, uint64_t N, uint64_t off,
                              uint64_t n, const uint32_t* dict, zi_index* idx) {
    ZI_LAUNCH(ctx, "finalize_index", k_finalize<D>, static_cast<unsigned>((idx->nblk + kFinWarps - 1) / kFinWarps),
              kFinWarps * 32, 0, keyw, val, N, off, n,
              dict, idx->planes.p, idx->keys.p, idx->bbox_min.p, idx->bbox_max.p, idx->nblk);
}

void project(zi_ctx* ctx, const uint8_t* d_img, int w, int C, const uint32_t* d_keys, uint64_t n,
             const int32_t* d_off, int m, const double* d_mean, const double* d_comp, int D, double* d_Y,
             unsigned long long* d_minmax) {
    if (n == 0) return;
    // lo slots start at the ordered max, hi slots at the ordered min; the projection folds in
    // its per-block min / max
    ZI_CUDA(cudaMemsetAsync(d_minmax, 0xff, D * sizeof(unsigned long long), ctx->stream));
    ZI_CUDA(cudaMemsetAsync(d_minmax + D, 0x00, D * sizeof(unsigned long long), ctx->stream));
    ZI_DIMS_SWITCH(D, launch_project_t, ctx, d_img, w, C, d_keys, n, d_off, m, d_mean, d_comp, d_Y, d_minmax);
}

void quantize_interleave(zi_ctx* ctx, const double* d_Y, const unsigned long long* d_minmax, uint64_t n, uint64_t N,
                         uint32_t layout, int D, uint32_t* d_keyw, uint32_t* d_val, uint32_t row_base) {
    if (n == 0) return;
    ZI_DIMS_SWITCH(D, launch_quantize_t, ctx, d_Y, d_minmax, n, N, layout, row_base, d_keyw, d_val);
}

void interleave_coords(zi_ctx* ctx, const uint8_t* d_coords, const uint32_t* d_keys_in, uint64_t n, int D,
                       uint32_t* d_keyw, uint32_t* d_val) {
    if (n == 0) return;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(ctx->num_sms) * 16));
    ZI_LAUNCH(ctx, "interleave_coords", k_interleave, grid, 256, 0, d_coords, d_keys_in, n, D, d_keyw, d_val);
}

void prepare_index(zi_index* idx, uint64_t n, int D) {
    idx->n = n;
    idx->dims = static_cast<uint32_t>(D);
    idx->planes_n = static_cast<uint32_t>((D + 3) / 4);
    idx->nblk = (n + 255) / 256;
    idx->planes.ensure(static_cast<size_t>(idx->planes_n) * (n ? n : 1));
    idx->keys.ensure(n ? n : 1);
    idx->bbox_min.ensure(static_cast<size_t>(idx->planes_n) * (idx->nblk ? idx->nblk : 1));
    idx->bbox_max.ensure(static_cast<size_t>(idx->planes_n) * (idx->nblk ? idx->nblk : 1));
}

template <int D>
static void launch_finalize_layouts_t(zi_ctx* ctx, const uint32_t* keyw, const uint32_t* val, uint64_t N, uint64_t n,
                                      const uint32_t* dict, const fin_job& J, uint64_t nblk, int nidx) {
    ZI_LAUNCH(ctx, "finalize_index", k_finalize_layouts<D>,
              dim3(static_cast<unsigned>((nblk + kFinWarps - 1) / kFinWarps), static_cast<unsigned>(nidx)), kFinWarps * 32, 0,
              keyw, val, N, n, dict, J, nblk);
}

// finalize of the nidx <= 8 layout indices whose sorted records sit layout-major (n each) in one launch
void finalize_layout_indexes(zi_ctx* ctx, const uint32_t* d_keyw, const uint32_t* d_val, uint64_t N, uint64_t n, int D,
                             const uint32_t* d_dict, zi_index* const* idx, int nidx) {
    fin_job J{};
    for (int l = 0; l < nidx; ++l) {
        prepare_index(idx[l], n, D);
        J.planes[l] = idx[l]->planes.p;
        J.keys[l] = idx[l]->keys.p;
        J.bmin[l] = idx[l]->bbox_min.p;
        J.bmax[l] = idx[l]->bbox_max.p;
    }
    if (n == 0 || nidx <= 0) return;
    ZI_DIMS_SWITCH(D, launch_finalize_layouts_t, ctx, d_keyw, d_val, N, n, d_dict, J, idx[0]->nblk, nidx);
}

void finalize_index(zi_ctx* ctx, const uint32_t* d_keyw, const uint32_t* d_val, uint64_t N, uint64_t off, uint64_t n,
                    int D, const uint32_t* d_dict, zi_index* idx) {
    prepare_index(idx, n, D);
    if (n == 0) return;
    ZI_DIMS_SWITCH(D, launch_finalize_t, ctx, d_keyw, d_val, N, off, n, d_dict, idx);
}

double ordered_to_double(unsigned long long u) { return ordered_to_double_hd(u); }

}  // namespace zi
