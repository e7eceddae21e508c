// k_proj_tc.cu -- K3 projection + quantisation on the int8 tensor cores, with an exact fp64
// fix-up: the same bytes as the canonical fp64 path (k_project + k_quantize, restating
// proj/src/builder.cpp:159-187 and pca.cpp:7-11), at tensor-core speed.
//
// Filter.  Every component c (|c| <= 1) is held as t = rint(c * 2^38), split into five balanced
// base-256 digits (int8).  For a u8 patch x the five column sums S_k = sum_j x_j digit_k(t_j) are
// EXACT tcgen05.mma.kind::i8 results (u8 x s8 -> s32, |S_k| <= 255*128*384 < 2^31).  Then
//     y' = sum_k S_k 2^(8k-38) - M,   M = sum_j mean_j c_j,
// and |y' - y| <= E = 255 * mc * (2^-39 + 2^-44) for the canonical fp64 value y (the fixed-point
// truncation bound plus a generous allowance for the fp64 roundings of y, M and y').
//
// Two passes over all patches (A tiles gathered from the L2-resident image straight into
// 128B-swizzled shared memory, no patch matrix in HBM; the digit matrix B stays in shared memory;
// one CTA per SM, two TMEM accumulators so the epilogue of tile i overlaps the MMAs of tile i+1):
//   pass 0  exact min / max of y' per (layout, dim)  ->  amin, amax
//   pass 1  the true lo, hi lie in [amin - E, amin + E], [amax - E, amax + E]; with z' =
//           255 (y' - amin) / (amax - amin) the reference's quantised value is floor(z' + 1/2)
//           unless z' + 1/2 is within Bz = 1.01 * 255 * 4E / (amax - amin) of an integer.  Such
//           (patch, layout) pairs, and the rows within 2E of amin / amax (the only rows that can
//           hold the true lo / hi), go to a list; everything else writes its Morton record now.
// Fix-up (k_pt_exact): the listed pairs are projected in the canonical fp64 order (the same
// sequential fma chain k_project runs on the FP64 MMA), giving the exact lo / hi (atomics over the
// candidates) and then their exact quantised Morton records.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace zi {

#ifndef ZI_PT_G8
#define ZI_PT_G8 0
#endif
#ifndef ZI_PT_SPLIT_LD
#define ZI_PT_SPLIT_LD 1
#endif
#ifndef ZI_PT_ONE_READ
#define ZI_PT_ONE_READ 0
#endif
constexpr int kPtRows = 128;
// epilogue warps 4 .. 4 + 4S - 1: TMEM lane quarter (w & 3), layouts li = (w >> 2) mod S.  S = 4 sets
// for D <= 10 (a group's layouts spread one per set); S = 3 above, where the larger per-layout
// register state would spill at the 80 registers a 21-warp CTA leaves per thread
// the min / max pass keeps running per-thread extremes when every epilogue warp set has exactly one
// layout of the group (the host's plan for D = 7..10: two groups of four layouts, four sets)
template <int D>
__host__ __device__ constexpr bool pt_running() {
    return D >= 7 && D <= 10;
}

template <int D, int MODE>
struct pt_shape {
    // gather warps 0 .. G-1: one thread per patch row (G = 4).  ZI_PT_G8 = 1 (A/B): two threads per
    // row for the min / max pass at D <= 8 -- the better shape while that pass ran once per layout
    // group and was bound by its gather (1.80 -> 1.55 ms at cfg4); with both groups fed from one
    // gathered tile the epilogue is the limit and the four extra warps cost registers (1.13 vs 1.02 ms)
    static constexpr int kGatherWarps = (D <= 8 && MODE == 0 && ZI_PT_G8) ? 8 : 4;
    static constexpr int kEpiSets = D <= 10 ? 4 : 3;
    static constexpr int kEpiWarps = 4 * kEpiSets;
    static constexpr int kMmaWarp = kGatherWarps + kEpiWarps;
    static constexpr int kThreads = (kMmaWarp + 1) * 32;
};
constexpr int kPtMaxFpad = 384;
constexpr int kPtMaxN = 256;
// t = rint(c * 2^38) in five balanced base-256 digits.  (Four digits put all 8 layouts of a D = 8
// build in one 256-column group, but their 256x larger E flags ~1.5 % of the cfg4 pairs for the
// fp64 fix-up -- low-variance dims have ranges of only a few units -- which costs more than the
// second group's gather saves.)
constexpr int kPtDigits = 5;
constexpr double kPtScale = 274877906944.0;      // 2^(8 * kPtDigits - 2)
constexpr double kPtUnit = 1.0 / kPtScale;       // 2^-38

struct pt_params {
    const uint8_t* img;
    int w, C, KC, F, Fpad;
    const uint32_t* keys;
    uint64_t n;
    uint32_t row_base;
    int payload_key;   // records carry the patch key as payload (the fused final sort pass), not (l << 29) | row
    const uint8_t* B;  // this group's digit matrix, pre-swizzled (Npad x Fpad)
    int Npad, l0, nl;
    int nhalf;  // layout groups in this launch (1, or 2: both groups' accumulators from one gathered A tile)
    const double* M;          // [8][D]
    unsigned long long* amm;  // approx min / max of y', ordered u64 [8][2][D]
    double E;
    uint32_t* keyw;
    uint32_t* val;
    uint64_t Nrec;
    uint32_t* list;  // (row << 3) | layout
    uint32_t* list_count;
    uint64_t ntiles;
    const int2* wtab;  // Fpad/4 gather words (pt_gather)
};

// byte offset of (row r, K-byte f) in a K-major, 128B-swizzled operand of `rows` rows
__host__ __device__ inline uint32_t sw128_off(int r, int f, int rows) {
    return static_cast<uint32_t>((f >> 7) * (rows * 128) + (r >> 3) * 1024 + (r & 7) * 128 +
                                 ((((f & 127) >> 4) ^ (r & 7)) << 4) + (f & 15));
}

__device__ __forceinline__ uint32_t pt_idesc(int N) {
    return (2u << 4)        // D format S32
           | (0u << 7)      // A unsigned 8-bit (u8 patches)
           | (1u << 10)     // B signed 8-bit (digits)
           | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(kPtRows >> 4) << 24);
}

__device__ __forceinline__ void pt_mma(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
        "l"(da), "l"(db), "r"(idesc), "r"(acc)
        : "memory");
}

// 4 image bytes starting at byte address a (two aligned word loads; the device image carries 16
// bytes of padding, so the second load never leaves the allocation)
__device__ __forceinline__ uint32_t pt_ld4(const uint8_t* __restrict__ img, uint32_t a) {
    const uint32_t* p = reinterpret_cast<const uint32_t*>(img + (a & ~3u));
    return __funnelshift_r(__ldg(p), __ldg(p + 1), (a & 3u) * 8u);
}

// A tile (128 patches x Fpad bytes, feature f = (rr*K + cc)*C + ch at byte f of the row) into the
// swizzled A buffer.  One thread per patch row (warps 0-3).  Word ow of every row reads the same
// patch-relative offsets, so they come from a warp-uniform table (pt_word_table): x = offset of
// the word's first byte (-1: zero word); y = -1 when the 4 bytes lie in one patch row, else
// (bytes taken from the first row) << 24 | offset of the next patch row (0xffffff: none).
__device__ __forceinline__ void pt_gather(const pt_params& P, const int2* s_wtab, uint64_t tile, uint32_t sA_addr, int r,
                                          int c0, int c1) {
    const uint64_t i = tile * kPtRows + r;
    uint32_t base = 0;
    const bool valid = i < P.n;
    if (valid) {
        const uint32_t key = __ldg(P.keys + i);
        base = ((key >> 16) * static_cast<uint32_t>(P.w) + (key & 0xffffu)) * static_cast<uint32_t>(P.C);
    }
#pragma unroll 2
    for (int c = c0; c < c1; ++c) {
        uint32_t wv[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int2 e = s_wtab[4 * c + t];
            uint32_t word = 0;
            if (e.x >= 0) {
                word = pt_ld4(P.img, base + static_cast<uint32_t>(e.x));
                if (e.y >= 0) {
                    const uint32_t sh = 8u * (static_cast<uint32_t>(e.y) >> 24), o1 = static_cast<uint32_t>(e.y) & 0xffffffu;
                    word &= (1u << sh) - 1u;
                    if (o1 != 0xffffffu) word |= pt_ld4(P.img, base + o1) << sh;
                }
            }
            // feature F (the first padding byte) is 1 for every real patch: the fused Gram reads
            // its column as the first moments; the projection's digits there are zero
            if (4 * c + t == (static_cast<int>(P.F) >> 2)) word |= 1u << (8 * (P.F & 3));
            wv[t] = valid ? word : 0u;
        }
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(sA_addr + sw128_off(r, c << 4, kPtRows)), "r"(wv[0]),
                     "r"(wv[1]), "r"(wv[2]), "r"(wv[3])
                     : "memory");
    }
}

// Static gather for a compile-time patch shape (K, C): half GH of a patch row (two threads per
// row).  Every patch row (segment) of K*C bytes is read as aligned words, realigned with one funnel
// shift per word and placed at its (static) byte position of the feature row; a 16-byte chunk is
// stored as soon as its last segment is in.  Half 0 stores the chunks that end before segment K/2,
// half 1 the rest (re-reading the segments the straddling chunk needs).
template <int K, int C, int GH>
__device__ __forceinline__ void pt_gather_static(const uint8_t* __restrict__ img, uint32_t base, uint32_t wC, bool valid,
                                                 uint32_t sA_addr, int r) {
    constexpr int KC = K * C, F = K * KC, FP = (F + 127) / 128 * 128, NCH = FP / 16;
    constexpr int KH = K / 2;
    constexpr int CSPLIT = (KH * KC) / 16;              // first chunk of half 1 (may straddle)
    constexpr int C0 = GH ? CSPLIT : 0, C1 = GH ? NCH : CSPLIT;
    constexpr int S0 = GH ? (16 * CSPLIT) / KC : 0, S1 = GH ? K : KH;
    constexpr int RB = (KC + 3) / 4;                     // realigned words of a segment
    constexpr int SW = (KC + 6) / 4;                     // aligned words covering it
    constexpr int NO = 4 * (C1 - C0);                    // output words of this half
    uint32_t out[NO];
#pragma unroll
    for (int i = 0; i < NO; ++i) out[i] = 0u;
    if constexpr (F / 4 - 4 * C0 >= 0 && F / 4 - 4 * C0 < NO) {  // feature F = 1: the ones column
        if (valid) out[F / 4 - 4 * C0] |= 1u << (8 * (F % 4));
    }
#pragma unroll
    for (int rr = S0; rr < S1; ++rr) {
        const uint32_t a = base + static_cast<uint32_t>(rr) * wC;
        const uint32_t* wp = reinterpret_cast<const uint32_t*>(img + (a & ~3u));
        const uint32_t sh = (a & 3u) * 8u;
        uint32_t wv[SW];
#pragma unroll
        for (int i = 0; i < SW; ++i) wv[i] = valid ? __ldg(wp + i) : 0u;
#pragma unroll
        for (int i = 0; i < RB; ++i) {
            uint32_t x = __funnelshift_r(wv[i], wv[i + 1], sh);
            if (4 * i + 4 > KC) x &= (1u << (8 * (KC - 4 * i))) - 1u;  // bytes past the segment
            const int o = rr * KC + 4 * i;                             // output byte of x's byte 0
            const int ow = o / 4 - 4 * C0, t = o % 4;
            if (ow >= 0 && ow < NO) out[ow] |= t ? (x << (8 * t)) : x;
            if (t && ow + 1 >= 0 && ow + 1 < NO) out[ow + 1] |= x >> (32 - 8 * t);
        }
        // chunks whose last feature byte lies in this segment (or, past F, after the last one)
#pragma unroll
        for (int c = C0; c < C1; ++c) {
            const int last = (16 * c + 15 < F ? 16 * c + 15 : F - 1) / KC;
            const int when = 16 * c >= F ? S1 - 1 : (last < S1 ? last : S1 - 1);
            if (when == rr) {
                const int q = 4 * (c - C0);
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(sA_addr + sw128_off(r, c << 4, kPtRows)),
                             "r"(out[q]), "r"(out[q + 1]), "r"(out[q + 2]), "r"(out[q + 3])
                             : "memory");
            }
        }
    }
}

template <int D, int MODE, int KT>
__global__ void __launch_bounds__(pt_shape<D, MODE>::kThreads, 1) k_proj_tc(const __grid_constant__ pt_params P) {
    constexpr int kPtEpiSets = pt_shape<D, MODE>::kEpiSets, kPtEpiWarps = pt_shape<D, MODE>::kEpiWarps;
    constexpr int kPtGatherWarps = pt_shape<D, MODE>::kGatherWarps;
    constexpr int kPtMmaWarp = pt_shape<D, MODE>::kMmaWarp, kPtThreads = pt_shape<D, MODE>::kThreads;
    constexpr int W = (D + 3) / 4;
    extern __shared__ uint8_t pt_raw[];
    uint8_t* sbase = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(pt_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    const uint32_t abytes = static_cast<uint32_t>(kPtRows * P.Fpad);
    uint8_t* sA = sbase;
    uint8_t* sB = sbase + 2 * abytes;
    __shared__ __align__(8) uint64_t s_afull[2], s_aempty[2], s_accfull[2], s_accempty[2];
    __shared__ uint32_t s_tmem;
    __shared__ double s_M[8][D];
    // quantise constants per (layout, dim): {za, zb} {bz, tlo} {thi, -} as two-word vectors (16 B loads)
    __shared__ __align__(16) double2 s_qc[8][D][3];
    // fp32 pre-filter of the quantise pass per (layout, dim): {za * 2^20, zb, bz + eps, 1 - bz - eps}
    __shared__ __align__(16) float4 s_qf[8][D];
    // lo / hi candidate thresholds on T >> 20 (floors of tlo, thi: a superset of the exact test)
    __shared__ __align__(8) int2 s_qt[8][D];
    // Morton spread table, four copies 8 banks apart (lane group g = lane >> 3 reads copy g)
    constexpr int kSpStride = 256 * W + 8;
    __shared__ uint32_t s_spread[4 * kSpStride];
    __shared__ int2 s_wtab[kPtMaxFpad / 4];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nl = P.nl;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc_smem(&s_tmem)), "r"(512u)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int s = 0; s < 2; ++s) {
            tc_mbar_init(tc_smem(&s_afull[s]), kPtGatherWarps);
            tc_mbar_init(tc_smem(&s_aempty[s]), 1);
            tc_mbar_init(tc_smem(&s_accfull[s]), 1);
            tc_mbar_init(tc_smem(&s_accempty[s]), kPtEpiWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    {  // the digit matrix (already in the swizzled layout) and the per-(layout, dim) constants
        const uint4* src = reinterpret_cast<const uint4*>(P.B);
        uint4* dst = reinterpret_cast<uint4*>(sB);
        const int nv = P.nhalf * P.Npad * P.Fpad / 16;
        for (int i = tid; i < nv; i += kPtThreads) dst[i] = __ldg(src + i);
        for (int i = tid; i < P.Fpad / 4; i += kPtThreads) s_wtab[i] = P.wtab[i];
        for (int i = tid; i < P.nhalf * nl * D; i += kPtThreads) {
            const int li = i / D, d = i - li * D, l = P.l0 + li;
            s_M[li][d] = P.M[l * D + d];
            if (MODE == 1) {
                const double lo = ordered_to_double_hd(P.amm[static_cast<size_t>(l) * 2 * D + d]);
                const double hi = ordered_to_double_hd(P.amm[static_cast<size_t>(l) * 2 * D + D + d]);
                const double R = hi - lo;
                const bool degen = !(R > 4.0 * P.E);
                const double M = s_M[li][d];
                // z' = T * za + zb = 255 (T 2^-38 - M - lo) / R + 1/2 (its rounding, ~1e-11 even
                // with cancellation, is inside Bz's 1e-9 slack)
                const double za = degen ? 0.0 : 255.0 * kPtUnit / R;
                const double zb = degen ? 0.0 : 0.5 - 255.0 * (M + lo) / R;
                const double bz = degen ? 1.0 : 1.01 * 255.0 * 4.0 * P.E / R + 1e-9;
                // lo / hi candidates: y' <= lo + 2E or y' >= hi - 2E, as T thresholds widened by
                // a margin (a superset is harmless: candidates only cost a fix-up)
                const double tl = (lo + 2.0 * P.E + M) * kPtScale, th = (hi - 2.0 * P.E + M) * kPtScale;
                const long long tlo = degen ? LLONG_MAX : static_cast<long long>(ceil(tl + fabs(tl) * 0x1p-40)) + 16;
                const long long thi = degen ? LLONG_MAX : static_cast<long long>(floor(th - fabs(th) * 0x1p-40)) - 16;
                s_qc[li][d][0] = make_double2(za, zb);
                s_qc[li][d][1] = make_double2(bz, __longlong_as_double(tlo));
                s_qc[li][d][2] = make_double2(__longlong_as_double(thi), 0.0);
                s_qt[li][d] = degen ? make_int2(INT_MAX, INT_MAX)
                                    : make_int2(static_cast<int>(max(min(tlo >> 20, static_cast<long long>(INT_MAX)), static_cast<long long>(INT_MIN))),
                                                static_cast<int>(max(min(thi >> 20, static_cast<long long>(INT_MAX)), static_cast<long long>(INT_MIN))));
                // z32 = fmaf(float(T >> 20), za * 2^20, zb) is within eps of z': the dropped low 20
                // bits of T (2^20 za), and five fp32 roundings of terms below |T za| + |zb| + 256,
                // where |T za| = 255 |y' + M| / R is bounded through the approximate range (a row
                // outside it is a lo / hi candidate, which the exact path also sees); doubled
                const double tza = degen ? 0.0 : 255.0 * fmax(fabs(lo + M), fabs(hi + M)) / R;
                const double eps = 2.0 * (0x1p20 * za + 0x1p-22 * (2.0 * tza + fabs(zb) + 256.0)) + 1e-9;
                s_qf[li][d] = degen ? make_float4(0.f, 0.f, 2.f, -1.f)  // never decided in fp32
                                    : make_float4(static_cast<float>(za * 0x1p20), static_cast<float>(zb),
                                                  static_cast<float>(bz + eps), static_cast<float>(1.0 - bz - eps));
            }
        }
        if (MODE == 1 && tid < 256) {
            uint32_t sp[W];
#pragma unroll
            for (int k = 0; k < W; ++k) sp[k] = 0;
#pragma unroll
            for (int L = 0; L < 8; ++L) sp[(L * D) >> 5] |= ((static_cast<uint32_t>(tid) >> L) & 1u) << ((L * D) & 31);
#pragma unroll
            for (int k = 0; k < W; ++k)
#pragma unroll
                for (int c = 0; c < 4; ++c) s_spread[c * kSpStride + tid * W + k] = sp[k];
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;
    const uint64_t nloc = blockIdx.x < P.ntiles ? (P.ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

    // MODE 0: lane-distributed (layout, dim) slots of min / max T
    long long tmn0 = LLONG_MAX, tmx0 = LLONG_MIN;
    if (warp == kPtMmaWarp) {
        if (lane == 0) {  // MMA issuer
            const uint32_t idesc = pt_idesc(P.Npad);
            const int KB = P.Fpad >> 7;
            const int NH = P.nhalf;
            const uint32_t bbytes = static_cast<uint32_t>(P.Npad * P.Fpad);
            for (uint64_t i = 0; i < nloc; ++i) {
                const int abuf = static_cast<int>(i & 1);
                tc_mbar_wait(tc_smem(&s_afull[abuf]), static_cast<uint32_t>(i >> 1) & 1);
                const uint32_t a0 = tc_smem(sA + abuf * abytes);
                for (int h = 0; h < NH; ++h) {  // unit u = NH i + h: accumulator buffer u & 1
                    const uint64_t u = i * NH + h;
                    const int buf = static_cast<int>(u & 1);
                    const uint32_t use = static_cast<uint32_t>(u >> 1);
                    if (u >= 2) tc_mbar_wait(tc_smem(&s_accempty[buf]), (use - 1) & 1);
                    tc_fence_after();
                    const uint32_t acc = tmem + static_cast<uint32_t>(buf * 256);
                    const uint32_t b0 = tc_smem(sB) + static_cast<uint32_t>(h) * bbytes;
                    for (int kb = 0; kb < KB; ++kb) {
                        const uint64_t da = tc_desc_k128(a0 + kb * kPtRows * 128);
                        const uint64_t db = tc_desc_k128(b0 + kb * P.Npad * 128);
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks) pt_mma(acc, da + 2 * ks, db + 2 * ks, idesc, (kb | ks) != 0 ? 1u : 0u);
                    }
                    if (h == NH - 1) tc_commit(tc_smem(&s_aempty[abuf]));
                    tc_commit(tc_smem(&s_accfull[buf]));
                }
            }
        }
    } else if (warp < kPtGatherWarps) {  // gather: two threads per patch row (the halves of its features)
        const int nchunk = P.Fpad >> 4, hc = (nchunk + 1) >> 1, gh = tid >> 7;
        constexpr bool kTwo = kPtGatherWarps == 8;  // else one thread does both halves
        for (uint64_t i = 0; i < nloc; ++i) {
            const int buf = static_cast<int>(i & 1);
            const uint32_t use = static_cast<uint32_t>(i >> 1);
            if (i >= 2) tc_mbar_wait(tc_smem(&s_aempty[buf]), (use - 1) & 1);
            const uint64_t tile = blockIdx.x + i * gridDim.x;
            if (KT == 0) {
                if (kTwo) pt_gather(P, s_wtab, tile, tc_smem(sA + buf * abytes), tid & 127, gh ? hc : 0, gh ? nchunk : hc);
                else pt_gather(P, s_wtab, tile, tc_smem(sA + buf * abytes), tid, 0, nchunk);
            } else {
                const int r = tid & 127;
                const uint64_t pr = tile * kPtRows + r;
                const bool valid = pr < P.n;
                uint32_t base = 0;
                if (valid) {
                    const uint32_t key = __ldg(P.keys + pr);
                    base = ((key >> 16) * static_cast<uint32_t>(P.w) + (key & 0xffffu)) * static_cast<uint32_t>(P.C);
                }
                const uint32_t wC = static_cast<uint32_t>(P.w * P.C), sa = tc_smem(sA + buf * abytes);
                if (KT == 1) {
                    if (!kTwo || !gh) pt_gather_static<9, 1, 0>(P.img, base, wC, valid, sa, r);
                    if (!kTwo || gh) pt_gather_static<9, 1, 1>(P.img, base, wC, valid, sa, r);
                } else {
                    if (!kTwo || !gh) pt_gather_static<11, 3, 0>(P.img, base, wC, valid, sa, r);
                    if (!kTwo || gh) pt_gather_static<11, 3, 1>(P.img, base, wC, valid, sa, r);
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) tc_mbar_arrive(tc_smem(&s_afull[buf]));
        }
    } else if (MODE == 0 && pt_running<D>()) {
        // min / max pass, one layout per warp set and half.  The exact int64 extremes of T live
        // in lane slots (lane h D + d of the warp holds those of its half-h layout's dim d); every
        // thread keeps only their floors by 2^20 as 32-bit filters.  A row can replace an extreme
        // only if floor(T / 2^20) -- nested 32-bit shifts of the digits -- reaches the filter; then
        // the warp assembles the 64-bit T of that dim, reduces it, the slot lane and every lane's
        // filter take the result (floor is monotone, so the filters stay the extremes' floors and
        // equal across the warp).  TMEM is read in two halves of the dims (registers).
        const int ew = warp - kPtGatherWarps, q4 = ew & 3, lpar = ew >> 2;
        constexpr int DH = ZI_PT_ONE_READ ? D : (D + 1) / 2, NHD = ZI_PT_ONE_READ ? 1 : 2;
        static_assert(2 * D <= 32, "lane slots: two halves of D dims");
        int fmn[2][D], fmx[2][D];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int d = 0; d < D; ++d) {
                fmn[h][d] = INT_MAX;  // everything passes until the first reduction
                fmx[h][d] = INT_MIN;
            }
        // |T| < 2^51: start values outside every T
        long long emn = 1ll << 51, emx = -(1ll << 51);
        const int NH = P.nhalf;
        for (uint64_t j = 0; j < nloc; ++j) {
            const uint64_t tile = blockIdx.x + j * gridDim.x;
            const bool valid = tile * kPtRows + q4 * 32 + lane < P.n;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (h < NH) {
                    const uint64_t u = j * NH + h;
                    const int buf = static_cast<int>(u & 1);
                    tc_mbar_wait(tc_smem(&s_accfull[buf]), static_cast<uint32_t>(u >> 1) & 1);
                    tc_fence_after();
                    const uint32_t ta = tmem + static_cast<uint32_t>(buf * 256) + (static_cast<uint32_t>(q4 * 32) << 16) +
                                        static_cast<uint32_t>(lpar * kPtDigits * D);
#pragma unroll
                    for (int hd = 0; hd < NHD; ++hd) {
                        constexpr int NV = kPtDigits * DH;
                        const int d0 = hd * DH, nd = hd ? D - DH : DH;
                        uint32_t v[NV];
                        if (lpar < nl) {
#pragma unroll
                            for (int c = 0; c + 4 <= NV; c += 4) {
                                uint32_t t4[4];
                                tc_ld_x4(ta + static_cast<uint32_t>(kPtDigits * d0 + c), t4);
#pragma unroll
                                for (int q = 0; q < 4; ++q) v[c + q] = t4[q];
                            }
#pragma unroll
                            for (int c = NV & ~3; c < NV; ++c) tc_ld_x1(ta + static_cast<uint32_t>(kPtDigits * d0 + c), v[c]);
                            tc_ld_wait();
                        }
                        if (hd == NHD - 1) {  // this buffer is read: release it to the MMA warp
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) tc_mbar_arrive(tc_smem(&s_accempty[buf]));
                        }
                        if (lpar < nl) {
                            uint32_t cm = 0;  // dims of this half whose filter the row reaches
#pragma unroll
                            for (int dd = 0; dd < DH; ++dd) {
                                if (dd < nd) {
                                    const uint32_t* vd = v + kPtDigits * dd;
                                    const int s0 = static_cast<int>(vd[0]) >> 8;
                                    const int s1 = (static_cast<int>(vd[1]) + s0) >> 8;
                                    const int s2 = (static_cast<int>(vd[2]) + s1) >> 4;
                                    const int t20 = static_cast<int>(vd[4] * 4096u + vd[3] * 16u + static_cast<uint32_t>(s2));
                                    if (t20 <= fmn[h][d0 + dd] || t20 >= fmx[h][d0 + dd]) cm |= 1u << dd;
                                }
                            }
                            const uint32_t any = __reduce_or_sync(0xffffffffu, valid ? cm : 0u);
                            if (any) {
#pragma unroll
                                for (int dd = 0; dd < DH; ++dd) {
                                    if (dd < nd && ((any >> dd) & 1u)) {
                                        const uint32_t* vd = v + kPtDigits * dd;
                                        const long long T = (static_cast<long long>(static_cast<int>(vd[4])) << 32) +
                                                            (static_cast<long long>(static_cast<int>(vd[3])) << 24) +
                                                            (static_cast<long long>(static_cast<int>(vd[2])) << 16) +
                                                            (static_cast<long long>(static_cast<int>(vd[1])) << 8) +
                                                            static_cast<long long>(static_cast<int>(vd[0]));
                                        const int th = static_cast<int>(T >> 32);
                                        const uint32_t tl = static_cast<uint32_t>(T);
                                        const int mh = __reduce_min_sync(0xffffffffu, valid ? th : 0x7fffffff);
                                        const uint32_t ml = __reduce_min_sync(0xffffffffu, (valid && th == mh) ? tl : 0xffffffffu);
                                        const int xh = __reduce_max_sync(0xffffffffu, valid ? th : static_cast<int>(0x80000000));
                                        const uint32_t xl = __reduce_max_sync(0xffffffffu, (valid && th == xh) ? tl : 0u);
                                        const long long wmn = (static_cast<long long>(mh) << 32) | ml;
                                        const long long wmx = (static_cast<long long>(xh) << 32) | xl;
                                        if (lane == h * D + d0 + dd) {
                                            emn = wmn < emn ? wmn : emn;
                                            emx = wmx > emx ? wmx : emx;
                                        }
                                        const int fn = static_cast<int>(wmn >> 20), fx = static_cast<int>(wmx >> 20);
                                        fmn[h][d0 + dd] = fn < fmn[h][d0 + dd] ? fn : fmn[h][d0 + dd];
                                        fmx[h][d0 + dd] = fx > fmx[h][d0 + dd] ? fx : fmx[h][d0 + dd];
                                    }
                                }
                            }
                        }
                    }
                }
            }
        }
        if (lpar < nl && lane < NH * D && emn <= emx) {  // the slot saw a valid row: one ordered atomic each
            const int h = lane / D, d = lane - h * D;
            const int li = h * nl + lpar, l = P.l0 + li;
            const double M = s_M[li][d];
            atomicMin(P.amm + static_cast<size_t>(l) * 2 * D + d, double_to_ordered(__dsub_rn(static_cast<double>(emn) * kPtUnit, M)));
            atomicMax(P.amm + static_cast<size_t>(l) * 2 * D + D + d,
                      double_to_ordered(__dsub_rn(static_cast<double>(emx) * kPtUnit, M)));
        }
    } else {  // epilogue: TMEM lane quarter ew & 3, layouts of parity ew >> 2, one patch row per thread
        const int ew = warp - kPtGatherWarps, q4 = ew & 3, lpar = ew >> 2;  // lpar in [0, kPtEpiSets)
        const uint64_t NH = static_cast<uint64_t>(P.nhalf);
        for (uint64_t u = 0; u < nloc * NH; ++u) {  // unit u = NH j + h: tile j, layout half h
            const uint64_t j = NH == 2 ? u >> 1 : u;
            const int h = NH == 2 ? static_cast<int>(u & 1) : 0, cb = h * nl;  // cb: first constant slot of the half
            const int buf = static_cast<int>(u & 1);
            tc_mbar_wait(tc_smem(&s_accfull[buf]), static_cast<uint32_t>(u >> 1) & 1);
            tc_fence_after();
            const uint64_t tile = blockIdx.x + j * gridDim.x;
            const uint64_t row = tile * kPtRows + q4 * 32 + lane;
            const bool valid = row < P.n;
            const uint32_t tbase = tmem + static_cast<uint32_t>(buf * 256) + (static_cast<uint32_t>(q4 * 32) << 16);
            if (lpar >= nl) {  // no layout for this warp in this group: release the accumulator at once
                tc_fence_before();
                __syncwarp();
                if (lane == 0) tc_mbar_arrive(tc_smem(&s_accempty[buf]));
            }
            for (int li = lpar; li < nl; li += kPtEpiSets) {
                constexpr int NC = kPtDigits * D;
                uint32_t v[NC];
                const uint32_t ta = tbase + static_cast<uint32_t>(li * NC);
                // MODE 1 reads the columns in two parts: the second part's loads are in flight while
                // the dims of the first are quantised (DB = the first dim that needs the second part)
                constexpr int C1 = (MODE == 1 && ZI_PT_SPLIT_LD && D >= 4) ? ((NC / 2) & ~3) : NC;
                constexpr int DB = C1 / kPtDigits;
#pragma unroll
                for (int c = 0; c + 4 <= C1; c += 4) {
                    uint32_t t4[4];
                    tc_ld_x4(ta + c, t4);
#pragma unroll
                    for (int u = 0; u < 4; ++u) v[c + u] = t4[u];
                }
                if constexpr (C1 == NC) {
#pragma unroll
                    for (int c = NC & ~3; c < NC; ++c) tc_ld_x1(ta + c, v[c]);
                }
                tc_ld_wait();
                if constexpr (C1 < NC) {
#pragma unroll
                    for (int c = C1; c + 4 <= NC; c += 4) {
                        uint32_t t4[4];
                        tc_ld_x4(ta + c, t4);
#pragma unroll
                        for (int u = 0; u < 4; ++u) v[c + u] = t4[u];
                    }
#pragma unroll
                    for (int c = C1 + ((NC - C1) & ~3); c < NC; ++c) tc_ld_x1(ta + c, v[c]);
                }
                if (C1 == NC && li + kPtEpiSets >= nl) {  // TMEM of this buffer fully read: release it to the MMA warp early
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) tc_mbar_arrive(tc_smem(&s_accempty[buf]));
                }
                uint32_t kw[W];
#pragma unroll
                for (int k = 0; k < W; ++k) kw[k] = 0;
                bool flag = false, cand = false;
#pragma unroll
                for (int d = 0; d < D; ++d) {
                    if constexpr (C1 < NC) {
                        if (d == DB) {  // the second part has landed; its registers are read only after this point
                            tc_ld_wait();
#pragma unroll
                            for (int c = C1; c < NC; ++c) asm volatile("" : "+r"(v[c]));
                            if (li + kPtEpiSets >= nl) {  // TMEM of this buffer fully read: release it to the MMA warp
                                tc_fence_before();
                                __syncwarp();
                                if (lane == 0) tc_mbar_arrive(tc_smem(&s_accempty[buf]));
                            }
                        }
                    }
                    // T = sum_k S_k 2^(8k) in int64 (exact, |T| < 2^51); the fp64 conversions run at a
                    // fraction of the integer rate, so the min / max pass stays integer and the
                    // quantise pass converts once: y' = fl(T * 2^-38 - M) (T exact in a double)
                    const uint32_t* vd = v + kPtDigits * d;
                    static_assert(kPtDigits == 5, "T assembly below is written for five digits");
                    if (MODE == 0) {
                        const long long T = (static_cast<long long>(static_cast<int>(vd[4])) << 32) +
                                            (static_cast<long long>(static_cast<int>(vd[3])) << 24) +
                                            (static_cast<long long>(static_cast<int>(vd[2])) << 16) +
                                            (static_cast<long long>(static_cast<int>(vd[1])) << 8) +
                                            static_cast<long long>(static_cast<int>(vd[0]));
                        // y' is monotone in T: min / max on T
                        const int th = static_cast<int>(T >> 32);
                        const uint32_t tl = static_cast<uint32_t>(T);
                        const int mh = __reduce_min_sync(0xffffffffu, valid ? th : 0x7fffffff);
                        const uint32_t ml = __reduce_min_sync(0xffffffffu, (valid && th == mh) ? tl : 0xffffffffu);
                        const int xh = __reduce_max_sync(0xffffffffu, valid ? th : static_cast<int>(0x80000000));
                        const uint32_t xl = __reduce_max_sync(0xffffffffu, (valid && th == xh) ? tl : 0u);
                        const long long wmn = (static_cast<long long>(mh) << 32) | ml;
                        const long long wmx = (static_cast<long long>(xh) << 32) | xl;
                        const int slot = (li / kPtEpiSets) * D + d;  // this warp's (layout, dim) slot (< 32)
                        if (slot == lane) {
                            tmn0 = wmn < tmn0 ? wmn : tmn0;
                            tmx0 = wmx > tmx0 ? wmx : tmx0;
                        }
                    } else {
                        // floor(T / 2^20) in 32-bit arithmetic (|T| < 2^51; nested floors of the low
                        // digits, wrap-around sums): the fast path never assembles the 64-bit T
                        const int s0 = static_cast<int>(vd[0]) >> 8;
                        const int s1 = (static_cast<int>(vd[1]) + s0) >> 8;
                        const int s2 = (static_cast<int>(vd[2]) + s1) >> 4;
                        const int t20 = static_cast<int>(vd[4] * 4096u + vd[3] * 16u + static_cast<uint32_t>(s2));
                        // degenerate ranges (amax - amin <= 4E) carry bz = 1 and thresholds INT_MAX:
                        // every row is flagged and a lo / hi candidate, with no branch here
                        const int2 qt = s_qt[cb + li][d];
                        cand = cand || (t20 <= qt.x) || (t20 >= qt.y);
                        // fp32 first: when z32's fraction keeps eps + bz off both integers, floor(z32)
                        // is floor(z') and the fp64 test below could not flag (|z32 - z'| <= eps)
                        const float4 qf32 = s_qf[cb + li][d];
                        const float z32 = __fmaf_rn(static_cast<float>(t20), qf32.x, qf32.y);
                        const float fl32 = floorf(z32);
                        const float fr32 = z32 - fl32;
                        int qi;
                        if (fr32 >= qf32.z && fr32 <= qf32.w) {
                            qi = static_cast<int>(fl32);
                        } else {
                            // T = sum_k S_k 2^(8k) in int64 (exact); y' = fl(T * 2^-38 - M)
                            const long long T = (static_cast<long long>(static_cast<int>(vd[4])) << 32) +
                                                (static_cast<long long>(static_cast<int>(vd[3])) << 24) +
                                                (static_cast<long long>(static_cast<int>(vd[2])) << 16) +
                                                (static_cast<long long>(static_cast<int>(vd[1])) << 8) +
                                                static_cast<long long>(static_cast<int>(vd[0]));
                            const double2 c0 = s_qc[cb + li][d][0];
                            const double zf = __fma_rn(__ll2double_rn(T), c0.x, c0.y);
                            // floor(zf) through the 2^52 rounding trick (no conversion): the nearest
                            // integer to zf - 1/2; a tie only happens at an integer zf, which the
                            // boundary test below flags anyway
                            const double tq = __dadd_rn(zf, 4503599627370495.5);  // zf - 0.5 + 2^52
                            const double qf = __dsub_rn(tq, 4503599627370496.0);
                            const double fr = zf - qf;
                            const double bz = s_qc[cb + li][d][1].x;
                            flag = flag || (fr < bz) || (fr > 1.0 - bz);
                            qi = static_cast<int>(static_cast<uint32_t>(__double_as_longlong(tq)));
                        }
                        const uint32_t q = static_cast<uint32_t>(min(max(qi, 0), 255));
                        if constexpr (D == 8) {
                            // the bytes of the 8 dims (dim 0 on top); the key is their 8x8 bit transpose
                            kw[d < 4 ? 1 : 0] |= q << (8 * (3 - (d & 3)));
                        } else {
                            const int sh = D - 1 - d;
                            uint32_t prev = 0;
#pragma unroll
                            for (int k = 0; k < W; ++k) {
                                const uint32_t cur = s_spread[(lane >> 3) * kSpStride + q * W + k];
                                kw[k] |= sh ? __funnelshift_l(prev, cur, sh) : cur;
                                prev = cur;
                            }
                        }
                    }
                }
                if constexpr (MODE == 1 && D == 8) {
                    // Morton key of 8 dims x 8 bits = the bit transpose of the 8x8 matrix whose row d
                    // is dim d's byte: two delta swaps inside each word, one nibble exchange across
                    uint32_t hi = kw[1], lo = kw[0], t;
                    t = (hi ^ (hi >> 7)) & 0x00AA00AAu, hi = hi ^ t ^ (t << 7);
                    t = (lo ^ (lo >> 7)) & 0x00AA00AAu, lo = lo ^ t ^ (t << 7);
                    t = (hi ^ (hi >> 14)) & 0x0000CCCCu, hi = hi ^ t ^ (t << 14);
                    t = (lo ^ (lo >> 14)) & 0x0000CCCCu, lo = lo ^ t ^ (t << 14);
                    kw[0] = (lo & 0x0F0F0F0Fu) | ((hi & 0x0F0F0F0Fu) << 4);
                    kw[1] = (hi & 0xF0F0F0F0u) | ((lo >> 4) & 0x0F0F0F0Fu);
                }
                if (MODE == 1) {
                    const uint32_t l = static_cast<uint32_t>(P.l0 + cb + li);
                    if (valid) {
                        const uint64_t e = static_cast<uint64_t>(l) * P.n + row;
#pragma unroll
                        for (int k = 0; k < W; ++k) P.keyw[static_cast<size_t>(k) * P.Nrec + e] = kw[k];
                        P.val[e] = P.payload_key ? __ldg(P.keys + row) : (l << 29) | (P.row_base + static_cast<uint32_t>(row));
                    }
                    flag = flag || cand;
                    const uint32_t m = __ballot_sync(0xffffffffu, valid && flag);
                    if (m) {
                        uint32_t base = 0;
                        if (lane == 0) base = atomicAdd(P.list_count, static_cast<uint32_t>(__popc(m)));
                        base = __shfl_sync(0xffffffffu, base, 0);
                        if (valid && flag)
                            P.list[base + __popc(m & ((1u << lane) - 1u))] =
                                (static_cast<uint32_t>(row) << 4) | (cand ? 8u : 0u) | l;
                    }
                }
            }
        }
    }
    if (MODE == 0 && !pt_running<D>() && warp >= kPtGatherWarps && warp < kPtMmaWarp) {
        const int lpar = (warp - kPtGatherWarps) >> 2;
        const int li = kPtEpiSets * (lane / D) + lpar, d = lane % D;
        if (li < nl && tmn0 <= tmx0) {  // the slot saw a valid row: y' of the extreme T (one rounding, as in the epilogue)
            const int l = P.l0 + li;
            const double M = s_M[li][d];
            atomicMin(P.amm + static_cast<size_t>(l) * 2 * D + d, double_to_ordered(__dsub_rn(static_cast<double>(tmn0) * kPtUnit, M)));
            atomicMax(P.amm + static_cast<size_t>(l) * 2 * D + D + d,
                      double_to_ordered(__dsub_rn(static_cast<double>(tmx0) * kPtUnit, M)));
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
    }
}

// ------------------------------------------------------------------ fused exact moments
// K2 without the patch matrix: the same 128-patch A tiles as the projection (gathered from the
// L2-resident image into 128B-swizzled shared memory, feature F = 1 for real patches), used as
// BOTH operands of X^T X through the MN-major (transposed) UMMA descriptors: per tile and per
// 128x128 feature-tile pair (ti <= tj) four tcgen05.mma.kind::i8 (K = 32 patches each) into a
// 128-column TMEM accumulator.  Each CTA (one per SM, more when an SM would get more than 512
// tiles: 65536 patches keep the u32 view of the s32 sums exact) sums its tiles and writes its
// partial Gram; k_gram_reduce adds the partials in int64 (fixed order, no atomics).  Two gather
// groups of 8 warps keep two tiles' gathers in flight.  At most 4 pairs (512 TMEM columns) per
// launch.
constexpr int kGmPairs = 4;
constexpr int kGmChunk = 512;
struct gm_params {
    pt_params P;  // gather fields: img, w, C, KC, F, Fpad, keys, n, ntiles, wtab
    int npair;
    int pti[kGmPairs], ptj[kGmPairs];
    unsigned long long* out;  // F + F*F
    uint32_t* part;           // per-CTA partial Grams [cta][pair][128][128] (k_gram_reduce folds them)
};

__device__ __forceinline__ uint64_t tc_desc_mn128(uint32_t saddr) {  // MN-major, 128B swizzle
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3fffu);
    d |= static_cast<uint64_t>(1u) << 16;            // leading byte offset (one 128-byte atom along M)
    d |= static_cast<uint64_t>(1024u >> 4) << 32;    // stride byte offset: next 8 patches
    d |= static_cast<uint64_t>(1u) << 46;
    d |= static_cast<uint64_t>(2u) << 61;
    return d;
}

#ifndef ZI_GM_GROUPS
#define ZI_GM_GROUPS 2
#endif
constexpr int kGmGroups = ZI_GM_GROUPS;                         // gather groups (tiles i, i + 1 in flight together)
constexpr int kGmThreads = (8 * kGmGroups + 1) * 32;  // 8 gather warps per group + the MMA warp

template <int KT>
__global__ void __launch_bounds__(kGmThreads, 1) k_gram_fused(const __grid_constant__ gm_params G) {
    const pt_params& P = G.P;
    extern __shared__ uint8_t gm_raw[];
    uint8_t* sA = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(gm_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    const uint32_t abytes = static_cast<uint32_t>(kPtRows * P.Fpad);
    constexpr int NB = 2 * kGmGroups;  // a 2-buffer ring per gather group
    __shared__ __align__(8) uint64_t s_afull[NB], s_aempty[NB], s_done;
    __shared__ uint32_t s_tmem;
    __shared__ int2 s_wtab[kPtMaxFpad / 4];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int kMmaWarp = 8 * kGmGroups;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc_smem(&s_tmem)), "r"(512u)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int b = 0; b < NB; ++b) {
            tc_mbar_init(tc_smem(&s_afull[b]), 8);
            tc_mbar_init(tc_smem(&s_aempty[b]), 1);
        }
        tc_mbar_init(tc_smem(&s_done), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < P.Fpad / 4; i += blockDim.x) s_wtab[i] = P.wtab[i];
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;
    // this CTA's tiles: blockIdx.x + i * gridDim.x, i < nloc <= kGmChunk (the host sizes the grid)
    const uint64_t nloc = blockIdx.x < P.ntiles ? (P.ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    if (warp == kMmaWarp) {
        if (lane == 0) {  // MMA issuer: tile i sits in buffer (i % groups) * 2 + ((i / groups) & 1)
            const uint32_t idesc = (2u << 4) | (1u << 15) | (1u << 16) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
            for (uint64_t i = 0; i < nloc; ++i) {
                const uint64_t j = i / kGmGroups;
                const int b = static_cast<int>(i % kGmGroups) * 2 + static_cast<int>(j & 1);
                tc_mbar_wait(tc_smem(&s_afull[b]), static_cast<uint32_t>((j >> 1) & 1));
                tc_fence_after();
                const uint32_t a0 = tc_smem(sA + b * abytes);
                for (int p = 0; p < G.npair; ++p) {
                    const uint32_t ta = a0 + static_cast<uint32_t>(G.pti[p]) * kPtRows * 128;
                    const uint32_t tb = a0 + static_cast<uint32_t>(G.ptj[p]) * kPtRows * 128;
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks)
                        pt_mma(tmem + static_cast<uint32_t>(p * 128), tc_desc_mn128(ta + ks * 4096), tc_desc_mn128(tb + ks * 4096),
                               idesc, (i | ks) != 0 ? 1u : 0u);
                }
                tc_commit(tc_smem(&s_aempty[b]));
            }
            tc_commit(tc_smem(&s_done));
        }
    } else {  // gather group g = warp / 8 takes tiles g, g + groups, ...: two threads per patch row
        const int g = warp / 8, gw = warp % 8;
        const int nchunk = P.Fpad >> 4, hc = (nchunk + 1) >> 1;
        const int r = (gw * 32 + lane) & 127, gh = gw >> 2;
        for (uint64_t i = g, j = 0; i < nloc; i += kGmGroups, ++j) {
            const int b = g * 2 + static_cast<int>(j & 1);
            if (j >= 2) tc_mbar_wait(tc_smem(&s_aempty[b]), static_cast<uint32_t>(((j >> 1) - 1) & 1));
            const uint64_t tile = blockIdx.x + i * gridDim.x;
            const uint32_t sa = tc_smem(sA + b * abytes);
            if (KT == 0) {
                pt_gather(P, s_wtab, tile, sa, r, gh ? hc : 0, gh ? nchunk : hc);
            } else {
                const uint64_t pr = tile * kPtRows + r;
                const bool valid = pr < P.n;
                uint32_t base = 0;
                if (valid) {
                    const uint32_t key = __ldg(P.keys + pr);
                    base = ((key >> 16) * static_cast<uint32_t>(P.w) + (key & 0xffffu)) * static_cast<uint32_t>(P.C);
                }
                const uint32_t wC = static_cast<uint32_t>(P.w * P.C);
                if (KT == 1) {
                    if (gh) pt_gather_static<9, 1, 1>(P.img, base, wC, valid, sa, r);
                    else pt_gather_static<9, 1, 0>(P.img, base, wC, valid, sa, r);
                } else {
                    if (gh) pt_gather_static<11, 3, 1>(P.img, base, wC, valid, sa, r);
                    else pt_gather_static<11, 3, 0>(P.img, base, wC, valid, sa, r);
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) tc_mbar_arrive(tc_smem(&s_afull[b]));
        }
        if (warp < 4) {  // epilogue: this CTA's partial Gram (TMEM lane = feature row of tile ti), u32 exact
            if (nloc > 0) {
                tc_mbar_wait(tc_smem(&s_done), 0);
                tc_fence_after();
            }
            const int row = warp * 32 + lane;
            for (int p = 0; p < G.npair; ++p) {
                uint4* dst = reinterpret_cast<uint4*>(G.part + ((static_cast<size_t>(blockIdx.x) * G.npair + p) * kPtRows + row) * 128);
                for (int cb = 0; cb < 128; cb += 4) {
                    uint32_t v[4] = {0u, 0u, 0u, 0u};
                    if (nloc > 0) {
                        tc_ld_x4(tmem + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>(p * 128 + cb), v);
                        tc_ld_wait();
                    }
                    dst[cb >> 2] = make_uint4(v[0], v[1], v[2], v[3]);
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
    }
}

// sum of the per-CTA partial Grams in int64 into the moments (every output has one owner: no atomics)
struct gm_pairs {
    int pti[kGmPairs], ptj[kGmPairs];
};
__global__ void __launch_bounds__(256) k_gram_reduce(const uint32_t* __restrict__ part, int nblocks, int npair,
                                                     const gm_pairs pairs, int F, unsigned long long* __restrict__ out) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= npair * 128 * 128) return;
    const int p = idx >> 14, r = (idx >> 7) & 127, c = idx & 127;
    const int fi = pairs.pti[p] * kPtRows + r, fj = pairs.ptj[p] * kPtRows + c;
    if (fi >= F || fj > F) return;
    unsigned long long acc = 0;
    const size_t stride = static_cast<size_t>(npair) * 128 * 128;
    for (int b = 0; b < nblocks; ++b) acc += __ldg(part + b * stride + idx);
    if (fj < F) out[F + static_cast<size_t>(fi) * F + fj] += acc;
    else out[fi] += acc;
}

template <int KT>
static void launch_gram(zi_ctx* ctx, const gm_params& G, size_t smem) {
    smem_attr(ctx->device, k_gram_fused<KT>, smem);
    // one CTA per SM, more when an SM would sum more than kGmChunk tiles (65536 patches: the
    // u32 view of the s32 accumulators stays exact)
    // -- rounded up to whole waves (the 512-column TMEM allocation keeps one CTA per SM, so a grid
    // of 1.5 waves would leave a third of the SMs idle for the second half)
    const uint64_t sms = static_cast<uint64_t>(ctx->num_sms);
    const uint64_t want = (std::max<uint64_t>(sms, (G.P.ntiles + kGmChunk - 1) / kGmChunk) + sms - 1) / sms * sms;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(G.P.ntiles, want));
    gm_params g = G;
    g.part = reinterpret_cast<uint32_t*>(ctx->scratch.ensure(static_cast<size_t>(grid) * G.npair * 128 * 128 * 4 + 256));
    ZI_LAUNCH(ctx, "patch_moments_fused", k_gram_fused<KT>, grid, kGmThreads, smem, g);
    gm_pairs pairs{};  // by value: no upload of the tile pairs
    for (int i = 0; i < kGmPairs; ++i) {
        pairs.pti[i] = G.pti[i];
        pairs.ptj[i] = G.ptj[i];
    }
    const int outs = G.npair * 128 * 128;
    ZI_LAUNCH(ctx, "patch_moments_reduce", k_gram_reduce, (outs + 255) / 256, 256, 0, g.part, static_cast<int>(grid), G.npair,
              pairs, G.P.F, G.out);
}

// exact moments of the n patches at d_keys (row-major key order) straight from the image;
// false when the patch shape is outside the envelope (F >= Fpad or Fpad > 384)
bool patch_moments_fused(zi_ctx* ctx, const uint8_t* d_img, int w, int C, int K, const uint32_t* d_keys, uint64_t n,
                         unsigned long long* d_out, dbuf<int2>& wtab) {
    static const bool off_env = std::getenv("ZI_MOMENTS_TMA") != nullptr;
    const int F = K * K * C, Fpad = (F + 127) / 128 * 128;
    if (off_env || F >= Fpad || Fpad > kPtMaxFpad || n == 0 || n >= (1ull << 31)) return false;
    {  // gather word table (as the projection's)
        const int KC = K * C, wC = w * C;
        std::vector<int2> tab(Fpad / 4);
        for (int ow = 0; ow < Fpad / 4; ++ow) {
            const int f = 4 * ow;
            if (f >= F) {
                tab[ow] = make_int2(-1, -1);
                continue;
            }
            const int rr = f / KC, k = f - rr * KC, rem = KC - k;
            int y = -1;
            if (rem < 4) y = (rem << 24) | (rr + 1 < K ? (rr + 1) * wC : 0xffffff);
            tab[ow] = make_int2(rr * wC + k, y);
        }
        wtab.ensure(tab.size());
        ZI_CUDA(cudaMemcpyAsync(wtab.p, tab.data(), tab.size() * sizeof(int2), cudaMemcpyHostToDevice, ctx->stream));
    }
    gm_params G{};
    G.P.img = d_img;
    G.P.w = w;
    G.P.C = C;
    G.P.KC = K * C;
    G.P.F = F;
    G.P.Fpad = Fpad;
    G.P.keys = d_keys;
    G.P.n = n;
    G.P.ntiles = (n + kPtRows - 1) / kPtRows;
    G.P.wtab = wtab.p;
    G.out = d_out;
    const int nt = Fpad / 128;
    const int kt = K * C == 9 && F == 81 ? 1 : (K * C == 33 && F == 363 ? 2 : 0);
    // >= 116 KB: one CTA per SM, so no second CTA waits on the first one's 512 TMEM columns
    const size_t smem = std::max<size_t>(2 * kGmGroups * static_cast<size_t>(kPtRows) * Fpad + 1024, 116 * 1024);
    if (smem > 220 * 1024) return false;
    std::vector<int2> pairs;
    for (int ti = 0; ti < nt; ++ti)
        for (int tj = ti; tj < nt; ++tj) pairs.push_back(make_int2(ti, tj));
    for (size_t p0 = 0; p0 < pairs.size(); p0 += kGmPairs) {
        G.npair = static_cast<int>(std::min<size_t>(kGmPairs, pairs.size() - p0));
        for (int p = 0; p < G.npair; ++p) {
            G.pti[p] = pairs[p0 + p].x;
            G.ptj[p] = pairs[p0 + p].y;
        }
        if (kt == 1) launch_gram<1>(ctx, G, smem);
        else if (kt == 2) launch_gram<2>(ctx, G, smem);
        else launch_gram<0>(ctx, G, smem);
    }
    return true;
}

// digit matrices of all groups (pre-zeroed) and M = sum_j mean_j c_j, from the device models
__global__ void k_pt_prep(const double* __restrict__ mean, const double* __restrict__ comp,
                          const int32_t* __restrict__ cols, int mc, int D, int nlmax, int Fpad,
                          const int* __restrict__ goff, const int* __restrict__ gnpad, uint8_t* __restrict__ B,
                          double* __restrict__ M) {
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int total = 8 * mc * D;
    if (tid < total) {
        const int l = tid / (mc * D), rem = tid - l * mc * D, j = rem / D, d = rem - j * D;
        const double c = comp[(static_cast<size_t>(l) * mc + j) * D + d];
        long long t = llrint(c * kPtScale);  // exact scaling by 2^38, then round to nearest
        const int g = l / nlmax, li = l - g * nlmax;
        const int f = cols[l * mc + j];
        for (int k = 0; k < kPtDigits; ++k) {
            long long dg = ((t + 128) & 255) - 128;  // balanced digit in [-128, 127]
            t = (t - dg) >> 8;
            const int row = (li * D + d) * kPtDigits + k;
            B[goff[g] + sw128_off(row, f, gnpad[g])] = static_cast<uint8_t>(static_cast<int8_t>(dg));
        }
    }
    if (tid < 8 * D) {
        const int l = tid / D, d = tid - l * D;
        double s = 0.0;
        for (int j = 0; j < mc; ++j) s = __fma_rn(mean[l * mc + j], comp[(static_cast<size_t>(l) * mc + j) * D + d], s);
        M[tid] = s;
    }
}

// Canonical fp64 projection of the listed (patch, layout) pairs: one warp per pair.  The lanes
// gather the pair's centred pixel values xc_j = x_j - mean_j into shared memory (independent
// loads), then lane d runs the dimension's fma chain over j ascending from +0.0 -- the order
// k_project runs on the FP64 MMA -- with the component loads pipelined ahead of the chain.
// MODE 0: exact lo / hi (ordered atomics, candidates only); MODE 1: exact quantised record.
constexpr int kPtxWarps = 4;
template <int D, int MODE>
__global__ void __launch_bounds__(kPtxWarps * 32) k_pt_exact(const uint8_t* __restrict__ img, int w, int C,
                                                             const uint32_t* __restrict__ keys, uint64_t n,
                                                             uint32_t row_base, const int32_t* __restrict__ off, int m,
                                                             const double* __restrict__ mean,
                                                             const double* __restrict__ comp,
                                                             const uint32_t* __restrict__ list,
                                                             const uint32_t* __restrict__ list_count,
                                                             unsigned long long* __restrict__ minmax,
                                                             uint32_t* __restrict__ keyw, uint32_t* __restrict__ val,
                                                             uint64_t Nrec, int payload_key) {
    constexpr int W = (D + 3) / 4;
    __shared__ double s_xc[kPtxWarps][232];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint32_t cnt = *list_count;
    const int mc = m * C;
    double* xc = s_xc[wib];
    for (uint64_t e = static_cast<uint64_t>(blockIdx.x) * kPtxWarps + wib; e < cnt;
         e += static_cast<uint64_t>(gridDim.x) * kPtxWarps) {
        const uint32_t ent = list[e];
        if (MODE == 0 && !(ent & 8u)) continue;  // only the lo / hi candidates take part in the min / max
        const uint32_t row = ent >> 4, l = ent & 7;
        const uint32_t key = keys[row];
        const uint8_t* pb = img + static_cast<size_t>((key >> 16) * static_cast<uint32_t>(w) + (key & 0xffffu)) * C;
        for (int j = lane; j < mc; j += 32) {
            const int p = j / C, ch = j - p * C;
            xc[j] = __dsub_rn(static_cast<double>(__ldg(pb + __ldg(off + l * m + p) + ch)), __ldg(mean + l * mc + j));
        }
        __syncwarp();
        double y = 0.0;
        if (lane < D) {
            const double* cp = comp + static_cast<size_t>(l) * mc * D + lane;
#pragma unroll 8
            for (int j = 0; j < mc; ++j) y = __fma_rn(xc[j], __ldg(cp + static_cast<size_t>(j) * D), y);
        }
        __syncwarp();
        unsigned long long* mm = minmax + static_cast<size_t>(l) * 2 * D;
        if (MODE == 0) {
            if (lane < D) {
                const unsigned long long o = double_to_ordered(y);
                atomicMin(mm + lane, o);
                atomicMax(mm + D + lane, o);
            }
        } else {
            uint32_t q = 0;
            if (lane < D) {
                const double lo = ordered_to_double_hd(mm[lane]), hi = ordered_to_double_hd(mm[D + lane]);
                const double rcp = hi > lo ? __ddiv_rn(1.0, __dsub_rn(hi, lo)) : 0.0;
                q = quantize_fast(lo, hi, rcp, y);
            }
            const uint64_t er = static_cast<uint64_t>(l) * n + row;
#pragma unroll
            for (int k = 0; k < W; ++k) {
                uint32_t part = 0;
                if (lane < D)
#pragma unroll
                    for (int L = 0; L < 8; ++L) {
                        const int pos = L * D + D - 1 - lane;
                        if ((pos >> 5) == k) part |= ((q >> L) & 1u) << (pos & 31);
                    }
                const uint32_t word = __reduce_or_sync(0xffffffffu, part);
                if (lane == 0) keyw[static_cast<size_t>(k) * Nrec + er] = word;
            }
            if (lane == 0) val[er] = payload_key ? key : (l << 29) | (row_base + row);
        }
    }
}

template <int D>
static void launch_pt_exact(zi_ctx* ctx, zi_multi_index* mi, const pt_params& P, int mode) {
    const unsigned grid = static_cast<unsigned>(ctx->num_sms) * 8;
    const uint32_t* keys = mi->dict.p + mi->row_begin;
    const uint32_t rb = static_cast<uint32_t>(mi->row_begin);
    if (mode == 0)
        ZI_LAUNCH(ctx, "project_tc_exact_minmax", (k_pt_exact<D, 0>), grid, kPtxWarps * 32, 0, mi->image.p, mi->w, mi->C, keys, mi->n,
                  rb, mi->layout_off.p, mi->m, mi->pca_mean.p, mi->pca_comp.p, P.list, P.list_count, mi->minmax.p, P.keyw,
                  P.val, P.Nrec, P.payload_key);
    else
        ZI_LAUNCH(ctx, "project_tc_fixup", (k_pt_exact<D, 1>), grid, kPtxWarps * 32, 0, mi->image.p, mi->w, mi->C, keys, mi->n, rb,
                  mi->layout_off.p, mi->m, mi->pca_mean.p, mi->pca_comp.p, P.list, P.list_count, mi->minmax.p, P.keyw,
                  P.val, P.Nrec, P.payload_key);
}

template <int D, int KT>
static void launch_pt_kt(zi_ctx* ctx, const pt_params& P, int mode, size_t smem) {
    if (mode == 0) smem_attr(ctx->device, k_proj_tc<D, 0, KT>, 200 * 1024);
    else smem_attr(ctx->device, k_proj_tc<D, 1, KT>, 200 * 1024);
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(P.ntiles, static_cast<uint64_t>(ctx->num_sms)));
    if (mode == 0) ZI_LAUNCH(ctx, "project_tc_minmax", (k_proj_tc<D, 0, KT>), grid, (pt_shape<D, 0>::kThreads), smem, P);
    else ZI_LAUNCH(ctx, "project_tc_quantize", (k_proj_tc<D, 1, KT>), grid, (pt_shape<D, 1>::kThreads), smem, P);
}

// patch shapes with a static gather: (9, 1) -> 1 (cfg1, cfg4), (11, 3) -> 2 (cfg2); for the dims
// those configs use, everything else takes the table-driven gather
template <int D>
static void launch_pt(zi_ctx* ctx, const pt_params& P, int mode, size_t smem) {
    const int kt = P.KC == 9 && P.F == 81 ? 1 : (P.KC == 33 && P.F == 363 ? 2 : 0);
    if constexpr (D == 8) {
        if (kt == 1) return launch_pt_kt<D, 1>(ctx, P, mode, smem);
    }
    if constexpr (D == 8 || D == 12) {
        if (kt == 2) return launch_pt_kt<D, 2>(ctx, P, mode, smem);
    }
    launch_pt_kt<D, 0>(ctx, P, mode, smem);
}

// The plan of one projection: eligibility, layout groups, scratch offsets, kernel parameters.
struct pt_plan {
    bool ok = false;
    uint8_t* s = nullptr;  // the scratch the offsets below point into
    int D = 0, ng = 0, nlmax = 0, goff[8] = {}, gnpad[8] = {};
    bool fuse = false;  // both layout groups in one launch (two accumulator halves per gathered tile)
    size_t smem = 0, btot = 0, o_B = 0, o_M = 0, o_amm = 0, o_cnt = 0, o_list = 0;
    pt_params P{};
};

// eligibility depends on the configuration only (dims, patch shape, the dictionary size), never on
// this rank's slice, so every shard of a sharded build takes the same path
static pt_plan pt_make_plan(zi_multi_index* mi, uint32_t* keyw, uint32_t* val, uint64_t Nrec) {
    pt_plan pl;
    static const bool off_env = std::getenv("ZI_PROJ_FP64") != nullptr;
    const int D = mi->dims, K = mi->K, C = mi->C, mc = mi->mc;
    const int F = K * K * C, Fpad = (F + 127) / 128 * 128;
    const uint64_t n = mi->n, ntot = mi->shard ? mi->n_total : mi->n;
    if (off_env || D < 1 || D > 16 || Fpad > kPtMaxFpad || mc > 232 || ntot == 0 || ntot >= (1ull << 27)) return pl;
    pl.D = D;
    // as few 256-column groups as fit, with the layouts spread evenly over them (D = 8: 4 + 4, not
    // 6 + 2 -- the small group's launch costs as much gather as the big one's)
    pl.nlmax = std::min(8, kPtMaxN / (kPtDigits * D));
    pl.ng = (8 + pl.nlmax - 1) / pl.nlmax;
    pl.nlmax = (8 + pl.ng - 1) / pl.ng;
    for (int g = 0; g < pl.ng; ++g) {
        const int nl = std::min(pl.nlmax, 8 - g * pl.nlmax);
        pl.gnpad[g] = (nl * kPtDigits * D + 15) / 16 * 16;
        pl.goff[g] = static_cast<int>(pl.btot);
        pl.btot += static_cast<size_t>(pl.gnpad[g]) * Fpad;
    }
    pl.smem = 2 * static_cast<size_t>(kPtRows) * Fpad + static_cast<size_t>(kPtMaxN) * Fpad + 1024;
    if (pl.smem > 200 * 1024) return pl;
    {
        // two equal groups of four layouts whose min / max pass keeps lane-slot extremes: one launch
        // gathers every A tile once and fills both groups' accumulators from it
        static const bool nofuse_env = std::getenv("ZI_PROJ_NOFUSE") != nullptr;
        const size_t fsmem = 2 * static_cast<size_t>(kPtRows) * Fpad + 2 * static_cast<size_t>(pl.gnpad[0]) * Fpad + 1024;
        pl.fuse = !nofuse_env && pl.ng == 2 && pl.nlmax == 4 && pl.gnpad[0] == pl.gnpad[1] && D >= 7 && D <= 10 &&
                  fsmem <= 200 * 1024;
        if (pl.fuse) pl.smem = std::max(pl.smem, fsmem);
    }
    // scratch: [goff/gnpad ints][B bytes][M doubles][amm][count][list]
    pl.o_B = 256;
    pl.o_M = (pl.o_B + pl.btot + 255) & ~size_t(255);
    pl.o_amm = pl.o_M + 8 * 16 * sizeof(double);
    pl.o_cnt = pl.o_amm + 8 * 2 * 16 * sizeof(unsigned long long);
    pl.o_list = pl.o_cnt + 256;
    uint8_t* s = mi->pt_scratch.ensure(pl.o_list + 8 * (n ? n : 1) * sizeof(uint32_t));
    pl.s = s;
    pt_params& P = pl.P;
    P.img = mi->image.p;
    P.w = mi->w;
    P.C = C;
    P.KC = K * C;
    P.F = F;
    P.Fpad = Fpad;
    P.keys = mi->dict.p + mi->row_begin;
    P.n = n;
    P.row_base = static_cast<uint32_t>(mi->row_begin);
    P.payload_key = mi->payload_key ? 1 : 0;
    P.M = reinterpret_cast<const double*>(s + pl.o_M);
    P.amm = reinterpret_cast<unsigned long long*>(s + pl.o_amm);
    P.E = 255.0 * mc * (0.5 * kPtUnit + 0x1p-44);
    P.keyw = keyw;
    P.val = val;
    P.Nrec = Nrec;
    P.list = reinterpret_cast<uint32_t*>(s + pl.o_list);
    P.list_count = reinterpret_cast<uint32_t*>(s + pl.o_cnt);
    P.ntiles = (n + kPtRows - 1) / kPtRows;
    P.wtab = mi->pt_wtab.p;
    pl.ok = true;
    return pl;
}

static void pt_launch_pass(zi_ctx* ctx, pt_plan& pl, int mode) {
    if (pl.P.n == 0) return;
    for (int g = 0; g < pl.ng; ++g) {
        pt_params P = pl.P;
        P.B = pl.s + pl.o_B + pl.goff[g];
        P.Npad = pl.gnpad[g];
        P.l0 = g * pl.nlmax;
        P.nl = std::min(pl.nlmax, 8 - g * pl.nlmax);
        P.nhalf = pl.fuse ? 2 : 1;
        switch (pl.D) {
#define ZI_PT_CASE(DD) \
    case DD: launch_pt<DD>(ctx, P, mode, pl.smem); break;
            ZI_PT_CASE(1) ZI_PT_CASE(2) ZI_PT_CASE(3) ZI_PT_CASE(4) ZI_PT_CASE(5) ZI_PT_CASE(6) ZI_PT_CASE(7)
            ZI_PT_CASE(8) ZI_PT_CASE(9) ZI_PT_CASE(10) ZI_PT_CASE(11) ZI_PT_CASE(12) ZI_PT_CASE(13)
            ZI_PT_CASE(14) ZI_PT_CASE(15) ZI_PT_CASE(16)
#undef ZI_PT_CASE
            default: throw error(ZI_E_INVALID, "projection: dims above 16");
        }
        if (pl.fuse) break;  // the launch covered both groups
    }
}

static void pt_launch_exact(zi_ctx* ctx, zi_multi_index* mi, pt_plan& pl, int mode) {
    if (pl.P.n == 0) return;
    switch (pl.D) {
#define ZI_PTX_CASE(DD) \
    case DD: launch_pt_exact<DD>(ctx, mi, pl.P, mode); break;
        ZI_PTX_CASE(1) ZI_PTX_CASE(2) ZI_PTX_CASE(3) ZI_PTX_CASE(4) ZI_PTX_CASE(5) ZI_PTX_CASE(6) ZI_PTX_CASE(7)
        ZI_PTX_CASE(8) ZI_PTX_CASE(9) ZI_PTX_CASE(10) ZI_PTX_CASE(11) ZI_PTX_CASE(12) ZI_PTX_CASE(13)
        ZI_PTX_CASE(14) ZI_PTX_CASE(15) ZI_PTX_CASE(16)
#undef ZI_PTX_CASE
        default: break;
    }
}

// phase A: digit matrices, gather table, identity ranges, the min / max pass -> approximate
// ranges (ordered u64) in the plan's scratch
static void pt_phase_a(zi_multi_index* mi, pt_plan& pl) {
    zi_ctx* ctx = mi->ctx;
    const int D = pl.D, K = mi->K, C = mi->C, m = mi->m, mc = mi->mc;
    const int F = K * K * C, Fpad = pl.P.Fpad;
    if (!mi->pca_cols_ready) {
        std::vector<int32_t> hc;
        for (int l = 0; l < 8; ++l)
            for (int p = 0; p < m; ++p)
                for (int ch = 0; ch < C; ++ch) hc.push_back((mi->L[l].rc[2 * p] * K + mi->L[l].rc[2 * p + 1]) * C + ch);
        mi->pca_cols.ensure(hc.size());
        ZI_CUDA(cudaMemcpyAsync(mi->pca_cols.p, hc.data(), hc.size() * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
        ZI_CUDA(cudaStreamSynchronize(ctx->stream));
        mi->pca_cols_ready = true;
    }
    uint8_t* s = pl.s;
    int hint[16];
    for (int g = 0; g < 8; ++g) {
        hint[g] = g < pl.ng ? pl.goff[g] : 0;
        hint[8 + g] = g < pl.ng ? pl.gnpad[g] : 0;
    }
    ZI_CUDA(cudaMemcpyAsync(s, hint, sizeof(hint), cudaMemcpyHostToDevice, ctx->stream));
    {  // gather word table: patch-relative byte offsets of every 4-byte word of the row
        const int KC = K * C, wC = mi->w * C;
        std::vector<int2> tab(Fpad / 4);
        for (int ow = 0; ow < Fpad / 4; ++ow) {
            const int f = 4 * ow;
            if (f >= F) {
                tab[ow] = make_int2(-1, -1);
                continue;
            }
            const int rr = f / KC, k = f - rr * KC, rem = KC - k;
            int y = -1;
            if (rem < 4) y = (rem << 24) | (rr + 1 < K ? (rr + 1) * wC : 0xffffff);
            tab[ow] = make_int2(rr * wC + k, y);
        }
        mi->pt_wtab.ensure(tab.size());
        ZI_CUDA(cudaMemcpyAsync(mi->pt_wtab.p, tab.data(), tab.size() * sizeof(int2), cudaMemcpyHostToDevice, ctx->stream));
        pl.P.wtab = mi->pt_wtab.p;
    }
    ZI_CUDA(cudaMemsetAsync(s + pl.o_B, 0, pl.btot, ctx->stream));
    ZI_CUDA(cudaMemsetAsync(s + pl.o_cnt, 0, sizeof(uint32_t), ctx->stream));
    unsigned long long* amm = pl.P.amm;
    for (int l = 0; l < 8; ++l) {
        ZI_CUDA(cudaMemsetAsync(amm + static_cast<size_t>(l) * 2 * D, 0xff, D * sizeof(unsigned long long), ctx->stream));
        ZI_CUDA(cudaMemsetAsync(amm + static_cast<size_t>(l) * 2 * D + D, 0, D * sizeof(unsigned long long), ctx->stream));
        ZI_CUDA(cudaMemsetAsync(mi->minmax.p + static_cast<size_t>(l) * 2 * D, 0xff, D * sizeof(unsigned long long), ctx->stream));
        ZI_CUDA(cudaMemsetAsync(mi->minmax.p + static_cast<size_t>(l) * 2 * D + D, 0, D * sizeof(unsigned long long), ctx->stream));
    }
    const int* dgoff = reinterpret_cast<const int*>(s);
    const int total = 8 * mc * D;
    ZI_LAUNCH(ctx, "project_tc_prep", k_pt_prep, (total + 255) / 256, 256, 0, mi->pca_mean.p, mi->pca_comp.p,
              mi->pca_cols.p, mc, D, pl.nlmax, Fpad, dgoff, dgoff + 8, s + pl.o_B, reinterpret_cast<double*>(s + pl.o_M));
    pt_launch_pass(ctx, pl, 0);
}

// phase B: the quantise pass with the (global) approximate ranges, then the exact lo / hi over the
// listed candidates into mi->minmax
static void pt_phase_b(zi_multi_index* mi, pt_plan& pl) {
    pt_launch_pass(mi->ctx, pl, 1);
    static const bool debug = std::getenv("ZI_DEBUG_PT") != nullptr;
    if (debug) {
        uint32_t cnt = 0;
        ZI_CUDA(cudaMemcpyAsync(&cnt, pl.P.list_count, sizeof(cnt), cudaMemcpyDeviceToHost, mi->ctx->stream));
        ZI_CUDA(cudaStreamSynchronize(mi->ctx->stream));
        std::vector<uint32_t> hl(cnt);
        if (cnt) ZI_CUDA(cudaMemcpy(hl.data(), pl.P.list, cnt * sizeof(uint32_t), cudaMemcpyDeviceToHost));
        uint64_t ncand = 0, per_l[8] = {};
        for (uint32_t e : hl) {
            ncand += (e >> 3) & 1u;
            ++per_l[e & 7u];
        }
        std::vector<unsigned long long> amm(16 * pl.D);
        ZI_CUDA(cudaMemcpy(amm.data(), pl.P.amm, amm.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        std::fprintf(stderr, "project_tc: n=%llu D=%d groups=%d fix-up list %u (%.4f%% of patch x layout pairs), %llu lo/hi candidates; per layout",
                     static_cast<unsigned long long>(pl.P.n), pl.D, pl.ng, cnt, 100.0 * cnt / (8.0 * std::max<uint64_t>(pl.P.n, 1)),
                     static_cast<unsigned long long>(ncand));
        for (int l = 0; l < 8; ++l) std::fprintf(stderr, " %llu", static_cast<unsigned long long>(per_l[l]));
        std::fprintf(stderr, "\n  ranges(layout 0):");
        for (int d = 0; d < pl.D; ++d) {
            const double lo = ordered_to_double_hd(amm[d]), hi = ordered_to_double_hd(amm[pl.D + d]);
            std::fprintf(stderr, " %.3g", hi - lo);
        }
        std::fprintf(stderr, "\n");
    }
    pt_launch_exact(mi->ctx, mi, pl, 0);
}

// phase C: the exact records of the listed pairs with the (global) exact lo / hi
static void pt_phase_c(zi_multi_index* mi, pt_plan& pl) { pt_launch_exact(mi->ctx, mi, pl, 1); }

bool project_quantize_tc(zi_multi_index* mi, uint32_t* keyw, uint32_t* val, uint64_t Nrec) {
    pt_plan pl = pt_make_plan(mi, keyw, val, Nrec);
    if (!pl.ok) return false;
    pt_phase_a(mi, pl);
    pt_phase_b(mi, pl);
    pt_phase_c(mi, pl);
    return true;
}

// sharded build (shard.cu): the same three phases with all-reduces between them
bool shard_tc_begin(zi_multi_index* mi, uint32_t* keyw, uint32_t* val, uint64_t Nrec, unsigned long long* amm_out) {
    pt_plan pl = pt_make_plan(mi, keyw, val, Nrec);
    if (!pl.ok) return false;
    pt_phase_a(mi, pl);
    ZI_CUDA(cudaMemcpyAsync(amm_out, pl.P.amm, static_cast<size_t>(8) * 2 * pl.D * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, mi->ctx->stream));
    ZI_CUDA(cudaStreamSynchronize(mi->ctx->stream));
    return true;
}

void shard_tc_quantize(zi_multi_index* mi, uint32_t* keyw, uint32_t* val, uint64_t Nrec, const unsigned long long* amm,
                       unsigned long long* exact_out) {
    pt_plan pl = pt_make_plan(mi, keyw, val, Nrec);
    ZI_CUDA(cudaMemcpyAsync(pl.P.amm, amm, static_cast<size_t>(8) * 2 * pl.D * sizeof(unsigned long long),
                            cudaMemcpyHostToDevice, mi->ctx->stream));
    pt_phase_b(mi, pl);
    ZI_CUDA(cudaMemcpyAsync(exact_out, mi->minmax.p, static_cast<size_t>(8) * 2 * pl.D * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, mi->ctx->stream));
    ZI_CUDA(cudaStreamSynchronize(mi->ctx->stream));
}

void shard_tc_fixup(zi_multi_index* mi, uint32_t* keyw, uint32_t* val, uint64_t Nrec) {
    pt_plan pl = pt_make_plan(mi, keyw, val, Nrec);
    pt_phase_c(mi, pl);
}

}  // namespace zi
