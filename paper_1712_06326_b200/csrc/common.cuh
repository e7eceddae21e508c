// common.cuh -- device helpers shared by the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "zi_internal.h"

#define ZI_LAUNCH(ctx, name, kernel, grid, block, smem, ...)                    \
    do {                                                                        \
        ::zi::launch_begin((ctx), (name));                                      \
        kernel<<<(grid), (block), (smem), (ctx)->stream>>>(__VA_ARGS__);        \
        ::zi::check_launch(name);                                               \
        ::zi::launch_end((ctx), (name));                                        \
    } while (0)

namespace zi {

constexpr uint64_t kU64Max = ~0ull;

// Order-preserving map of a finite double onto uint64 (used for atomic min/max of lo/hi).
__host__ __device__ inline unsigned long long double_to_ordered(double x) {
    unsigned long long b;
#ifdef __CUDA_ARCH__
    b = static_cast<unsigned long long>(__double_as_longlong(x));
#else
    std::memcpy(&b, &x, sizeof(b));
#endif
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

__host__ __device__ inline double ordered_to_double_hd(unsigned long long u) {
    const unsigned long long b = (u & 0x8000000000000000ull) ? (u & 0x7fffffffffffffffull) : ~u;
#ifdef __CUDA_ARCH__
    return __longlong_as_double(static_cast<long long>(b));
#else
    double x;
    std::memcpy(&x, &b, sizeof(x));
    return x;
#endif
}

// quantizer::quantize (proj/src/builder.cpp:55-61): IEEE ops spelled out so nothing is fused.
__device__ inline uint8_t quantize_rn(double l, double h, double y) {
    if (!(h > l)) return 0;
    const double c = y < l ? l : (h < y ? h : y);
    const double v = __ddiv_rn(__dmul_rn(255.0, __dsub_rn(c, l)), __dsub_rn(h, l));
    return static_cast<uint8_t>(llround(v));
}

// Same result as quantize_rn with the IEEE division replaced by a multiply with the rounded
// reciprocal whenever that provably cannot change llround(): |t*r - t/(h-l)| < 2^-44.5 for
// quotients below 256, so unless the approximate quotient lies within 8 ulp (2^-41) of a
// half-integer the rounded integer is the same; otherwise the exact __ddiv_rn is taken.
__device__ inline uint8_t quantize_fast(double l, double h, double rcp, double y) {
    if (!(h > l)) return 0;
    const double c = y < l ? l : (h < y ? h : y);
    const double t = __dmul_rn(255.0, __dsub_rn(c, l));
    double v = __dmul_rn(t, rcp);
    const double f = v - floor(v);
    if (fabs(f - 0.5) <= 4.547473508864641e-13 /* 2^-41 */) v = __ddiv_rn(t, __dsub_rn(h, l));
    return static_cast<uint8_t>(llround(v));
}

// less_most_significant_bit / morton_less (proj/include/zinpaint/morton.hpp:10-29)
__device__ inline bool less_msb(uint32_t a, uint32_t b) { return (a < b) && (a < (a ^ b)); }

__device__ inline uint32_t plane_byte(uint32_t w, int d) { return (w >> ((d & 3) * 8)) & 0xffu; }

// Morton bit position (from the LSB) of bit L of dim d in a D-dim, 8-bit interleave:
// level 7 first, dim 0 first within a level  ->  u = L*D + (D-1-d).
__host__ __device__ inline int morton_bit(int L, int d, int D) { return L * D + (D - 1 - d); }

__device__ inline uint64_t pack_candidate(uint32_t dist, uint32_t key) {
    return (static_cast<uint64_t>(dist) << 32) | key;
}

// distance of 4 packed bytes (L2 squared / L1)
__device__ inline uint32_t dist4(uint32_t a, uint32_t b, int norm, uint32_t acc) {
    const uint32_t d = __vabsdiffu4(a, b);
    return norm == 0 ? __dp4a(d, d, acc) : __dp4a(d, 0x01010101u, acc);
}

// lower bound of the distance from q to the byte box [mn, mx] over 4 packed dims
__device__ inline uint32_t gap4(uint32_t q, uint32_t mn, uint32_t mx, int norm, uint32_t acc) {
    const uint32_t g = __vsubus4(mn, q) | __vsubus4(q, mx);
    return norm == 0 ? __dp4a(g, g, acc) : __dp4a(g, 0x01010101u, acc);
}

template <typename T>
__device__ inline T warp_min(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        T u = __shfl_xor_sync(0xffffffffu, v, o);
        v = u < v ? u : v;
    }
    return v;
}

// Morton key words -> dim planes (4 dims per u32), shared by finalize (k_build.cu) and the sort's
// fused last pass (k_sort.cu).  Morton de-interleave by 8x8 bit-matrix transposes, no tables (a lookup per key byte and plane
// word was 12% slower in finalize; the quantiser keeps its spread table, which measured faster).  Key bit L*D + D-1-d
// is bit L of dim d (proj/include/zinpaint/morton.hpp:14-29); dims go in chunks of 8: chunk c
// holds dims 8c..8c+7, and its level-L byte (bit 7-r = bit L of dim 8c+r) sits at key bit
// L*D + D-8-8c (a negative offset drops the bits of dims >= D, which are zero).
__device__ __forceinline__ uint64_t transpose8x8(uint64_t x) {  // byte i bit j <-> byte j bit i
    x = (x & 0xAA55AA55AA55AA55ull) | ((x & 0x00AA00AA00AA00AAull) << 7) | ((x >> 7) & 0x00AA00AA00AA00AAull);
    x = (x & 0xCCCC3333CCCC3333ull) | ((x & 0x0000CCCC0000CCCCull) << 14) | ((x >> 14) & 0x0000CCCC0000CCCCull);
    x = (x & 0xF0F0F0F00F0F0F0Full) | ((x & 0x00000000F0F0F0F0ull) << 28) | ((x >> 28) & 0x00000000F0F0F0F0ull);
    return x;
}

template <int D>
__device__ __forceinline__ void morton_deinterleave8(const uint32_t (&kw)[(D + 3) / 4], uint32_t (&pw)[(D + 3) / 4]) {
    constexpr int W = (D + 3) / 4;
#pragma unroll
    for (int k = 0; k < W; ++k) pw[k] = 0;
#pragma unroll
    for (int c = 0; c < (D + 7) / 8; ++c) {
        uint64_t m = 0;
#pragma unroll
        for (int L = 0; L < 8; ++L) {
            const int sh = D - 8 - 8 * c;
            const int pos = L * D + (sh >= 0 ? sh : 0);
            const int nb = sh >= 0 ? 8 : 8 + sh;  // bits of this level byte present in the key
            const int wd = pos >> 5, off = pos & 31;
            uint32_t v = kw[wd] >> off;
            if (off + nb > 32 && wd + 1 < W) v |= kw[wd + 1] << (32 - off);
            v &= (1u << nb) - 1u;
            if (sh < 0) v <<= -sh;
            m |= static_cast<uint64_t>(v) << (8 * L);
        }
        m = transpose8x8(m);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int d = 8 * c + r;
            if (d < D) pw[d >> 2] |= (static_cast<uint32_t>(m >> (8 * (7 - r))) & 0xffu) << (8 * (d & 3));
        }
    }
}

}  // namespace zi
