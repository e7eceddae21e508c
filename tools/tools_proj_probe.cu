// Dev probe: CUDA-core fp64 projection variants (P patches per thread, min blocks, prefetch
// distance) on a cfg2-shaped workload; checks every variant bit-identical to a naive chain.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ inline unsigned long long d2o(double x) {
    const unsigned long long b = __double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

template <int D>
__global__ void k_naive(const uint8_t* img, int w, int C, const uint32_t* keys, uint64_t n, const int32_t* off, int mc,
                        const double* mean, const double* comp, double* Y) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t key = keys[i];
    const uint8_t* pb = img + (size_t)((key >> 16) * (uint32_t)w + (key & 0xffffu)) * C;
    for (int d = 0; d < D; ++d) {
        double y = 0.0;
        for (int j = 0; j < mc; ++j) y = __fma_rn(comp[j * D + d], __dsub_rn((double)pb[off[j]], mean[j]), y);
        Y[(size_t)d * n + i] = y;
    }
}

// mcp = mc rounded up to PF; padded columns have comp 0, mean 0, offset 0 (exact no-ops)
template <int D, int P, int MINB, int PF, int T, int CV>
__global__ void __launch_bounds__(T, MINB) k_fma(const uint8_t* __restrict__ img, int w, int C,
                                                 const uint32_t* __restrict__ keys, uint64_t n,
                                                 const int32_t* __restrict__ off, int mc, const double* __restrict__ mean,
                                                 const double* __restrict__ comp, double* __restrict__ Y,
                                                 unsigned long long* __restrict__ minmax) {
    constexpr int Dp = (D + 1) & ~1;
    extern __shared__ double sm[];
    const int mcp = (mc + PF - 1) / PF * PF;
    double* s_comp = sm;
    double* s_mean = s_comp + (size_t)mcp * Dp;
    int* s_joff = reinterpret_cast<int*>(s_mean + mcp);
    for (int idx = threadIdx.x; idx < mcp * Dp; idx += T) {
        const int j = idx / Dp, d = idx % Dp;
        s_comp[idx] = (j < mc && d < D) ? comp[j * D + d] : 0.0;
    }
    for (int j = threadIdx.x; j < mcp; j += T) {
        s_mean[j] = j < mc ? mean[j] : 0.0;
        s_joff[j] = j < mc ? off[j] : 0;
    }
    __shared__ unsigned long long s_mm[2][D];
    if (threadIdx.x < 2 * D) s_mm[threadIdx.x / D][threadIdx.x % D] = threadIdx.x < D ? ~0ull : 0ull;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    constexpr uint64_t tile = (uint64_t)T * P;
    for (uint64_t base = blockIdx.x * tile; base < n; base += (uint64_t)gridDim.x * tile) {
        const uint8_t* pb[P];
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const uint64_t i = base + (uint64_t)p * T + threadIdx.x;
            const uint32_t key = keys[i < n ? i : n - 1];
            pb[p] = img + (size_t)((key >> 16) * (uint32_t)w + (key & 0xffffu)) * C;
        }
        double acc[P][D];
#pragma unroll
        for (int p = 0; p < P; ++p)
#pragma unroll
            for (int d = 0; d < D; ++d) acc[p][d] = 0.0;
        uint32_t xr[PF][P];
#pragma unroll
        for (int s = 0; s < PF; ++s) {
            const int o = s_joff[s];
#pragma unroll
            for (int p = 0; p < P; ++p) xr[s][p] = __ldg(pb[p] + o);
        }
        for (int j0 = 0; j0 < mcp; j0 += PF) {
            const bool more = j0 + PF < mcp;
#pragma unroll
            for (int s = 0; s < PF; ++s) {
                const int j = j0 + s;
                double a[P];
                const double mj = s_mean[j];
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    double xd;
                    if (CV == 0) xd = (double)xr[s][p];
                    else if (CV == 1) xd = __dsub_rn(__hiloint2double(0x43300000, (int)xr[s][p]), 4503599627370496.0);
                    else {
                        const float f = __uint_as_float(0x4B000000u | xr[s][p]) - 8388608.0f;
                        const unsigned hb = (__float_as_uint(f) >> 3) + 0x38000000u;
                        xd = __hiloint2double(xr[s][p] ? (int)hb : 0, 0);
                    }
                    a[p] = __dsub_rn(xd, mj);
                }
                if (more) {
                    const int o = s_joff[j + PF];
#pragma unroll
                    for (int p = 0; p < P; ++p) xr[s][p] = CV == 3 ? ((o + p * 77 + threadIdx.x * 5) & 255) : __ldg(pb[p] + o);
                }
                const double2* row = reinterpret_cast<const double2*>(s_comp + (size_t)j * Dp);
#pragma unroll
                for (int q = 0; q < Dp / 2; ++q) {
                    const double2 v = row[q];
#pragma unroll
                    for (int p = 0; p < P; ++p) {
                        acc[p][2 * q] = __fma_rn(v.x, a[p], acc[p][2 * q]);
                        if (2 * q + 1 < D) acc[p][2 * q + 1] = __fma_rn(v.y, a[p], acc[p][2 * q + 1]);
                    }
                }
            }
        }
#pragma unroll
        for (int d = 0; d < D; ++d) {
            unsigned long long lo = ~0ull, hi = 0ull;
#pragma unroll
            for (int p = 0; p < P; ++p) {
                const uint64_t i = base + (uint64_t)p * T + threadIdx.x;
                if (i < n) {
                    Y[(size_t)d * n + i] = acc[p][d];
                    const unsigned long long o = d2o(acc[p][d]);
                    lo = o < lo ? o : lo;
                    hi = o > hi ? o : hi;
                }
            }
#pragma unroll
            for (int s = 16; s > 0; s >>= 1) {
                const unsigned long long lo2 = __shfl_xor_sync(0xffffffffu, lo, s);
                const unsigned long long hi2 = __shfl_xor_sync(0xffffffffu, hi, s);
                lo = lo2 < lo ? lo2 : lo;
                hi = hi2 > hi ? hi2 : hi;
            }
            if (lane == 0) {
                atomicMin(&s_mm[0][d], lo);
                atomicMax(&s_mm[1][d], hi);
            }
        }
    }
    __syncthreads();
    if (threadIdx.x < D) {
        atomicMin(minmax + threadIdx.x, s_mm[0][threadIdx.x]);
        atomicMax(minmax + D + threadIdx.x, s_mm[1][threadIdx.x]);
    }
}

constexpr int D = 12;
struct Bufs { uint8_t* img; uint32_t* keys; int32_t* off; double *mean, *comp, *Y, *Yref; unsigned long long* mm; uint64_t n; int w, C, mc; };

template <int P, int MINB, int PF, int T, int GM, int CV = 0>
void run(const Bufs& b, int nsm) {
    const int mcp = (b.mc + PF - 1) / PF * PF;
    const size_t smem = (size_t)mcp * ((D + 1) & ~1) * 8 + (size_t)mcp * 12;
    cudaFuncSetAttribute(k_fma<D, P, MINB, PF, T, CV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const uint64_t tiles = (b.n + T * P - 1) / (T * P);
    const int grid = (int)std::min<uint64_t>(tiles, (uint64_t)nsm * GM);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9;
    for (int r = 0; r < 6; ++r) {
        cudaEventRecord(e0);
        k_fma<D, P, MINB, PF, T, CV><<<grid, T, smem>>>(b.img, b.w, b.C, b.keys, b.n, b.off, b.mc, b.mean, b.comp, b.Y, b.mm);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (r) best = ms < best ? ms : best;
    }
    cudaError_t e = cudaGetLastError();
    std::vector<double> y(b.n * D), yr(b.n * D);
    cudaMemcpy(y.data(), b.Y, y.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(yr.data(), b.Yref, yr.size() * 8, cudaMemcpyDeviceToHost);
    size_t diff = 0;
    for (size_t i = 0; i < y.size(); ++i) diff += y[i] != yr[i];
    const double flops = 2.0 * b.n * b.mc * D;
    printf("CV=%d P=%d minB=%d PF=%d T=%d grid=%d: %.4f ms  %.2f TFLOP/s useful  diff=%zu %s\n", CV, P, MINB, PF, T, grid, best,
           flops / best / 1e9, diff, cudaGetErrorString(e));
}

int main() {
    Bufs b;
    b.w = 1024; b.C = 3; const int H = 1024, K = 11; b.mc = K * K * b.C; b.n = 950771;
    std::vector<uint8_t> img((size_t)H * b.w * b.C);
    srand(1);
    for (auto& v : img) v = rand() & 255;
    std::vector<uint32_t> keys(b.n);
    for (uint64_t i = 0; i < b.n; ++i) { const uint32_t y = (uint32_t)(i / (b.w - K + 1)), x = (uint32_t)(i % (b.w - K + 1)); keys[i] = (y << 16) | x; }
    std::vector<int32_t> off(b.mc);
    for (int j = 0; j < b.mc; ++j) { const int p = j / b.C, c = j % b.C; off[j] = ((p / K) * b.w + p % K) * b.C + c; }
    std::vector<double> mean(b.mc), comp((size_t)b.mc * D);
    for (auto& v : mean) v = 100 + (rand() / (double)RAND_MAX) * 50;
    for (auto& v : comp) v = (rand() / (double)RAND_MAX - 0.5) * 0.2;
    cudaMalloc(&b.img, img.size()); cudaMemcpy(b.img, img.data(), img.size(), cudaMemcpyHostToDevice);
    cudaMalloc(&b.keys, b.n * 4); cudaMemcpy(b.keys, keys.data(), b.n * 4, cudaMemcpyHostToDevice);
    cudaMalloc(&b.off, b.mc * 4); cudaMemcpy(b.off, off.data(), b.mc * 4, cudaMemcpyHostToDevice);
    cudaMalloc(&b.mean, b.mc * 8); cudaMemcpy(b.mean, mean.data(), b.mc * 8, cudaMemcpyHostToDevice);
    cudaMalloc(&b.comp, comp.size() * 8); cudaMemcpy(b.comp, comp.data(), comp.size() * 8, cudaMemcpyHostToDevice);
    cudaMalloc(&b.Y, b.n * D * 8); cudaMalloc(&b.Yref, b.n * D * 8); cudaMalloc(&b.mm, 2 * D * 8);
    k_naive<D><<<(b.n + 255) / 256, 256>>>(b.img, b.w, b.C, b.keys, b.n, b.off, b.mc, b.mean, b.comp, b.Yref);
    cudaDeviceSynchronize();
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    run<2, 2, 4, 256, 2, 0>(b, nsm);
    run<2, 2, 4, 256, 2, 3>(b, nsm);
    run<4, 1, 8, 256, 1, 3>(b, nsm);
    return 0;
}
