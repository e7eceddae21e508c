// Dev probe: DFMA vs DMMA throughput, alone and concurrently (do they share the FP64 datapath?).
#include <cstdio>
#include <cuda_runtime.h>
// mode 0: all warps DMMA; 1: all warps DFMA; 2: even warps DMMA, odd warps DFMA
__global__ void k(double* out, int iters, int mode) {
    const int warp = threadIdx.x >> 5;
    const bool mma = mode == 0 || (mode == 2 && (warp & 1) == 0);
    double a = threadIdx.x * 1e-3, b = 1.0 + 1e-9;
    double d[8][2];
    for (int j = 0; j < 8; ++j) d[j][0] = d[j][1] = j;
    if (mma) {
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int j = 0; j < 8; ++j)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d[j][0]), "+d"(d[j][1]) : "d"(a), "d"(b));
    } else {
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // 16 DFMA per 8 "mma slots" (same flops as... see host)
                asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(d[j][0]) : "d"(a), "d"(b));
                asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(d[j][1]) : "d"(a), "d"(b));
            }
    }
    double s = 0;
    for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    double* o; cudaMalloc(&o, 148 * 4 * 1024 * 8);
    const int iters = 8192, warps = 16, blocks = 148 * 2;
    for (int mode = 0; mode < 3; ++mode) {
        k<<<blocks, warps * 32>>>(o, 16, mode);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k<<<blocks, warps * 32>>>(o, iters, mode);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double mma_warps = mode == 0 ? warps : mode == 2 ? warps / 2 : 0;
        const double fma_warps = warps - mma_warps;
        const double fl_mma = (double)blocks * mma_warps * iters * 8 * 512;
        const double fl_fma = (double)blocks * fma_warps * iters * 16 * 64;
        printf("mode %d: %.3f ms  dmma %.2f TF  dfma %.2f TF  total %.2f TF\n", mode, ms, fl_mma / ms / 1e9, fl_fma / ms / 1e9,
               (fl_mma + fl_fma) / ms / 1e9);
    }
    return 0;
}
