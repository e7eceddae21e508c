// Dev probe: DFMA rate with the projection's operand pattern (12 comp values x P a-values x
// 12P accumulators) vs reused operands; and with the I2F + DADD per a-value.
#include <cstdio>
#include <cuda_runtime.h>
template <int P, int MODE>
__global__ void k(double* out, const double* src, int iters) {
    double c[12], a[P], acc[P][12];
    for (int d = 0; d < 12; ++d) c[d] = src[d] + threadIdx.x;
    for (int p = 0; p < P; ++p) { a[p] = src[12 + p]; for (int d = 0; d < 12; ++d) acc[p][d] = d; }
    unsigned x = threadIdx.x;
    for (int it = 0; it < iters; ++it) {
        if (MODE == 1) {  // new a per column: I2F + DADD
#pragma unroll
            for (int p = 0; p < P; ++p) { x = x * 1664525u + 1013904223u; a[p] = __dsub_rn((double)(x >> 24), c[p]); }
        }
        if (MODE == 2) {  // new c per column (rotate)
#pragma unroll
            for (int d = 0; d < 12; ++d) c[d] = __shfl_xor_sync(0xffffffffu, c[d], 1);
        }
#pragma unroll
        for (int p = 0; p < P; ++p)
#pragma unroll
            for (int d = 0; d < 12; ++d) acc[p][d] = __fma_rn(c[d], a[p], acc[p][d]);
    }
    double s = 0;
    for (int p = 0; p < P; ++p) for (int d = 0; d < 12; ++d) s += acc[p][d];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int P, int MODE>
void run(double* o, double* src) {
    const int iters = 4096, T = 256, B = 148 * 2;
    k<P, MODE><<<B, T>>>(o, src, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<P, MODE><<<B, T>>>(o, src, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("P=%d mode=%d: %.2f TFLOP/s (useful DFMA)\n", P, MODE, 2.0 * B * T * iters * P * 12 / ms / 1e9);
}
int main() {
    double *o, *src; cudaMalloc(&o, 148 * 2 * 256 * 8); cudaMalloc(&src, 64 * 8); cudaMemset(src, 0, 64 * 8);
    run<1, 0>(o, src); run<2, 0>(o, src); run<4, 0>(o, src);
    run<1, 1>(o, src); run<2, 1>(o, src); run<4, 1>(o, src);
    run<2, 2>(o, src);
    return 0;
}
