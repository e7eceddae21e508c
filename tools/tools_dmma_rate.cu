// Dev probe: FP64 MMA pipe throughput per shape (flop/s with 4 independent accumulators per warp).
#include <cstdio>
#include <cuda_runtime.h>
template <int S>
__global__ void k(double* out, int iters) {
    double a[8], b[4], d[4][4];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
    for (int i = 0; i < 4; ++i) b[i] = 1.0 + i * 1e-9;
    for (int j = 0; j < 4; ++j) for (int i = 0; i < 4; ++i) d[j][i] = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (S == 0)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d[j][0]), "+d"(d[j][1]) : "d"(a[0]), "d"(b[0]));
            else if (S == 1)
                asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};" : "+d"(d[j][0]), "+d"(d[j][1]), "+d"(d[j][2]), "+d"(d[j][3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
            else if (S == 2)
                asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};" : "+d"(d[j][0]), "+d"(d[j][1]), "+d"(d[j][2]), "+d"(d[j][3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
            else
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};" : "+d"(d[j][0]), "+d"(d[j][1]), "+d"(d[j][2]), "+d"(d[j][3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
        }
    }
    double s = 0;
    for (int j = 0; j < 4; ++j) for (int i = 0; i < 4; ++i) s += d[j][i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int S>
void run(const char* name, double flop_per_mma) {
    double* o; cudaMalloc(&o, 148 * 8 * 1024 * 8);
    int iters = 4096;
    for (int warps : {4, 8, 16}) {
        k<S><<<148 * 2, warps * 32>>>(o, 16);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k<S><<<148 * 2, warps * 32>>>(o, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double fl = 148.0 * 2 * warps * iters * 4 * flop_per_mma;
        printf("%-10s warps/CTA %2d: %.2f TFLOP/s\n", name, warps, fl / ms / 1e9);
    }
}
int main() {
    run<0>("m8n8k4", 2.0 * 8 * 8 * 4);
    run<1>("m16n8k4", 2.0 * 16 * 8 * 4);
    run<2>("m16n8k8", 2.0 * 16 * 8 * 8);
    run<3>("m16n8k16", 2.0 * 16 * 8 * 16);
    return 0;
}
