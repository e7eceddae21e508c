// Dev probe: is mma.sync.m8n8k4.f64 bit-identical to four sequential fma's in k order?
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void k(const double* A, const double* B, const double* C, double* Dm, double* Ds, int trials) {
    const int lane = threadIdx.x & 31;
    for (int t = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; t < trials; t += gridDim.x * (blockDim.x / 32)) {
        const double* a = A + t * 32;  // 8x4 row-major
        const double* b = B + t * 32;  // 4x8 (k x n) row-major
        const double* c = C + t * 64;  // 8x8
        // fragment layout m8n8k4 f64: a: row = lane/4, col = lane%4; b: row(k) = lane%4, col = lane/4;
        // c/d: row = lane/4, cols 2*(lane%4) + {0,1}
        double fa = a[(lane / 4) * 4 + lane % 4];
        double fb = b[(lane % 4) * 8 + lane / 4];
        double c0 = c[(lane / 4) * 8 + 2 * (lane % 4)], c1 = c[(lane / 4) * 8 + 2 * (lane % 4) + 1];
        double d0, d1;
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
                     : "=d"(d0), "=d"(d1)
                     : "d"(fa), "d"(fb), "d"(c0), "d"(c1));
        Dm[t * 64 + (lane / 4) * 8 + 2 * (lane % 4)] = d0;
        Dm[t * 64 + (lane / 4) * 8 + 2 * (lane % 4) + 1] = d1;
        for (int e = lane; e < 64; e += 32) {
            const int r = e / 8, cc = e % 8;
            double acc = c[e];
            for (int kk = 0; kk < 4; ++kk) acc = __fma_rn(a[r * 4 + kk], b[kk * 8 + cc], acc);
            Ds[t * 64 + e] = acc;
        }
    }
}

int main() {
    const int trials = 1 << 16;
    double *A, *B, *C, *Dm, *Ds;
    cudaMallocManaged(&A, trials * 32 * 8);
    cudaMallocManaged(&B, trials * 32 * 8);
    cudaMallocManaged(&C, trials * 64 * 8);
    cudaMallocManaged(&Dm, trials * 64 * 8);
    cudaMallocManaged(&Ds, trials * 64 * 8);
    srand(1);
    auto rnd = [] { return (rand() / (double)RAND_MAX - 0.5) * (rand() % 2 ? 1e3 : 1e-2); };
    for (int i = 0; i < trials * 32; ++i) { A[i] = (rand() % 256) - 127.3 + rnd() * 1e-3; B[i] = rnd(); }
    for (int i = 0; i < trials * 64; ++i) C[i] = rnd() * 100;
    k<<<256, 256>>>(A, B, C, Dm, Ds, trials);
    cudaDeviceSynchronize();
    long diff = 0, diff_alt = 0;
    for (int i = 0; i < trials * 64; ++i) if (Dm[i] != Ds[i]) ++diff;
    // alternative: exact 4-term sum then one rounding with C (compare via long double)
    for (int t = 0; t < 1024; ++t)
        for (int e = 0; e < 64; ++e) {
            const int r = e / 8, cc = e % 8;
            long double s = C[t * 64 + e];
            for (int kk = 0; kk < 4; ++kk) s += (long double)A[t * 32 + r * 4 + kk] * B[t * 32 + kk * 8 + cc];
            if ((double)s != Dm[t * 64 + e]) ++diff_alt;
        }
    printf("elements %d  mma!=seqfma %ld  mma!=onerounding(longdouble,1024 trials) %ld\n", trials * 64, diff, diff_alt);
    return 0;
}
