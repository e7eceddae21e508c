// Dev probe: are mma.sync.m16n8k4/k8/k16.f64 bit-identical to sequential fma's in k order?
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int K>
__global__ void k(const double* A, const double* B, const double* C, double* Dm, double* Ds, int trials) {
    const int lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    for (int tr = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; tr < trials; tr += gridDim.x * (blockDim.x / 32)) {
        const double* a = A + tr * 16 * K;  // 16 x K row-major
        const double* b = B + tr * K * 8;   // K x 8 row-major
        const double* c = C + tr * 128;     // 16 x 8
        double d[4];
        // C/D fragment m16n8: d0,d1 = (row g, cols 2t, 2t+1); d2,d3 = (row g+8, ...)
        d[0] = c[g * 8 + 2 * t]; d[1] = c[g * 8 + 2 * t + 1];
        d[2] = c[(g + 8) * 8 + 2 * t]; d[3] = c[(g + 8) * 8 + 2 * t + 1];
        if (K == 4) {
            // A m16k4: a0 = (row g, col t), a1 = (row g+8, col t); B k4n8: b0 = (row t, col g)
            double a0 = a[g * K + t], a1 = a[(g + 8) * K + t], b0 = b[t * 8 + g];
            asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                         : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a0), "d"(a1), "d"(b0));
        } else if (K == 8) {
            // A m16k8: a0=(g,t) a1=(g+8,t) a2=(g,t+4) a3=(g+8,t+4); B k8n8: b0=(t,g) b1=(t+4,g)
            double a0 = a[g * K + t], a1 = a[(g + 8) * K + t], a2 = a[g * K + t + 4], a3 = a[(g + 8) * K + t + 4];
            double b0 = b[t * 8 + g], b1 = b[(t + 4) * 8 + g];
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
        } else {
            double av[8], bv[4];
            for (int q = 0; q < 4; ++q) { av[2 * q] = a[g * K + t + 4 * q]; av[2 * q + 1] = a[(g + 8) * K + t + 4 * q]; bv[q] = b[(t + 4 * q) * 8 + g]; }
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                         : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
                         : "d"(av[0]), "d"(av[1]), "d"(av[2]), "d"(av[3]), "d"(av[4]), "d"(av[5]), "d"(av[6]), "d"(av[7]),
                           "d"(bv[0]), "d"(bv[1]), "d"(bv[2]), "d"(bv[3]));
        }
        Dm[tr * 128 + g * 8 + 2 * t] = d[0]; Dm[tr * 128 + g * 8 + 2 * t + 1] = d[1];
        Dm[tr * 128 + (g + 8) * 8 + 2 * t] = d[2]; Dm[tr * 128 + (g + 8) * 8 + 2 * t + 1] = d[3];
        for (int e = lane; e < 128; e += 32) {
            const int r = e / 8, cc = e % 8;
            double acc = c[e];
            for (int kk = 0; kk < K; ++kk) acc = __fma_rn(a[r * K + kk], b[kk * 8 + cc], acc);
            Ds[tr * 128 + e] = acc;
        }
    }
}

template <int K>
void run() {
    const int trials = 1 << 14;
    double *A, *B, *C, *Dm, *Ds;
    cudaMallocManaged(&A, trials * 16 * K * 8); cudaMallocManaged(&B, trials * K * 8 * 8);
    cudaMallocManaged(&C, trials * 128 * 8); cudaMallocManaged(&Dm, trials * 128 * 8); cudaMallocManaged(&Ds, trials * 128 * 8);
    srand(K);
    auto rnd = [] { return (rand() / (double)RAND_MAX - 0.5) * (rand() % 2 ? 1e3 : 1e-2); };
    for (int i = 0; i < trials * 16 * K; ++i) A[i] = (rand() % 256) - 127.3 + rnd() * 1e-3;
    for (int i = 0; i < trials * K * 8; ++i) B[i] = rnd();
    for (int i = 0; i < trials * 128; ++i) C[i] = rnd() * 100;
    k<K><<<128, 256>>>(A, B, C, Dm, Ds, trials);
    cudaError_t e = cudaDeviceSynchronize();
    long diff = 0;
    for (int i = 0; i < trials * 128; ++i) if (Dm[i] != Ds[i]) ++diff;
    printf("m16n8k%d: %s, elements %d, mma != sequential fma: %ld\n", K, cudaGetErrorString(e), trials * 128, diff);
}

int main() { run<4>(); run<8>(); run<16>(); return 0; }
