// dev probe: does tcgen05.mma.kind::i8 accept MN-major (transposed) shared-memory operands, and with
// which descriptor strides?  A 128-patch x 128-feature u8 tile stored K-major by features (rows =
// patches, 128B swizzle, as the projection kernel's A tiles) is used as BOTH operands of X^T X
// (M = N = 128 features, K = 128 patches) through the transpose bits; result vs the host Gram.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda.h>
#include "../paper_1712_06326_b200/csrc/tc_ptx.cuh"

using namespace zi;

__device__ __forceinline__ uint64_t desc_mn(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3fffu);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3fffu) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3fffu) << 32;
    d |= static_cast<uint64_t>(1u) << 46;
    d |= static_cast<uint64_t>(2u) << 61;  // SWIZZLE_128B
    return d;
}

__global__ void k_probe(const uint8_t* X /* 128 rows(patches) x 128 cols(features) */, uint32_t lbo, uint32_t sbo,
                        int kstep_bytes, uint32_t* out /* 128 x 128 */) {
    __shared__ __align__(1024) uint8_t sA[128 * 128];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t s_tmem;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // K-major SW128 store: row r, 16-byte chunk c at (r/8)*1024 + (r%8)*128 + ((c ^ r%8) << 4)
    for (int i = tid; i < 128 * 8; i += blockDim.x) {
        const int r = i / 8, c = i % 8;
        const uint4 v = *reinterpret_cast<const uint4*>(X + r * 128 + c * 16);
        *reinterpret_cast<uint4*>(sA + (r / 8) * 1024 + (r % 8) * 128 + ((c ^ (r % 8)) << 4)) = v;
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc_smem(&s_tmem)), "r"(128u) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        tc_mbar_init(tc_smem(&bar), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;
    if (tid == 0) {
        const uint32_t idesc = (2u << 4) | (0u << 7) | (0u << 10) | (1u << 15) | (1u << 16) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
        const uint32_t base = tc_smem(sA);
        for (int ks = 0; ks < 4; ++ks) {
            const uint64_t d = desc_mn(base + ks * kstep_bytes, lbo, sbo);
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem), "l"(d), "l"(d), "r"(idesc), "r"(ks)
                : "memory");
        }
        tc_commit(tc_smem(&bar));
    }
    __syncwarp();
    tc_mbar_wait(tc_smem(&bar), 0);
    tc_fence_after();
    for (int cb = 0; cb < 128; cb += 4) {
        uint32_t v[4];
        tc_ld_x4(tmem + (static_cast<uint32_t>(warp * 32) << 16) + cb, v);
        tc_ld_wait();
        for (int q = 0; q < 4; ++q) out[(warp * 32 + lane) * 128 + cb + q] = v[q];
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128u) : "memory");
}

int main() {
    std::vector<uint8_t> X(128 * 128);
    uint32_t seed = 12345;
    for (auto& x : X) { seed = seed * 1664525u + 1013904223u; x = static_cast<uint8_t>(seed >> 24); }
    std::vector<uint32_t> ref(128 * 128, 0);
    for (int i = 0; i < 128; ++i)
        for (int j = 0; j < 128; ++j) {
            uint32_t s = 0;
            for (int p = 0; p < 128; ++p) s += static_cast<uint32_t>(X[p * 128 + i]) * X[p * 128 + j];
            ref[i * 128 + j] = s;
        }
    uint8_t* dX; uint32_t* dO;
    cudaMalloc(&dX, X.size()); cudaMalloc(&dO, 128 * 128 * 4);
    cudaMemcpy(dX, X.data(), X.size(), cudaMemcpyHostToDevice);
    const uint32_t lbos[] = {16, 128, 1024, 2048, 4096, 8192};
    const uint32_t sbos[] = {16, 128, 1024, 2048, 4096, 8192};
    const int ksteps[] = {4096, 32};
    for (int ksb : ksteps)
        for (uint32_t lbo : lbos)
            for (uint32_t sbo : sbos) {
                cudaMemset(dO, 0, 128 * 128 * 4);
                k_probe<<<1, 128>>>(dX, lbo, sbo, ksb, dO);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("kstep %d lbo %u sbo %u: %s\n", ksb, lbo, sbo, cudaGetErrorString(e)); return 1; }
                std::vector<uint32_t> o(128 * 128);
                cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost);
                int bad = 0;
                for (int i = 0; i < 128 * 128; ++i) bad += o[i] != ref[i];
                printf("kstep %5d lbo %5u sbo %5u: mismatches %d%s\n", ksb, lbo, sbo, bad, bad == 0 ? "   <== MATCH" : "");
            }
    return 0;
}
