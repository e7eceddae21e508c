// tc_ptx.cuh -- tcgen05 / TMEM / TMA / mbarrier primitives shared by the 5th-generation
// tensor-core kernels (k_tc.cu: patch moments; k_proj_tc.cu: projection filter).
#pragma once
#include <cuda.h>

#include <cstdint>

namespace zi {

__device__ __forceinline__ uint32_t tc_smem(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void tc_mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void tc_mbar_expect(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// the suspend-time hint lets a waiting thread sleep in hardware until the phase completes (or the
// limit passes) instead of re-issuing try_wait: a polling MMA lane or gather warp otherwise takes
// issue slots from the epilogue warps (15 % of the min / max pass's executed instructions)
#ifndef ZI_MBAR_HINT_NS
#define ZI_MBAR_HINT_NS 20000u
#endif
__device__ __forceinline__ void tc_mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "TC_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra TC_WAIT_%=;\n}" ::"r"(bar),
        "r"(parity), "r"(ZI_MBAR_HINT_NS)
        : "memory");
}
__device__ __forceinline__ void tc_tma_load_2d(uint32_t dst, const CUtensorMap* tm, int x, int y, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(bar)
        : "memory");
}
// UMMA shared-memory matrix descriptor: K-major, 128B swizzle (8-row x 128 B atoms, atoms 1024 B
// apart), sm_100 version 1
__device__ __forceinline__ uint64_t tc_desc_k128(uint32_t saddr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3fffu);   // start address
    d |= static_cast<uint64_t>(1u) << 16;                 // leading byte offset (unused for swizzled K-major)
    d |= static_cast<uint64_t>(1024u >> 4) << 32;         // stride byte offset: next 8-row group
    d |= static_cast<uint64_t>(1u) << 46;                 // descriptor version (sm_100)
    d |= static_cast<uint64_t>(2u) << 61;                 // SWIZZLE_128B
    return d;
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// 4 consecutive TMEM columns of this warp's 32 lanes (one register per column)
__device__ __forceinline__ void tc_ld_x4(uint32_t taddr, uint32_t (&v)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "r"(taddr));
}
__device__ __forceinline__ void tc_ld_x1(uint32_t taddr, uint32_t& v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(taddr));
}
__device__ __forceinline__ void tc_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

}  // namespace zi
