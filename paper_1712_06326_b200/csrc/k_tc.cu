// k_tc.cu -- 5th-generation tensor-core (tcgen05 + TMEM + TMA) kernels.
//
// K2b' patch moments, tcgen05 path: the exact integer Gram X^T X of the u8 patch matrix (and,
// through an all-ones feature row, the first moments) -- the same numbers k_moments computes
// with mma.sync, restating proj/src/pca.cpp:20-37 (mean + covariance accumulation) in exact
// integers.  XT is the feature-major patch matrix [Fpad][npad] written by k_patch_matrix; row F
// is all ones over the real patches, so G[f][F] = sum_i x_f(i).
//
// One CTA = one 128x128 feature tile pair (ti <= tj) x one patch chunk (<= 65536 patches, so the
// s32 accumulators read as u32 are exact: 65536 * 255^2 < 2^32).  Warp 0 (one lane) streams
// 128-patch stages of both tiles with TMA (2D tensor map, 128B swizzle) into a 6-stage ring;
// warp 1 (one lane) issues tcgen05.mma.kind::i8 (M = N = 128, K = 32, u8 x u8 -> s32) into a
// 128-column TMEM accumulator and frees each stage with tcgen05.commit; after the last stage all
// four warps read TMEM (tcgen05.ld 32x32b: warp w owns rows 32w..32w+31) and fold the chunk into
// the int64 moments with atomics (order-free -> deterministic).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "tc_ptx.cuh"
#include "zi_internal.h"

namespace zi {

constexpr int kTcTile = 128;            // feature rows per tile (UMMA M = N)
constexpr int kTcStageK = 128;          // patches per stage (128 B rows: one swizzle atom wide)
constexpr int kTcStages = 6;
constexpr int kTcTileBytes = kTcTile * kTcStageK;  // 16 KB
constexpr uint64_t kTcMaxChunk = 65536;

// instruction descriptor: kind::i8, u8 x u8 -> s32, both K-major, M = N = 128
constexpr uint32_t kTcIdesc = (2u << 4)                  // D format S32
                              | (0u << 7) | (0u << 10)   // A, B unsigned 8-bit
                              | (static_cast<uint32_t>(kTcTile >> 3) << 17)  // N >> 3
                              | (static_cast<uint32_t>(kTcTile >> 4) << 24); // M >> 4

__device__ __forceinline__ void tc_mma_i8(uint32_t tmem, uint64_t da, uint64_t db, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
        "l"(da), "l"(db), "r"(kTcIdesc), "r"(accumulate)
        : "memory");
}
__global__ void __launch_bounds__(128, 1) k_gram_tc(const __grid_constant__ CUtensorMap tm, int F, int ntile,
                                                    uint64_t npad, uint64_t chunk, unsigned long long* __restrict__ out) {
    extern __shared__ uint8_t tc_raw[];
    uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tc_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    __shared__ __align__(8) uint64_t s_full[kTcStages], s_empty[kTcStages], s_done;
    __shared__ uint32_t s_tmem;
    int pr = blockIdx.x, ti = 0;
    while (pr >= ntile - ti) {
        pr -= ntile - ti;
        ++ti;
    }
    const int tj = ti + pr;
    const bool diag = ti == tj;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t c0 = static_cast<uint64_t>(blockIdx.y) * chunk;
    const uint64_t c1 = c0 + chunk < npad ? c0 + chunk : npad;
    const int nst = static_cast<int>((c1 - c0 + kTcStageK - 1) / kTcStageK);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc_smem(&s_tmem)),
                     "r"(static_cast<uint32_t>(kTcTile))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int s = 0; s < kTcStages; ++s) {
            tc_mbar_init(tc_smem(&s_full[s]), 1);
            tc_mbar_init(tc_smem(&s_empty[s]), 1);
        }
        tc_mbar_init(tc_smem(&s_done), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    const uint32_t stage_bytes = diag ? kTcTileBytes : 2 * kTcTileBytes;
    if (warp == 0 && lane == 0) {  // TMA producer
        for (int st = 0; st < nst; ++st) {
            const int s = st % kTcStages;
            if (st >= kTcStages) tc_mbar_wait(tc_smem(&s_empty[s]), ((st / kTcStages) + 1) & 1);
            const uint32_t full = tc_smem(&s_full[s]);
            tc_mbar_expect(full, stage_bytes);
            const uint32_t a = tc_smem(ring + static_cast<size_t>(s) * 2 * kTcTileBytes);
            const int x = static_cast<int>(c0 + static_cast<uint64_t>(st) * kTcStageK);
            tc_tma_load_2d(a, &tm, x, ti * kTcTile, full);
            if (!diag) tc_tma_load_2d(a + kTcTileBytes, &tm, x, tj * kTcTile, full);
        }
    } else if (warp == 1 && lane == 0) {  // MMA issuer
        for (int st = 0; st < nst; ++st) {
            const int s = st % kTcStages;
            tc_mbar_wait(tc_smem(&s_full[s]), (st / kTcStages) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t a = tc_smem(ring + static_cast<size_t>(s) * 2 * kTcTileBytes);
            const uint64_t da = tc_desc_k128(a), db = tc_desc_k128(diag ? a : a + kTcTileBytes);
#pragma unroll
            for (int k = 0; k < kTcStageK / 32; ++k)  // K = 32 bytes per MMA: +2 in the 16-byte address units
                tc_mma_i8(tmem, da + 2 * k, db + 2 * k, (st | k) != 0 ? 1u : 0u);
            tc_commit(tc_smem(&s_empty[s]));
        }
        tc_commit(tc_smem(&s_done));
    }
    __syncwarp();
    tc_mbar_wait(tc_smem(&s_done), 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // epilogue: row fi = ti*128 + 32w + lane; 32 columns per tcgen05.ld
    const int fi = ti * kTcTile + warp * 32 + lane;
#pragma unroll 1
    for (int cb = 0; cb < kTcTile; cb += 32) {
        uint32_t v[32];
        const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>(cb);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (fi < F) {
#pragma unroll
            for (int q = 0; q < 32; ++q) {
                const int fj = tj * kTcTile + cb + q;
                if (v[q] == 0u) continue;
                if (fj < F) atomicAdd(out + F + static_cast<size_t>(fi) * F + fj, static_cast<unsigned long long>(v[q]));
                else if (fj == F) atomicAdd(out + fi, static_cast<unsigned long long>(v[q]));
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(static_cast<uint32_t>(kTcTile))
                     : "memory");
}

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        ZI_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) throw error(ZI_E_CUDA, "cuTensorMapEncodeTiled unavailable");
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

// out[0..F) += row sums, out[F + fi*F + fj] += Gram (upper tile pairs, full diagonal tiles), from
// XT [Fpad][npad] (Fpad % 128 == 0, Fpad > F, row F all ones, npad % 128 == 0).  Output zeroed by
// the caller.
void gram_u8_tc(zi_ctx* ctx, const uint8_t* XT, int F, int Fpad, uint64_t npad, unsigned long long* out) {
    CUtensorMap tm;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(npad), static_cast<cuuint64_t>(Fpad)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(npad)};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(kTcStageK), static_cast<cuuint32_t>(kTcTile)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = tensor_map_encoder()(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(XT), dims, strides,
                                            box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw error(ZI_E_CUDA, "cuTensorMapEncodeTiled failed");
    const int ntile = Fpad / kTcTile;
    const int npairs = ntile * (ntile + 1) / 2;
    // about one CTA per SM: split the patches into chunks of <= 65536 (a multiple of the stage)
    const uint64_t want = std::max<uint64_t>(1, static_cast<uint64_t>(ctx->num_sms) / npairs);
    uint64_t chunk = (npad + want - 1) / want;
    chunk = std::min<uint64_t>(kTcMaxChunk, (chunk + kTcStageK - 1) / kTcStageK * kTcStageK);
    const uint64_t nchunk = (npad + chunk - 1) / chunk;
    const size_t smem = static_cast<size_t>(kTcStages) * 2 * kTcTileBytes + 1024;
    smem_attr(ctx->device, k_gram_tc, smem);
    ZI_LAUNCH(ctx, "patch_moments", k_gram_tc, dim3(npairs, static_cast<unsigned>(nchunk)), 128, smem, tm, F, ntile, npad,
              chunk, out);
}

}  // namespace zi
