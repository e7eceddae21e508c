// shard.cu -- one rank's part of a range-partitioned multi_index.
//
// The reference builds every layout index on one host (multi_index::build,
// proj/src/builder.cpp:202-224; zcurve_index::from_descriptors, proj/src/zcurve.cpp:108-138).
// Across G GPUs the dictionary rows are split into G contiguous slices (shard_ranges) and the
// build runs as stages separated by collectives that the host layer (sharding.py, over
// torch.distributed / NCCL) performs between the calls below:
//
//   moments      exact int64 partial Gram of the rank's rows            -> all-reduce SUM
//                (integer sums: the total is bit-identical for any G)
//   fit_project  8 PCA models from the global moments (identical on every rank, same device
//                code as the single-GPU build) and the min / max pass of the tensor-core
//                projection (k_proj_tc.cu) over the rank's rows: partial approximate ranges as
//                order-preserving int64                                  -> all-reduce MIN / MAX
//   refine       the quantise pass with the global approximate ranges (records of every pair
//                the bracket decides; candidates and ambiguous pairs listed), exact lo / hi over
//                the rank's candidates                                   -> all-reduce MIN / MAX
//                (configurations outside the tensor-core envelope project in fp64 at
//                fit_project, return exact ranges there and pass them through here)
//   quantize     global exact lo/hi -> the listed pairs' exact records (payload = global row),
//                local hybrid sort, regular samples                      -> all-gather samples
//   partition    splitters (zi_shard_splitters) -> lower bounds in the local sorted layouts,
//                send buffer packed destination-major                    -> all-gather counts,
//                                                                           all-to-all records
//   receive      unpack, sort (the received runs come in row order, so the stable sort keeps
//                the reference's tie order), then the rebalancing plan that gives rank r
//                exactly global positions shard_ranges(n, G)[r] of every layout
//                                                                        -> all-to-all records
//   finish       unpack in (layout, source) order -- already sorted -- and finalise the 8
//                index shards (planes, keys, bbox)
//
// Result: rank r's layout-l index = positions [B_r, E_r) of the single-GPU layout-l index,
// byte for byte, so the shards' concatenation is the reference's global order and every shard
// of every layout has the same size (= the rank's dictionary slice).
#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"

struct zi_shard {
    zi_multi_index* mi = nullptr;  // image, global dictionary, models; after finish the 8 shards
    int rank = 0, world = 1;
    uint64_t n_total = 0, row_b = 0, row_e = 0;
    int D = 0, W = 0;
    int stage = 0;                  // 0 created, 1 moments, 2 fit, 3 quantized, 4 partitioned, 5 received, 6 done
    zi::dbuf<double> Y;             // 8 x D x n_r projections
    zi::dbuf<uint32_t> send;        // AoS records, (W+1) words each
    zi::dbuf<uint64_t> pos;         // lower bounds of the splitters
    zi::dbuf<uint32_t> small;       // splitters / samples / segment tables
    uint64_t held = 0;              // records held after the first exchange
    bool tc = false;                // projection on the int8 tensor cores (k_proj_tc.cu)
    bool refined = false;           // refine_ranges ran after fit_project
    uint32_t* sorted[10] = {};      // the locally sorted records (word k at sorted[k], stride 8n)
};

namespace zi {

namespace {

constexpr uint32_t kSentinel = 0xffffffffu;  // "no sample" / +infinity splitter payload
constexpr int kMaxSegs = 1024;

struct seg_t {
    unsigned long long src, dst, len;
};

// record e of a SoA record array (W key words of stride N, payload at word W) < the AoS row s
__device__ __forceinline__ bool rec_less_row(const uint32_t* __restrict__ recs, uint64_t N, int W, uint64_t e,
                                             const uint32_t* s) {
    for (int k = W - 1; k >= 0; --k) {
        const uint32_t a = recs[static_cast<size_t>(k) * N + e], b = s[k];
        if (a != b) return a < b;
    }
    return recs[static_cast<size_t>(W) * N + e] < s[W];
}

// lower bound of every splitter inside its layout's sorted segment [l*seg, (l+1)*seg)
__global__ void k_shard_bounds(const uint32_t* __restrict__ recs, uint64_t N, int W, uint64_t seg,
                               const uint32_t* __restrict__ spl, int per_layout, unsigned long long* __restrict__ out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 8 * per_layout) return;
    const int l = t / per_layout;
    const uint32_t* s = spl + static_cast<size_t>(t) * (W + 1);
    uint64_t lo = static_cast<uint64_t>(l) * seg, hi = lo + seg;
    if (s[W] == kSentinel) {
        out[t] = seg;
        return;
    }
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (rec_less_row(recs, N, W, mid, s)) lo = mid + 1;
        else hi = mid;
    }
    out[t] = lo - static_cast<uint64_t>(l) * seg;
}

// S regular samples of every layout's sorted segment, AoS rows of W+1 words
__global__ void k_shard_samples(const uint32_t* __restrict__ recs, uint64_t N, int W, uint64_t seg, int S,
                                uint32_t* __restrict__ out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 8 * S) return;
    const int l = t / S, j = t % S;
    uint32_t* o = out + static_cast<size_t>(t) * (W + 1);
    if (seg == 0) {
        for (int k = 0; k <= W; ++k) o[k] = kSentinel;
        return;
    }
    const uint64_t e = static_cast<uint64_t>(l) * seg + (static_cast<uint64_t>(2 * j + 1) * seg) / (2ull * S);
    for (int k = 0; k <= W; ++k) o[k] = recs[static_cast<size_t>(k) * N + e];
}

// Record moves by a segment table (segments sorted by dst and tiling [0, total)).  A stride of 0
// means AoS (W1 consecutive words per record), otherwise SoA with that word stride.
__global__ void __launch_bounds__(256) k_seg_move(const uint32_t* __restrict__ in, uint64_t in_stride,
                                                  uint32_t* __restrict__ out, uint64_t out_stride, int W1,
                                                  const seg_t* __restrict__ segs, int nseg, uint64_t total) {
    __shared__ unsigned long long s_dst[kMaxSegs];
    for (int i = threadIdx.x; i < nseg; i += blockDim.x) s_dst[i] = segs[i].dst;
    __syncthreads();
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t o = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; o < total; o += stride) {
        int lo = 0, hi = nseg - 1;  // last segment with dst <= o
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s_dst[mid] <= o) lo = mid;
            else hi = mid - 1;
        }
        const uint64_t e = segs[lo].src + (o - s_dst[lo]);
        for (int k = 0; k < W1; ++k) {
            const uint32_t v = in_stride ? in[static_cast<size_t>(k) * in_stride + e] : in[e * W1 + k];
            if (out_stride) out[static_cast<size_t>(k) * out_stride + o] = v;
            else out[o * W1 + k] = v;
        }
    }
}

// host composite order: layout, Morton words (most significant last), payload
bool host_rec_less(const uint32_t* a, const uint32_t* b, int W) {
    const uint32_t la = a[W] >> 29, lb = b[W] >> 29;
    if (la != lb) return la < lb;
    for (int k = W - 1; k >= 0; --k)
        if (a[k] != b[k]) return a[k] < b[k];
    return a[W] < b[W];
}

void move_segments(zi_shard* sh, const uint32_t* in, uint64_t in_stride, uint32_t* out, uint64_t out_stride,
                   std::vector<seg_t> segs, uint64_t total) {
    zi_ctx* ctx = sh->mi->ctx;
    if (total == 0) return;
    // drop empty segments (the kernel's search needs strictly covering entries)
    segs.erase(std::remove_if(segs.begin(), segs.end(), [](const seg_t& s) { return s.len == 0; }), segs.end());
    std::sort(segs.begin(), segs.end(), [](const seg_t& a, const seg_t& b) { return a.dst < b.dst; });
    if (segs.empty() || segs.size() > static_cast<size_t>(kMaxSegs)) throw error(ZI_E_INVALID, "shard: bad segment table");
    const size_t words = (segs.size() * sizeof(seg_t) + 3) / 4;
    uint32_t* d = sh->small.ensure(words);
    ZI_CUDA(cudaMemcpyAsync(d, segs.data(), segs.size() * sizeof(seg_t), cudaMemcpyHostToDevice, ctx->stream));
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((total + 255) / 256, static_cast<uint64_t>(ctx->num_sms) * 8));
    ZI_LAUNCH(ctx, "shard_move", k_seg_move, grid, 256, 0, in, in_stride, out, out_stride, sh->W + 1,
              reinterpret_cast<const seg_t*>(d), static_cast<int>(segs.size()), total);
    ZI_CUDA(cudaStreamSynchronize(ctx->stream));  // segs is a host local
}

}  // namespace

void shard_ranges(uint64_t n, int world, int r, uint64_t* b, uint64_t* e) {
    const uint64_t base = n / world, extra = n % world;
    const uint64_t rr = static_cast<uint64_t>(r);
    *b = rr * base + std::min<uint64_t>(rr, extra);
    *e = *b + base + (rr < extra ? 1 : 0);
}

// (re)start the stage machine: the dictionary from the device-resident mask, this rank's rows
static void shard_start(zi_shard* sh) {
    zi_multi_index* mi = sh->mi;
    const int rank = sh->rank, world = sh->world;
    mi->n_total = collect_dictionary(mi->ctx, mi->known.p, mi->w, mi->h, mi->K, mi->dict);
    if (mi->n_total == 0) throw error(ZI_E_EMPTY_DICT, "no fully known patch window; inpainting impossible");
    if (mi->n_total >= (1ull << 29) - 1) throw error(ZI_E_INVALID, "dictionary above 2^29 patches");
    sh->n_total = mi->n_total;
    shard_ranges(sh->n_total, world, rank, &sh->row_b, &sh->row_e);
    mi->row_begin = sh->row_b;
    mi->n = sh->row_e - sh->row_b;
    mi->dims = static_cast<int>(std::min<uint64_t>(static_cast<uint64_t>(mi->cfg.dims),
                                                   std::min<uint64_t>(static_cast<uint64_t>(mi->mc), sh->n_total)));
    mi->F = mi->K * mi->K * mi->C;
    sh->D = mi->dims;
    sh->W = (sh->D + 3) / 4;
    sh->stage = 0;
    sh->held = 0;
    sh->refined = false;
}

zi_shard* shard_create(zi_multi_index* mi, int rank, int world) {
    auto* sh = new zi_shard();
    sh->mi = mi;
    sh->rank = rank;
    sh->world = world;
    mi->shard = true;
    try {
        shard_start(sh);
    } catch (...) {
        delete sh;
        throw;
    }
    return sh;
}

// the next build over the same device-resident image and mask, every buffer kept
void shard_rebuild(zi_shard* sh) { shard_start(sh); }

void shard_moments(zi_shard* sh, int64_t* out) {
    zi_multi_index* mi = sh->mi;
    zi_ctx* ctx = mi->ctx;
    const int F = mi->F;
    const size_t nmom = static_cast<size_t>(F) + static_cast<size_t>(F) * F;
    mi->moments.ensure(nmom);
    ZI_CUDA(cudaMemsetAsync(mi->moments.p, 0, nmom * sizeof(unsigned long long), ctx->stream));
    if (mi->n) patch_moments(ctx, mi->image.p, mi->w, mi->C, mi->K, mi->dict.p + sh->row_b, mi->n, mi->moments.p);
    ZI_CUDA(cudaMemcpyAsync(out, mi->moments.p, nmom * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
    ZI_CUDA(cudaStreamSynchronize(ctx->stream));
    sh->stage = 1;
}

static inline int64_t ordered_to_i64(unsigned long long u) { return static_cast<int64_t>(u ^ (1ull << 63)); }
static inline unsigned long long i64_to_ordered(int64_t v) { return static_cast<unsigned long long>(v) ^ (1ull << 63); }

void shard_fit_project(zi_shard* sh, const int64_t* moments, int64_t* lo_out, int64_t* hi_out) {
    if (sh->stage != 1) throw error(ZI_E_INVALID, "shard: fit_project before moments");
    zi_multi_index* mi = sh->mi;
    zi_ctx* ctx = mi->ctx;
    const int F = mi->F, D = sh->D, m = mi->m, mc = mi->mc;
    const size_t nmom = static_cast<size_t>(F) + static_cast<size_t>(F) * F;
    ZI_CUDA(cudaMemcpyAsync(mi->moments.p, moments, nmom * sizeof(unsigned long long), cudaMemcpyHostToDevice,
                            ctx->stream));
    fit_models(mi, sh->n_total);
    const uint64_t n = mi->n, N = 8 * n;
    const int W = sh->W;
    mi->minmax.ensure(static_cast<size_t>(8) * 2 * D);
    std::vector<unsigned long long> hmm(static_cast<size_t>(8) * 2 * D);
    // tensor-core path: the records are written by the quantise pass (phase B), so they exist now
    mi->recs.ensure(static_cast<size_t>(W + 1) * (N ? N : 1));
    sh->tc = shard_tc_begin(mi, mi->recs.p, mi->recs.p + static_cast<size_t>(W) * N, N, hmm.data());
    if (!sh->tc) {
        // empty slices keep the identity ranges (lo = +max, hi = -max in the ordered encoding)
        for (int l = 0; l < 8; ++l) {
            ZI_CUDA(cudaMemsetAsync(mi->minmax.p + static_cast<size_t>(l) * 2 * D, 0xff, D * sizeof(unsigned long long), ctx->stream));
            ZI_CUDA(cudaMemsetAsync(mi->minmax.p + static_cast<size_t>(l) * 2 * D + D, 0, D * sizeof(unsigned long long), ctx->stream));
        }
        sh->Y.ensure(static_cast<size_t>(8) * D * (n ? n : 1));
        for (int l = 0; l < 8; ++l)
            project(ctx, mi->image.p, mi->w, mi->C, mi->dict.p + sh->row_b, n, mi->layout_off.p + static_cast<size_t>(l) * m, m,
                    mi->pca_mean.p + static_cast<size_t>(l) * mc, mi->pca_comp.p + static_cast<size_t>(l) * mc * D, D,
                    sh->Y.p + static_cast<size_t>(l) * D * n, mi->minmax.p + static_cast<size_t>(l) * 2 * D);
        ZI_CUDA(cudaMemcpyAsync(hmm.data(), mi->minmax.p, hmm.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                ctx->stream));
        ZI_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    for (int l = 0; l < 8; ++l)
        for (int d = 0; d < D; ++d) {
            lo_out[l * D + d] = ordered_to_i64(hmm[static_cast<size_t>(l) * 2 * D + d]);
            hi_out[l * D + d] = ordered_to_i64(hmm[static_cast<size_t>(l) * 2 * D + D + d]);
        }
    sh->refined = false;
    mi->host_model = false;
    mi->host_lohi = false;
    sh->stage = 2;
}

void shard_refine_ranges(zi_shard* sh, const int64_t* lo, const int64_t* hi, int64_t* lo_out, int64_t* hi_out) {
    if (sh->stage != 2 || sh->refined) throw error(ZI_E_INVALID, "shard: refine_ranges out of order");
    const int D = sh->D;
    if (!sh->tc) {  // the fp64 path's ranges are exact already
        std::copy(lo, lo + 8 * D, lo_out);
        std::copy(hi, hi + 8 * D, hi_out);
        sh->refined = true;
        return;
    }
    zi_multi_index* mi = sh->mi;
    const int W = sh->W;
    const uint64_t N = 8 * mi->n;
    std::vector<unsigned long long> amm(static_cast<size_t>(8) * 2 * D), ex(static_cast<size_t>(8) * 2 * D);
    for (int l = 0; l < 8; ++l)
        for (int d = 0; d < D; ++d) {
            amm[static_cast<size_t>(l) * 2 * D + d] = i64_to_ordered(lo[l * D + d]);
            amm[static_cast<size_t>(l) * 2 * D + D + d] = i64_to_ordered(hi[l * D + d]);
        }
    shard_tc_quantize(mi, mi->recs.p, mi->recs.p + static_cast<size_t>(W) * N, N, amm.data(), ex.data());
    for (int l = 0; l < 8; ++l)
        for (int d = 0; d < D; ++d) {
            lo_out[l * D + d] = ordered_to_i64(ex[static_cast<size_t>(l) * 2 * D + d]);
            hi_out[l * D + d] = ordered_to_i64(ex[static_cast<size_t>(l) * 2 * D + D + d]);
        }
    sh->refined = true;
}

void shard_quantize_sort(zi_shard* sh, const int64_t* lo, const int64_t* hi, uint32_t S, uint32_t* samples_out) {
    if (sh->stage != 2 || !sh->refined) throw error(ZI_E_INVALID, "shard: quantize before fit_project / refine_ranges");
    zi_multi_index* mi = sh->mi;
    zi_ctx* ctx = mi->ctx;
    const int D = sh->D, W = sh->W;
    const uint64_t n = mi->n, N = 8 * n;
    std::vector<unsigned long long> hmm(static_cast<size_t>(8) * 2 * D);
    for (int l = 0; l < 8; ++l)
        for (int d = 0; d < D; ++d) {
            hmm[static_cast<size_t>(l) * 2 * D + d] = i64_to_ordered(lo[l * D + d]);
            hmm[static_cast<size_t>(l) * 2 * D + D + d] = i64_to_ordered(hi[l * D + d]);
        }
    ZI_CUDA(cudaMemcpyAsync(mi->minmax.p, hmm.data(), hmm.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice,
                            ctx->stream));
    mi->recs.ensure(static_cast<size_t>(W + 1) * (N ? N : 1));
    uint32_t* keyw = mi->recs.p;
    uint32_t* val = mi->recs.p + static_cast<size_t>(W) * N;
    if (sh->tc) {
        shard_tc_fixup(mi, keyw, val, N);  // the exact records of the listed pairs
    } else {
        for (int l = 0; l < 8; ++l)
            quantize_interleave(ctx, sh->Y.p + static_cast<size_t>(l) * D * n, mi->minmax.p + static_cast<size_t>(l) * 2 * D,
                                n, N, static_cast<uint32_t>(l), D, keyw, val, static_cast<uint32_t>(sh->row_b));
    }
    // the 8 layouts are equal groups of n records: sorted each on its own (no layout-digit pass)
    for (int k = 0; k <= W; ++k) sh->sorted[k] = keyw + static_cast<size_t>(k) * N;
    if (N) morton_sort_records(ctx, keyw, val, n, 8, D, true, sh->sorted);
    if (sh->world > 1 && sh->sorted[0] != keyw) {
        // the sort left the records in the context scratch; another shard of this process (or
        // the receive-side sort) reuses it before partition: keep them in the shard's buffer
        for (int k = 0; k <= W; ++k) {
            ZI_CUDA(cudaMemcpyAsync(keyw + static_cast<size_t>(k) * N, sh->sorted[k], N * sizeof(uint32_t),
                                    cudaMemcpyDeviceToDevice, ctx->stream));
            sh->sorted[k] = keyw + static_cast<size_t>(k) * N;
        }
    }
    if (S) {
        uint32_t* d = sh->small.ensure(static_cast<size_t>(8) * S * (W + 1));
        ZI_LAUNCH(ctx, "shard_samples", k_shard_samples, (8 * S + 255) / 256, 256, 0, sh->sorted[0], N, W, n,
                  static_cast<int>(S), d);
        ZI_CUDA(cudaMemcpyAsync(samples_out, d, static_cast<size_t>(8) * S * (W + 1) * sizeof(uint32_t),
                                cudaMemcpyDeviceToHost, ctx->stream));
    }
    ZI_CUDA(cudaStreamSynchronize(ctx->stream));
    sh->stage = 3;
}

void shard_splitters(const uint32_t* samples, uint64_t count, int W, int world, uint32_t* out) {
    const int W1 = W + 1;
    std::vector<std::vector<const uint32_t*>> by(8);
    for (uint64_t i = 0; i < count; ++i) {
        const uint32_t* r = samples + i * W1;
        if (r[W] == kSentinel) continue;
        by[r[W] >> 29].push_back(r);
    }
    for (int l = 0; l < 8; ++l) {
        auto& v = by[l];
        std::sort(v.begin(), v.end(), [W](const uint32_t* a, const uint32_t* b) { return host_rec_less(a, b, W); });
        for (int j = 1; j < world; ++j) {
            uint32_t* o = out + (static_cast<size_t>(l) * (world - 1) + (j - 1)) * W1;
            if (v.empty()) {
                for (int k = 0; k < W1; ++k) o[k] = kSentinel;
            } else {
                const uint32_t* r = v[(static_cast<uint64_t>(j) * v.size()) / world];
                std::memcpy(o, r, W1 * sizeof(uint32_t));
            }
        }
    }
}

void shard_partition(zi_shard* sh, const uint32_t* splitters, uint64_t* counts_out, const uint32_t** d_send) {
    if (sh->stage != 3) throw error(ZI_E_INVALID, "shard: partition before quantize");
    zi_multi_index* mi = sh->mi;
    zi_ctx* ctx = mi->ctx;
    const int W = sh->W, G = sh->world, P = G - 1;
    const uint64_t n = mi->n, N = 8 * n;
    std::vector<uint64_t> bounds(static_cast<size_t>(8) * (P + 2), 0);  // [l][0..G]: 0, lower bounds, n
    if (P > 0 && n > 0) {
        uint32_t* d = sh->small.ensure(static_cast<size_t>(8) * P * (W + 1));
        ZI_CUDA(cudaMemcpyAsync(d, splitters, static_cast<size_t>(8) * P * (W + 1) * sizeof(uint32_t),
                                cudaMemcpyHostToDevice, ctx->stream));
        unsigned long long* dp = reinterpret_cast<unsigned long long*>(sh->pos.ensure(static_cast<size_t>(8) * P));
        ZI_LAUNCH(ctx, "shard_bounds", k_shard_bounds, (8 * P + 127) / 128, 128, 0, sh->sorted[0], N, W, n, d, P, dp);
        std::vector<uint64_t> hp(static_cast<size_t>(8) * P);
        ZI_CUDA(cudaMemcpyAsync(hp.data(), dp, hp.size() * sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
        ZI_CUDA(cudaStreamSynchronize(ctx->stream));
        for (int l = 0; l < 8; ++l)
            for (int j = 0; j < P; ++j) bounds[static_cast<size_t>(l) * (P + 2) + 1 + j] = hp[static_cast<size_t>(l) * P + j];
    }
    for (int l = 0; l < 8; ++l) {
        bounds[static_cast<size_t>(l) * (P + 2) + P + 1] = n;
        for (int j = 1; j <= P + 1; ++j)  // splitters are sorted, but keep the bounds monotone regardless
            bounds[static_cast<size_t>(l) * (P + 2) + j] =
                std::max(bounds[static_cast<size_t>(l) * (P + 2) + j], bounds[static_cast<size_t>(l) * (P + 2) + j - 1]);
    }
    std::vector<seg_t> segs;
    uint64_t dst = 0;
    for (int g = 0; g < G; ++g)
        for (int l = 0; l < 8; ++l) {
            const uint64_t b = bounds[static_cast<size_t>(l) * (P + 2) + g], e = bounds[static_cast<size_t>(l) * (P + 2) + g + 1];
            counts_out[static_cast<size_t>(g) * 8 + l] = e - b;
            segs.push_back({static_cast<unsigned long long>(static_cast<uint64_t>(l) * n + b), dst, e - b});
            dst += e - b;
        }
    sh->send.ensure(static_cast<size_t>(W + 1) * (N ? N : 1));
    move_segments(sh, sh->sorted[0], N, sh->send.p, 0, segs, N);
    *d_send = sh->send.p;
    sh->stage = 4;
}

void shard_rebalance_plan(const uint64_t* all_counts, int world, uint64_t n_total, int me, uint64_t* send_counts,
                          uint64_t* send_starts) {
    const int G = world;
    for (int l = 0; l < 8; ++l) {
        uint64_t P = 0, c = 0;  // global position of my first held record of layout l, my held count
        for (int r = 0; r < G; ++r)
            for (int s = 0; s < G; ++s) {
                const uint64_t v = all_counts[(static_cast<size_t>(s) * G + r) * 8 + l];
                if (r < me) P += v;
                if (r == me) c += v;
            }
        for (int g = 0; g < G; ++g) {
            uint64_t B, E;
            shard_ranges(n_total, G, g, &B, &E);
            const uint64_t lo = std::max(B, P), hi = std::min(E, P + c);
            send_counts[static_cast<size_t>(g) * 8 + l] = hi > lo ? hi - lo : 0;
            send_starts[static_cast<size_t>(g) * 8 + l] = hi > lo ? lo - P : 0;
        }
    }
}

void shard_receive(zi_shard* sh, const uint32_t* d_recv, const uint64_t* all_counts, uint64_t* counts2_out,
                   const uint32_t** d_send2) {
    if (sh->stage != 4) throw error(ZI_E_INVALID, "shard: receive before partition");
    zi_multi_index* mi = sh->mi;
    zi_ctx* ctx = mi->ctx;
    const int W = sh->W, G = sh->world, me = sh->rank;
    uint64_t N1 = 0;
    std::vector<uint64_t> held(8, 0);
    for (int s = 0; s < G; ++s)
        for (int l = 0; l < 8; ++l) {
            const uint64_t v = all_counts[(static_cast<size_t>(s) * G + me) * 8 + l];
            held[l] += v;
            N1 += v;
        }
    sh->held = N1;
    mi->recs.ensure(static_cast<size_t>(W + 1) * (N1 ? N1 : 1));
    if (N1) {
        move_segments(sh, d_recv, 0, mi->recs.p, N1, {{0ull, 0ull, N1}}, N1);  // AoS -> SoA
        // one rank receives its own locally sorted records back in order: nothing to merge
        if (G > 1) morton_sort_layouts(ctx, mi->recs.p, mi->recs.p + static_cast<size_t>(W) * N1, N1, sh->D);
    }
    std::vector<uint64_t> starts(static_cast<size_t>(G) * 8);
    shard_rebalance_plan(all_counts, G, sh->n_total, me, counts2_out, starts.data());
    std::vector<seg_t> segs;
    uint64_t dst = 0, lbase[8], acc = 0;  // the sorted records are layout-major
    for (int l = 0; l < 8; ++l) {
        lbase[l] = acc;
        acc += held[l];
    }
    for (int g = 0; g < G; ++g)
        for (int l = 0; l < 8; ++l) {
            const uint64_t c = counts2_out[static_cast<size_t>(g) * 8 + l];
            segs.push_back({lbase[l] + starts[static_cast<size_t>(g) * 8 + l], dst, c});
            dst += c;
        }
    sh->send.ensure(static_cast<size_t>(W + 1) * (N1 ? N1 : 1));
    if (N1) move_segments(sh, mi->recs.p, N1, sh->send.p, 0, segs, N1);
    *d_send2 = sh->send.p;
    sh->stage = 5;
}

void shard_finish(zi_shard* sh, const uint32_t* d_recv2, const uint64_t* all_counts2) {
    if (sh->stage != 5) throw error(ZI_E_INVALID, "shard: finish before receive");
    zi_multi_index* mi = sh->mi;
    zi_ctx* ctx = mi->ctx;
    const int W = sh->W, G = sh->world, me = sh->rank, D = sh->D;
    const uint64_t n = mi->n, N = 8 * n;
    // incoming order: source-major, then layout; target: layout-major, then source
    std::vector<seg_t> segs;
    uint64_t src = 0;
    std::vector<uint64_t> fill(8, 0);
    for (int s = 0; s < G; ++s)
        for (int l = 0; l < 8; ++l) {
            const uint64_t c = all_counts2[(static_cast<size_t>(s) * G + me) * 8 + l];
            segs.push_back({src, static_cast<unsigned long long>(static_cast<uint64_t>(l) * n + fill[l]), c});
            src += c;
            fill[l] += c;
        }
    for (int l = 0; l < 8; ++l)
        if (fill[l] != n) throw error(ZI_E_RUNTIME, "shard: rebalanced layout size disagrees with the shard range");
    mi->recs.ensure(static_cast<size_t>(W + 1) * (N ? N : 1));
    if (N) move_segments(sh, d_recv2, 0, mi->recs.p, N, segs, N);
    for (int l = 0; l < 8; ++l) {
        mi->L[l].index.ctx = ctx;
        mi->L[l].index.layout_id = static_cast<uint32_t>(l);
        finalize_index(ctx, mi->recs.p, mi->recs.p + static_cast<size_t>(W) * N, N, static_cast<uint64_t>(l) * n, n, D,
                       mi->dict.p, &mi->L[l].index);
    }
    ZI_CUDA(cudaStreamSynchronize(ctx->stream));
    sh->Y.release();
    sh->send.release();
    mi->host_lohi = false;
    sh->stage = 6;
}

// one rank: the locally sorted layouts ARE the index -- finalise them, no exchange
void shard_finish_local(zi_shard* sh) {
    if (sh->stage != 3 || sh->world != 1) throw error(ZI_E_INVALID, "shard: finish_local needs world 1 after quantize");
    zi_multi_index* mi = sh->mi;
    zi_ctx* ctx = mi->ctx;
    const int W = sh->W, D = sh->D;
    const uint64_t n = mi->n, N = 8 * n;
    for (int l = 0; l < 8; ++l) {
        mi->L[l].index.ctx = ctx;
        mi->L[l].index.layout_id = static_cast<uint32_t>(l);
        finalize_index(ctx, sh->sorted[0], sh->sorted[W], N, static_cast<uint64_t>(l) * n, n, D, mi->dict.p,
                       &mi->L[l].index);
    }
    mi->host_lohi = false;
    sh->held = N;
    sh->stage = 6;
}

zi_multi_index* shard_multi_index(zi_shard* sh) { return sh->mi; }

void shard_destroy(zi_shard* sh) { delete sh; }

void shard_info(const zi_shard* sh, uint64_t* v) {
    v[0] = sh->n_total;
    v[1] = sh->row_b;
    v[2] = sh->row_e;
    v[3] = static_cast<uint64_t>(sh->mi->F);
    v[4] = static_cast<uint64_t>(sh->D);
    v[5] = static_cast<uint64_t>(sh->W);
    v[6] = static_cast<uint64_t>(sh->rank);
    v[7] = static_cast<uint64_t>(sh->world);
    v[8] = static_cast<uint64_t>(sh->stage);
    v[9] = sh->held;
}

}  // namespace zi
