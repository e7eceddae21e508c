// build.cu -- multi_index::build on the device (proj/src/builder.cpp:129-224).
//
// Pipeline (one stream, everything device resident except the tiny eigen-solves):
//   K1 collect_dictionary -> n keys (row-major)                       builder.cpp:74-108
//   K2 exact int64 moments of the full K*K*C vector (one Gram serves
//      all 8 layouts: each layout's covariance is a sub-block)        pca.cpp:20-37
//   8 covariance + eigen-solves, one CTA per layout (k_pca.cu; host
//      fallback host_pca.cpp when mc > 224 or ZI_HOST_PCA is set)      pca.cpp:39-67
//   per layout: K3 project (fp64 canonical) -> min/max -> quantise +
//      Morton interleave -> K4 onesweep radix sort -> K5 finalize      builder.cpp:159-195
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <thread>
#include <vector>

#include "common.cuh"

namespace zi {

// device moments -> host s, S (full symmetric; k_moments computes tile pairs ti <= tj only)
static void moments_to_host(zi_ctx* ctx, const unsigned long long* d_mom, int F, hbuf<unsigned long long>& stage,
                            std::vector<int64_t>& s, std::vector<int64_t>& S) {
    const size_t nmom = static_cast<size_t>(F) + static_cast<size_t>(F) * F;
    unsigned long long* hm = stage.ensure(nmom);
    ZI_CUDA(cudaMemcpyAsync(hm, d_mom, nmom * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
    ZI_CUDA(cudaStreamSynchronize(ctx->stream));
    s.assign(F, 0);
    S.assign(static_cast<size_t>(F) * F, 0);
    for (int i = 0; i < F; ++i) s[i] = static_cast<int64_t>(hm[i]);
    constexpr int kTile = 128;
    for (int i = 0; i < F; ++i)
        for (int j = 0; j < F; ++j) {
            const int a = (i / kTile <= j / kTile) ? i : j, b = (i / kTile <= j / kTile) ? j : i;
            S[static_cast<size_t>(i) * F + j] = static_cast<int64_t>(hm[F + static_cast<size_t>(a) * F + b]);
        }
}

static void sync_moments(zi_multi_index* mi) { moments_to_host(mi->ctx, mi->moments.p, mi->F, mi->hmom, mi->s, mi->S); }

void finish_build_timing(zi_multi_index* mi) {
    if (!mi->build_ms_pending) return;
    ZI_CUDA(cudaEventSynchronize(mi->ev1));
    float ms = 0.f;
    ZI_CUDA(cudaEventElapsedTime(&ms, mi->ev0, mi->ev1));
    mi->build_ms = ms;
    mi->build_ms_pending = false;
}

void sync_host_model(zi_multi_index* mi) {
    if (!mi->host_lohi && mi->n > 0) {
        const int D = mi->dims;
        std::vector<unsigned long long> hmm(static_cast<size_t>(8) * 2 * D);
        ZI_CUDA(cudaMemcpyAsync(hmm.data(), mi->minmax.p, hmm.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                mi->ctx->stream));
        ZI_CUDA(cudaStreamSynchronize(mi->ctx->stream));
        for (int l = 0; l < 8; ++l) {
            mi->L[l].lo.resize(D);
            mi->L[l].hi.resize(D);
            for (int d = 0; d < D; ++d) {
                mi->L[l].lo[d] = ordered_to_double(hmm[static_cast<size_t>(l) * 2 * D + d]);
                mi->L[l].hi[d] = ordered_to_double(hmm[static_cast<size_t>(l) * 2 * D + D + d]);
            }
        }
        mi->host_lohi = true;
    }
    if (mi->host_model || mi->n == 0) return;
    zi_ctx* ctx = mi->ctx;
    const int mc = mi->mc, D = mi->dims;
    sync_moments(mi);
    std::vector<double> hmean(static_cast<size_t>(8) * mc), hcomp(static_cast<size_t>(8) * mc * D),
        heig(static_cast<size_t>(8) * D);
    ZI_CUDA(cudaMemcpyAsync(hmean.data(), mi->pca_mean.p, hmean.size() * sizeof(double), cudaMemcpyDeviceToHost,
                            ctx->stream));
    ZI_CUDA(cudaMemcpyAsync(hcomp.data(), mi->pca_comp.p, hcomp.size() * sizeof(double), cudaMemcpyDeviceToHost,
                            ctx->stream));
    ZI_CUDA(cudaMemcpyAsync(heig.data(), mi->pca_eig.p, heig.size() * sizeof(double), cudaMemcpyDeviceToHost,
                            ctx->stream));
    ZI_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int l = 0; l < 8; ++l) {
        auto& L = mi->L[l];
        L.mean.assign(hmean.begin() + static_cast<size_t>(l) * mc, hmean.begin() + static_cast<size_t>(l + 1) * mc);
        L.comp.assign(static_cast<size_t>(D) * mc, 0.0);
        for (int j = 0; j < mc; ++j)
            for (int d = 0; d < D; ++d)
                L.comp[static_cast<size_t>(d) * mc + j] = hcomp[(static_cast<size_t>(l) * mc + j) * D + d];
        L.eig.assign(heig.begin() + static_cast<size_t>(l) * D, heig.begin() + static_cast<size_t>(l + 1) * D);
    }
    mi->host_model = true;
}

void fit_models(zi_multi_index* mi, uint64_t n) {
    zi_ctx* ctx = mi->ctx;
    const int K = mi->K, C = mi->C, F = mi->F, D = mi->dims, mc = mi->mc, m = mi->m;
    mi->pca_mean.ensure(static_cast<size_t>(8) * mc);
    mi->pca_comp.ensure(static_cast<size_t>(8) * mc * D);
    mi->host_model = false;
    const auto te0 = std::chrono::steady_clock::now();
    static const bool host_pca = std::getenv("ZI_HOST_PCA") != nullptr;
    bool on_device = false;
    if (!host_pca) {
        if (!mi->pca_cols_ready) {
            std::vector<int32_t> hc;
            for (int l = 0; l < 8; ++l)
                for (int p = 0; p < m; ++p)
                    for (int ch = 0; ch < C; ++ch)
                        hc.push_back((mi->L[l].rc[2 * p] * K + mi->L[l].rc[2 * p + 1]) * C + ch);
            mi->pca_cols.ensure(hc.size());
            ZI_CUDA(cudaMemcpyAsync(mi->pca_cols.p, hc.data(), hc.size() * sizeof(int32_t), cudaMemcpyHostToDevice,
                                    ctx->stream));
            ZI_CUDA(cudaStreamSynchronize(ctx->stream));  // hc is a pageable local
            mi->pca_cols_ready = true;
        }
        mi->pca_eig.ensure(static_cast<size_t>(8) * 32);
        mi->pca_work.ensure(pca_work_doubles(mc, D));
        mi->pca_status.ensure(8);
        on_device = pca_on_device(ctx, mi->moments.p, F, n, mi->pca_cols.p, mc, D, mi->pca_mean.p, mi->pca_comp.p,
                                  mi->pca_eig.p, mi->pca_work.p, mi->pca_status.p);
    }
    mi->device_pca = on_device;
    if (!on_device) {
        // host eigen-solves, one thread per layout
        sync_moments(mi);
        std::vector<std::thread> th;
        for (int l = 0; l < 8; ++l) {
            th.emplace_back([mi, l, F, n, D, C, K, m] {
                auto& L = mi->L[l];
                std::vector<int32_t> cols;
                for (int p = 0; p < m; ++p)
                    for (int ch = 0; ch < C; ++ch) cols.push_back((L.rc[2 * p] * K + L.rc[2 * p + 1]) * C + ch);
                pca_fit_layout(mi->s, mi->S, F, n, cols, D, L.mean, L.comp, L.eig);
            });
        }
        for (auto& t : th) t.join();
        // upload the 8 models: mean [l][j], comp [l][j][d]
        std::vector<double> hmean(static_cast<size_t>(8) * mc), hcomp(static_cast<size_t>(8) * mc * D);
        for (int l = 0; l < 8; ++l) {
            std::copy(mi->L[l].mean.begin(), mi->L[l].mean.end(), hmean.begin() + static_cast<size_t>(l) * mc);
            for (int j = 0; j < mc; ++j)
                for (int d = 0; d < D; ++d)
                    hcomp[(static_cast<size_t>(l) * mc + j) * D + d] = mi->L[l].comp[static_cast<size_t>(d) * mc + j];
        }
        ZI_CUDA(cudaMemcpyAsync(mi->pca_mean.p, hmean.data(), hmean.size() * sizeof(double), cudaMemcpyHostToDevice,
                                ctx->stream));
        ZI_CUDA(cudaMemcpyAsync(mi->pca_comp.p, hcomp.data(), hcomp.size() * sizeof(double), cudaMemcpyHostToDevice,
                                ctx->stream));
        ZI_CUDA(cudaStreamSynchronize(ctx->stream));  // hmean / hcomp are pageable locals
        mi->host_model = true;
    }
    mi->eigen_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - te0).count();

}

void build_multi_index(zi_multi_index* mi) {
    zi_ctx* ctx = mi->ctx;
    const auto wall0 = std::chrono::steady_clock::now();
    if (!mi->ev0) {
        ZI_CUDA(cudaEventCreate(&mi->ev0));
        ZI_CUDA(cudaEventCreate(&mi->ev1));
    }
    ZI_CUDA(cudaEventRecord(mi->ev0, ctx->stream));
    const int K = mi->K, C = mi->C, w = mi->w, h = mi->h;

    // K1
    mi->n = collect_dictionary(ctx, mi->known.p, w, h, K, mi->dict);
    if (mi->n == 0) throw error(ZI_E_EMPTY_DICT, "no fully known patch window; inpainting impossible");
    const uint64_t n = mi->n;
    if (mi->dict_out) {  // zi_multi_index_build_to: the dictionary goes home while the build runs
        if (n > mi->dict_cap) throw error(ZI_E_INVALID, "build_to: dictionary larger than the output buffer");
        ZI_CUDA(cudaEventRecord(ctx->ev_dict, ctx->stream));
        ZI_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_dict, 0));
        ZI_CUDA(cudaMemcpyAsync(mi->dict_out, mi->dict.p, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->copy_stream));
        ZI_CUDA(cudaEventRecord(ctx->ev_copy, ctx->copy_stream));
    }
    if (mi->image_on_copy) ZI_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_img, 0));  // the moments read it
    mi->dims = static_cast<int>(std::min<uint64_t>(static_cast<uint64_t>(mi->cfg.dims),
                                                   std::min<uint64_t>(static_cast<uint64_t>(mi->mc), n)));
    const int D = mi->dims, mc = mi->mc, m = mi->m;

    // K2
    const int F = K * K * C;
    mi->F = F;
    const size_t nmom = static_cast<size_t>(F) + static_cast<size_t>(F) * F;
    mi->moments.ensure(nmom);
    patch_moments(ctx, mi->image.p, w, C, K, mi->dict.p, n, mi->moments.p);
    fit_models(mi, n);

    mi->minmax.ensure(static_cast<size_t>(8) * 2 * D);

    // per layout: project, lo/hi, quantise + interleave into one 8n-record array; then ONE
    // radix sort over all layouts (better occupancy than 8 small sorts) and per-layout finalize
    const int W = (D + 3) / 4;
    const uint64_t N = 8 * n;
    if (N > (1ull << 30)) throw error(ZI_E_INVALID, "dictionary above 2^27 patches");
    zi::dbuf<uint32_t>& recs = mi->recs;
    recs.ensure(static_cast<size_t>(W + 1) * N);
    uint32_t* keyw = recs.p;
    uint32_t* val = recs.p + static_cast<size_t>(W) * N;
    // a sort that goes straight to LSD passes writes the indices in its last pass; its records
    // then carry the patch key as payload (same tie order as the row: the dictionary is ascending)
    static const bool no_fuse = std::getenv("ZI_SORT_NO_FUSE") != nullptr;  // A/B: separate finalize
    bool fuse = !no_fuse && layouts_sort_fuses(ctx, D);
    mi->payload_key = fuse;
    if (!project_quantize_tc(mi, keyw, val, N)) {
        mi->payload_key = fuse = false;  // the fp64 fallback writes (layout << 29) | row
        for (int l = 0; l < 8; ++l) {
            unsigned long long* mm = mi->minmax.p + static_cast<size_t>(l) * 2 * D;
            mi->proj.ensure(static_cast<size_t>(D) * n);
            project(ctx, mi->image.p, w, C, mi->dict.p, n, mi->layout_off.p + static_cast<size_t>(l) * m, m,
                    mi->pca_mean.p + static_cast<size_t>(l) * mc, mi->pca_comp.p + static_cast<size_t>(l) * mc * D, D,
                    mi->proj.p, mm);
            quantize_interleave(ctx, mi->proj.p, mm, n, N, static_cast<uint32_t>(l), D, keyw, val);
        }
    }
    uint32_t* sorted[10];  // the sorted records, possibly in the sort's scratch (no copy back)
    // when the sort ends in an LSD pass, that pass writes the indices' planes and keys itself
    final_sink sink{};
    for (int l = 0; l < 8; ++l) {
        zi_index* idx = &mi->L[l].index;
        idx->ctx = ctx;
        idx->layout_id = static_cast<uint32_t>(l);
        prepare_index(idx, n, D);
        sink.planes[l] = idx->planes.p;
        sink.keys[l] = idx->keys.p;
    }
    sink.dict = nullptr;  // the payload is the key
    const bool fused = morton_sort_records(ctx, keyw, val, n, 8, D, true, sorted, true, fuse ? &sink : nullptr);
    if (fuse != fused) throw error(ZI_E_RUNTIME, "build: the layout sort did not take its fused path");
    mi->payload_key = false;
    if (fused) {
        zi_index* idx[8];
        for (int l = 0; l < 8; ++l) idx[l] = &mi->L[l].index;
        finalize_index_bboxes(ctx, idx, 8);
    } else {
        zi_index* idx[8];
        for (int l = 0; l < 8; ++l) idx[l] = &mi->L[l].index;
        finalize_layout_indexes(ctx, sorted[0], sorted[W], N, n, D, mi->dict.p, idx, 8);
    }
    if (mi->dict_out) ZI_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_copy, 0));
    ZI_CUDA(cudaEventRecord(mi->ev1, ctx->stream));
    mi->build_ms_pending = true;
    mi->host_lohi = false;
    mi->wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
}

// build_index (proj/src/builder.cpp:129-195) for ONE layout over the caller's dictionary: the
// moments of the full K*K*C vector (the layout's covariance is a sub-block), one device
// eigen-solve, the canonical fp64 projection + min/max, quantise + Morton interleave, the hybrid
// Morton sort and finalize.  The reference's per-layout entry point (builder.hpp:77-81); the
// multi-index path (build_multi_index) runs the same stages for eight layouts at once.
void build_patch_index(zi_patch_index* pi) {
    zi_ctx* ctx = pi->ctx;
    const int K = pi->K, C = pi->C, m = pi->m, mc = pi->mc, F = K * K * C;
    const uint64_t n = pi->n;
    pi->F = F;
    pi->dims = static_cast<int>(std::min<uint64_t>(static_cast<uint64_t>(pi->cfg.dims),
                                                   std::min<uint64_t>(static_cast<uint64_t>(mc), n)));
    const int D = pi->dims;
    cudaEvent_t e0, e1, e2;
    ZI_CUDA(cudaEventCreate(&e0));
    ZI_CUDA(cudaEventCreate(&e1));
    ZI_CUDA(cudaEventCreate(&e2));
    ZI_CUDA(cudaEventRecord(e0, ctx->stream));
    pi->moments.ensure(static_cast<size_t>(F) + static_cast<size_t>(F) * F);
    patch_moments(ctx, pi->image.p, pi->w, C, K, pi->dict.p, n, pi->moments.p);
    pi->mean.ensure(mc);
    pi->comp.ensure(static_cast<size_t>(mc) * D);
    pi->eig.ensure(32);
    pi->work.ensure(pca_work_doubles(mc, D));
    static const bool host_pca = std::getenv("ZI_HOST_PCA") != nullptr;
    pi->device_pca = !host_pca && pca_on_device_n(ctx, 1, pi->moments.p, F, n, pi->cols.p, mc, D, pi->mean.p,
                                                  pi->comp.p, pi->eig.p, pi->work.p);
    if (!pi->device_pca) {
        hbuf<unsigned long long> stage;
        std::vector<int64_t> hs, hS;
        moments_to_host(ctx, pi->moments.p, F, stage, hs, hS);
        std::vector<int32_t> cols;
        for (int p = 0; p < m; ++p)
            for (int ch = 0; ch < C; ++ch) cols.push_back((pi->rc[2 * p] * K + pi->rc[2 * p + 1]) * C + ch);
        std::vector<double> mean, comp, eig;
        pca_fit_layout(hs, hS, F, n, cols, D, mean, comp, eig);
        std::vector<double> cjd(static_cast<size_t>(mc) * D);
        for (int j = 0; j < mc; ++j)
            for (int d = 0; d < D; ++d) cjd[static_cast<size_t>(j) * D + d] = comp[static_cast<size_t>(d) * mc + j];
        ZI_CUDA(cudaMemcpyAsync(pi->mean.p, mean.data(), mc * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        ZI_CUDA(cudaMemcpyAsync(pi->comp.p, cjd.data(), cjd.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        ZI_CUDA(cudaMemcpyAsync(pi->eig.p, eig.data(), D * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        ZI_CUDA(cudaStreamSynchronize(ctx->stream));  // pageable locals
    }
    pi->minmax.ensure(static_cast<size_t>(2) * D);
    pi->proj.ensure(static_cast<size_t>(D) * n);
    const int W = (D + 3) / 4;
    pi->recs.ensure(static_cast<size_t>(W + 1) * n);
    uint32_t* keyw = pi->recs.p;
    uint32_t* val = pi->recs.p + static_cast<size_t>(W) * n;
    project(ctx, pi->image.p, pi->w, C, pi->dict.p, n, pi->off.p, m, pi->mean.p, pi->comp.p, D, pi->proj.p,
            pi->minmax.p);
    quantize_interleave(ctx, pi->proj.p, pi->minmax.p, n, n, 0, D, keyw, val);
    ZI_CUDA(cudaEventRecord(e1, ctx->stream));
    uint32_t* sorted[10];
    morton_sort_records(ctx, keyw, val, n, 1, D, false, sorted);
    pi->index.ctx = ctx;
    pi->index.layout_id = 0;
    finalize_index(ctx, sorted[0], sorted[W], n, 0, n, D, pi->dict.p, &pi->index);
    ZI_CUDA(cudaEventRecord(e2, ctx->stream));
    ZI_CUDA(cudaEventSynchronize(e2));
    float a = 0.f, b = 0.f;
    ZI_CUDA(cudaEventElapsedTime(&a, e0, e2));
    ZI_CUDA(cudaEventElapsedTime(&b, e1, e2));
    pi->build_ms = a;
    pi->sort_ms = b;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(e2);
    patch_index_sync_host(pi);
}

void patch_index_sync_host(zi_patch_index* pi) {
    zi_ctx* ctx = pi->ctx;
    const int mc = pi->mc, D = pi->dims;
    std::vector<double> cjd(static_cast<size_t>(mc) * D);
    std::vector<unsigned long long> mm(static_cast<size_t>(2) * D);
    pi->h_mean.resize(mc);
    pi->h_eig.resize(D);
    ZI_CUDA(cudaMemcpyAsync(pi->h_mean.data(), pi->mean.p, mc * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    ZI_CUDA(cudaMemcpyAsync(cjd.data(), pi->comp.p, cjd.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    ZI_CUDA(cudaMemcpyAsync(pi->h_eig.data(), pi->eig.p, D * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    ZI_CUDA(cudaMemcpyAsync(mm.data(), pi->minmax.p, mm.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                            ctx->stream));
    ZI_CUDA(cudaStreamSynchronize(ctx->stream));
    pi->h_comp.assign(static_cast<size_t>(D) * mc, 0.0);
    for (int j = 0; j < mc; ++j)
        for (int d = 0; d < D; ++d) pi->h_comp[static_cast<size_t>(d) * mc + j] = cjd[static_cast<size_t>(j) * D + d];
    pi->h_lo.resize(D);
    pi->h_hi.resize(D);
    for (int d = 0; d < D; ++d) {
        pi->h_lo[d] = ordered_to_double(mm[d]);
        pi->h_hi[d] = ordered_to_double(mm[D + d]);
    }
}

}  // namespace zi
