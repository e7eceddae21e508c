// api.cu -- the extern "C" boundary (include/zinpaint_b200.h).  Every entry point catches
// internal exceptions and returns a zi_status; zi_last_error() holds the message.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace {
thread_local std::string g_err;

zi_status fail(zi_status s, const std::string& m) {
    g_err = m;
    return s;
}

template <typename F>
zi_status guard(F&& f) {
    try {
        f();
        g_err.clear();
        return ZI_OK;
    } catch (const zi::error& e) {
        return fail(e.code, e.what());
    } catch (const std::bad_alloc&) {
        return fail(ZI_E_OOM, "host allocation failed");
    } catch (const std::exception& e) {
        return fail(ZI_E_RUNTIME, e.what());
    }
}

void require(bool ok, const char* msg) {
    if (!ok) throw zi::error(ZI_E_INVALID, msg);
}

// guard() with the handle's device current and its stream + pool bound for stream-ordered
// allocations; the caller's current device is restored on exit
struct ctx_scope {
    cudaStream_t prev;
    cudaMemPool_t prev_pool;
    int prev_dev = -1;
    explicit ctx_scope(const zi_ctx* ctx) : prev(zi::tls_alloc_stream), prev_pool(zi::tls_alloc_pool) {
        zi::tls_alloc_stream = ctx ? ctx->stream : nullptr;
        zi::tls_alloc_pool = ctx ? ctx->pool : nullptr;
        int d = -1;
        if (ctx && cudaGetDevice(&d) == cudaSuccess && d != ctx->device && cudaSetDevice(ctx->device) == cudaSuccess)
            prev_dev = d;
    }
    ~ctx_scope() {
        zi::tls_alloc_stream = prev;
        zi::tls_alloc_pool = prev_pool;
        if (prev_dev >= 0) cudaSetDevice(prev_dev);
    }
};
template <typename F>
zi_status guard(const zi_ctx* ctx, F&& f) {
    ctx_scope sc(ctx);
    return guard(std::forward<F>(f));
}
}  // namespace

namespace zi {
thread_local cudaStream_t tls_alloc_stream = nullptr;
thread_local cudaMemPool_t tls_alloc_pool = nullptr;

void set_smem_attr(const void* fn, int device, size_t bytes) {
    static std::mutex mx;
    static std::map<std::pair<const void*, int>, size_t> done;
    std::lock_guard<std::mutex> lk(mx);
    size_t& have = done[{fn, device}];
    if (bytes <= have) return;
    ZI_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
    have = bytes;
}
}

namespace zi {

static bool profiled(const zi_ctx* ctx, const char* name) {
    if (!ctx->profiling) return false;
    if (ctx->prof_filter.empty()) return true;
    for (const auto& f : ctx->prof_filter)
        if (f == name) return true;
    return false;
}

void launch_begin(zi_ctx* ctx, const char* name) {
    ++ctx->launches;
    if (!profiled(ctx, name)) return;
    prof_slot* s = nullptr;
    for (auto& p : ctx->prof)
        if (std::strcmp(p.name, name) == 0) s = &p;
    if (!s) {
        ctx->prof.emplace_back();
        s = &ctx->prof.back();
        s->name = name;
    }
    if (s->used == s->events.size()) {
        cudaEvent_t a, b;
        ZI_CUDA(cudaEventCreate(&a));
        ZI_CUDA(cudaEventCreate(&b));
        s->events.emplace_back(a, b);
    }
    ZI_CUDA(cudaEventRecord(s->events[s->used].first, ctx->stream));
}

void launch_end(zi_ctx* ctx, const char* name) {
    static const bool sync_check = std::getenv("ZI_SYNC_CHECK") != nullptr;
    if (sync_check) {  // debug: attribute asynchronous faults to the kernel that caused them
        const cudaError_t e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) throw error(ZI_E_CUDA, std::string("kernel ") + name + ": " + cudaGetErrorString(e));
    }
    if (!profiled(ctx, name)) return;
    for (auto& p : ctx->prof)
        if (std::strcmp(p.name, name) == 0) {
            ZI_CUDA(cudaEventRecord(p.events[p.used].second, ctx->stream));
            ++p.used;
            ++p.launches;
            return;
        }
}

}  // namespace zi

static void upload_layouts(zi_multi_index* mi) {
    std::vector<int32_t> rc;
    mi->m = zi::subset_layouts(mi->K, mi->cfg.coverage, rc);
    mi->mc = mi->m * mi->C;
    std::vector<int32_t> off(static_cast<size_t>(8) * mi->m), loc(static_cast<size_t>(8) * mi->m);
    for (int l = 0; l < 8; ++l) {
        mi->L[l].rc.assign(rc.begin() + static_cast<size_t>(l) * mi->m * 2, rc.begin() + static_cast<size_t>(l + 1) * mi->m * 2);
        for (int p = 0; p < mi->m; ++p) {
            const int r = mi->L[l].rc[2 * p], c = mi->L[l].rc[2 * p + 1];
            off[static_cast<size_t>(l) * mi->m + p] = (r * mi->w + c) * mi->C;
            loc[static_cast<size_t>(l) * mi->m + p] = r * mi->K + c;
        }
    }
    mi->layout_off.ensure(off.size());
    mi->layout_local.ensure(loc.size());
    ZI_CUDA(cudaMemcpyAsync(mi->layout_off.p, off.data(), off.size() * sizeof(int32_t), cudaMemcpyHostToDevice, mi->ctx->stream));
    ZI_CUDA(cudaMemcpyAsync(mi->layout_local.p, loc.data(), loc.size() * sizeof(int32_t), cudaMemcpyHostToDevice, mi->ctx->stream));
}

static void ensure_copy_stream(zi_ctx* ctx) {
    if (ctx->copy_stream) return;
    ZI_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    for (cudaEvent_t* e : {&ctx->ev_alloc, &ctx->ev_img, &ctx->ev_dict, &ctx->ev_copy})
        ZI_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
}

static void upload_image(zi_multi_index* mi, const uint8_t* image, const uint8_t* known) {
    const size_t npx = static_cast<size_t>(mi->w) * mi->h;
    zi_ctx* ctx = mi->ctx;
    mi->image.ensure(npx * mi->C + 16);  // +16: aligned word loads past the last byte (k_proj_tc gather)
    mi->known.ensure(npx);
    ZI_CUDA(cudaMemcpyAsync(mi->known.p, known, npx, cudaMemcpyHostToDevice, ctx->stream));
    if (mi->image_on_copy) {  // the mask is all the dictionary needs: the image follows on the copy engine
        ensure_copy_stream(ctx);
        ZI_CUDA(cudaEventRecord(ctx->ev_alloc, ctx->stream));  // after the (stream-ordered) allocation
        ZI_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_alloc, 0));
        ZI_CUDA(cudaMemcpyAsync(mi->image.p, image, npx * mi->C, cudaMemcpyHostToDevice, ctx->copy_stream));
        ZI_CUDA(cudaEventRecord(ctx->ev_img, ctx->copy_stream));
    } else {
        ZI_CUDA(cudaMemcpyAsync(mi->image.p, image, npx * mi->C, cudaMemcpyHostToDevice, ctx->stream));
    }
}

static zi_multi_index* new_multi_index(zi_ctx* ctx, const uint8_t* image, const uint8_t* known, int32_t w, int32_t h,
                                       int32_t C, const zi_index_config* cfg, bool image_on_copy = false) {
    require(ctx && image && known && cfg, "null argument");
    require(w > 0 && h > 0 && (C == 1 || C == 3), "raster_image: bad dimensions");
    require(w <= 65535 && h <= 65535, "image side above the 16-bit patch_key range");
    require(static_cast<uint64_t>(w) * h * C < (1ull << 31), "image above 2^31 bytes");
    zi::validate_config(*cfg, C);
    auto* mi = new zi_multi_index();
    mi->ctx = ctx;
    mi->cfg = *cfg;
    mi->w = w;
    mi->h = h;
    mi->C = C;
    mi->K = cfg->patch_size;
    mi->image_on_copy = image_on_copy;
    try {
        upload_layouts(mi);
        upload_image(mi, image, known);
    } catch (...) {
        delete mi;
        throw;
    }
    return mi;
}

extern "C" {

const char* zi_last_error(void) { return g_err.c_str(); }
const char* zi_version(void) { return "zinpaint_b200 0.1 (sm_100a)"; }

zi_status zi_ctx_create(int device, zi_ctx** out) {
    return guard([&] {
        require(out != nullptr, "null argument");
        ZI_CUDA(cudaSetDevice(device));
        auto* c = new zi_ctx();
        c->device = device;
        cudaDeviceProp prop;
        ZI_CUDA(cudaGetDeviceProperties(&prop, device));
        c->num_sms = prop.multiProcessorCount;
        ZI_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        // a private pool: the no-trim threshold applies to this ctx's allocations only, not to the
        // device's default pool that other libraries in the process (torch, NCCL) allocate from
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = device;
        ZI_CUDA(cudaMemPoolCreate(&c->pool, &props));
        uint64_t keep = ~0ull;  // never trim: rebuilds reuse the pool's HBM
        ZI_CUDA(cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &keep));
        ZI_CUDA(cudaEventCreate(&c->t0));
        ZI_CUDA(cudaEventCreate(&c->t1));
        *out = c;
    });
}

zi_status zi_ctx_destroy(zi_ctx* ctx) {
    return guard(ctx, [&] {
        if (!ctx) return;
        cudaStreamSynchronize(ctx->stream);
        for (auto& p : ctx->prof)
            for (auto& e : p.events) {
                cudaEventDestroy(e.first);
                cudaEventDestroy(e.second);
            }
        cudaEventDestroy(ctx->t0);
        cudaEventDestroy(ctx->t1);
        if (ctx->copy_stream) {
            cudaStreamSynchronize(ctx->copy_stream);
            for (cudaEvent_t e : {ctx->ev_alloc, ctx->ev_img, ctx->ev_dict, ctx->ev_copy}) cudaEventDestroy(e);
            cudaStreamDestroy(ctx->copy_stream);
        }
        ctx->scratch.release();  // stream-ordered frees before the stream goes away
        ctx->ss_buf.release();
        ctx->counter.release();
        ctx->flush.release();
        ctx->gm_wtab.release();
        cudaStreamSynchronize(ctx->stream);
        cudaStreamDestroy(ctx->stream);
        if (ctx->pool) cudaMemPoolDestroy(ctx->pool);  // released once its last allocation is freed
        delete ctx;
    });
}

zi_status zi_ctx_synchronize(zi_ctx* ctx) {
    return guard(ctx, [&] { ZI_CUDA(cudaStreamSynchronize(ctx->stream)); });
}

zi_status zi_timer_start(zi_ctx* ctx) {
    return guard(ctx, [&] { ZI_CUDA(cudaEventRecord(ctx->t0, ctx->stream)); });
}

zi_status zi_timer_stop(zi_ctx* ctx, double* ms) {
    return guard(ctx, [&] {
        ZI_CUDA(cudaEventRecord(ctx->t1, ctx->stream));
        ZI_CUDA(cudaEventSynchronize(ctx->t1));
        float f = 0.f;
        ZI_CUDA(cudaEventElapsedTime(&f, ctx->t0, ctx->t1));
        *ms = f;
    });
}

uint64_t zi_ctx_kernel_launches(const zi_ctx* ctx) { return ctx ? ctx->launches : 0; }

zi_status zi_ctx_flush_l2(zi_ctx* ctx) {
    return guard(ctx, [&] {
        const size_t bytes = size_t(256) << 20;
        uint8_t* p = ctx->flush.ensure(bytes);
        ZI_CUDA(cudaMemsetAsync(p, ctx->flush_toggle++ & 0xff, bytes, ctx->stream));
    });
}

zi_status zi_ctx_set_profiling(zi_ctx* ctx, int on) {
    return guard(ctx, [&] {
        ZI_CUDA(cudaStreamSynchronize(ctx->stream));
        ctx->profiling = on != 0;
        for (auto& p : ctx->prof) {
            p.used = 0;
            p.launches = 0;
        }
    });
}

zi_status zi_ctx_set_sort_policy(zi_ctx* ctx, int32_t dims, int32_t policy) {
    return guard(ctx, [&] {
        require(ctx != nullptr, "null argument");
        require(dims >= 1 && dims <= 32, "sort policy: dims must be in [1, 32]");
        require(policy >= -1 && policy <= dims - 3, "sort policy: -1, 0 or an MSD depth in [1, dims - 3]");
        ctx->sort_depth[dims][1] = policy;
    });
}

zi_status zi_ctx_set_profile_filter(zi_ctx* ctx, const char* names) {
    return guard(ctx, [&] {
        require(ctx != nullptr, "null argument");
        ctx->prof_filter.clear();
        if (!names) return;
        std::string cur;
        for (const char* c = names;; ++c) {
            if (*c == ',' || *c == 0) {
                if (!cur.empty()) ctx->prof_filter.push_back(cur);
                cur.clear();
                if (*c == 0) break;
            } else {
                cur += *c;
            }
        }
    });
}

zi_status zi_ctx_profile(const zi_ctx* ctx, int slot, double* ms, uint64_t* launches, const char** name) {
    return guard(ctx, [&] {
        require(slot >= 0 && static_cast<size_t>(slot) < ctx->prof.size(), "profile slot out of range");
        ZI_CUDA(cudaStreamSynchronize(ctx->stream));
        const auto& p = ctx->prof[slot];
        double total = 0.0;
        for (size_t i = 0; i < p.used; ++i) {
            float f = 0.f;
            ZI_CUDA(cudaEventElapsedTime(&f, p.events[i].first, p.events[i].second));
            total += f;
        }
        if (ms) *ms = total;
        if (launches) *launches = p.launches;
        if (name) *name = p.name;
    });
}

int zi_less_most_significant_bit(int a, int b) {
    const uint8_t ua = static_cast<uint8_t>(a), ub = static_cast<uint8_t>(b);
    return (ua < ub) && (ua < (ua ^ ub));
}

int zi_morton_less(const uint8_t* a, const uint8_t* b, uint32_t dims) {
    uint8_t best_diff = 0;
    uint32_t best_dim = 0;
    for (uint32_t d = 0; d < dims; ++d) {
        const uint8_t diff = static_cast<uint8_t>(a[d] ^ b[d]);
        if (zi_less_most_significant_bit(best_diff, diff)) {
            best_diff = diff;
            best_dim = d;
        }
    }
    return dims ? a[best_dim] < b[best_dim] : 0;
}

int zi_subset_pixel_count(int patch_size, double coverage) { return zi::subset_pixel_count(patch_size, coverage); }

zi_status zi_subset_layouts(int patch_size, double coverage, int32_t* rc_out, int32_t* m_out) {
    return guard([&] {
        std::vector<int32_t> rc;
        const int m = zi::subset_layouts(patch_size, coverage, rc);
        if (rc_out) std::memcpy(rc_out, rc.data(), rc.size() * sizeof(int32_t));
        if (m_out) *m_out = m;
    });
}

zi_status zi_subset_layout_anchors(int patch_size, int32_t* rc_out) {
    return guard([&] {
        require(rc_out != nullptr, "null argument");
        if (patch_size < 3 || patch_size % 2 == 0) throw zi::error(ZI_E_INVALID, "subset layouts: K must be odd and >= 3");
        zi::layout_anchors(patch_size, rc_out);
    });
}

void zi_index_config_default(zi_index_config* c) {
    c->patch_size = 9;
    c->coverage = 0.6;
    c->dims = 10;
    c->knn = 80;
    c->mu = 256;
    c->nu = 2048;
    c->norm = ZI_NORM_L2;
}

zi_status zi_index_config_validate(const zi_index_config* cfg, int channels) {
    return guard([&] { zi::validate_config(*cfg, channels); });
}

// ---------------------------------------------------------------- z-curve index
zi_status zi_index_from_descriptors(zi_ctx* ctx, const uint8_t* coords, const uint32_t* keys, uint64_t n, uint32_t dims,
                                    uint32_t layout_id, zi_index** out) {
    return guard(ctx, [&] {
        require(ctx && out, "null argument");
        if (dims == 0 || dims > 32) throw zi::error(ZI_E_INVALID, "zcurve_index: dims must be in [1, 32]");
        require(n == 0 || (coords && keys), "null argument");
        auto* idx = new zi_index();
        idx->ctx = ctx;
        idx->layout_id = layout_id;
        try {
            const int W = static_cast<int>((dims + 3) / 4);
            zi::dbuf<uint8_t> dc;
            zi::dbuf<uint32_t> recs;
            if (n) {
                dc.ensure(n * dims);
                recs.ensure(static_cast<size_t>(W + 1) * n + n);
                uint32_t* keys_in = recs.p + static_cast<size_t>(W + 1) * n;
                ZI_CUDA(cudaMemcpyAsync(dc.p, coords, n * dims, cudaMemcpyHostToDevice, ctx->stream));
                ZI_CUDA(cudaMemcpyAsync(keys_in, keys, n * sizeof(uint32_t), cudaMemcpyHostToDevice, ctx->stream));
                bool ascending = true;
                for (uint64_t i = 1; i < n && ascending; ++i) ascending = keys[i - 1] < keys[i];
                uint32_t* keyw = recs.p;
                uint32_t* val = recs.p + static_cast<size_t>(W) * n;
                zi::interleave_coords(ctx, dc.p, keys_in, n, static_cast<int>(dims), keyw, val);
                uint32_t* sorted[10];
                zi::morton_sort_records(ctx, keyw, val, n, 1, static_cast<int>(dims), false, sorted, ascending);
                zi::finalize_index(ctx, sorted[0], sorted[W], n, 0, n, static_cast<int>(dims), nullptr, idx);
                ZI_CUDA(cudaStreamSynchronize(ctx->stream));
            } else {
                zi::finalize_index(ctx, nullptr, nullptr, 0, 0, 0, static_cast<int>(dims), nullptr, idx);
            }
        } catch (...) {
            delete idx;
            throw;
        }
        *out = idx;
    });
}

zi_status zi_index_destroy(zi_index* idx) {
    return guard(idx ? idx->ctx : nullptr, [&] { delete idx; });
}

zi_status zi_index_size(const zi_index* idx, uint64_t* n, uint32_t* dims) {
    return guard(idx ? idx->ctx : nullptr, [&] {
        if (n) *n = idx->n;
        if (dims) *dims = idx->dims;
    });
}

static void export_index(zi_index* idx, uint8_t* coords_out, uint32_t* keys_out) {
    zi_ctx* ctx = idx->ctx;
    const uint64_t n = idx->n;
    if (n == 0) return;
    if (keys_out) ZI_CUDA(cudaMemcpyAsync(keys_out, idx->keys.p, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
    if (coords_out) {
        std::vector<uint32_t> planes(static_cast<size_t>(idx->planes_n) * n);
        ZI_CUDA(cudaMemcpyAsync(planes.data(), idx->planes.p, planes.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                                ctx->stream));
        ZI_CUDA(cudaStreamSynchronize(ctx->stream));
        const uint32_t D = idx->dims;
        for (uint64_t i = 0; i < n; ++i)
            for (uint32_t d = 0; d < D; ++d)
                coords_out[i * D + d] = static_cast<uint8_t>((planes[static_cast<size_t>(d >> 2) * n + i] >> ((d & 3) * 8)) & 0xff);
    }
    ZI_CUDA(cudaStreamSynchronize(ctx->stream));
}

zi_status zi_index_export(zi_index* idx, uint8_t* coords_out, uint32_t* keys_out) {
    return guard(idx ? idx->ctx : nullptr, [&] { export_index(idx, coords_out, keys_out); });
}

zi_status zi_knn_search(zi_index* idx, const uint8_t* query, uint32_t k, uint32_t mu, int32_t norm, uint64_t* packed_out,
                        uint32_t* count_out) {
    return guard(idx ? idx->ctx : nullptr, [&] {
        require(idx && query && packed_out && count_out, "null argument");
        require(norm == ZI_NORM_L2 || norm == ZI_NORM_L1, "norm must be l2 or l1");
        (void)mu;  // leaf threshold of the CPU traversal; the GPU scan has no leaves
        *count_out = zi::knn_search(idx, query, k, norm, packed_out);
    });
}

zi_status zi_knn_search_batch(zi_index* idx, const uint8_t* queries, uint64_t nq, uint32_t k, int32_t norm,
                              uint64_t* packed_out, uint32_t* counts_out) {
    return guard(idx ? idx->ctx : nullptr, [&] {
        require(idx && (nq == 0 || (queries && packed_out && counts_out)), "null argument");
        require(norm == ZI_NORM_L2 || norm == ZI_NORM_L1, "norm must be l2 or l1");
        zi::knn_search_batch(idx, queries, nq, k, norm, packed_out, counts_out);
    });
}

zi_status zi_knn_batch_bench(zi_index* idx, const uint8_t* queries, uint64_t nq, uint32_t k, int32_t norm, int32_t reps,
                             double* ms_per_batch, uint64_t* stats3, uint64_t* packed_out, uint32_t* counts_out) {
    return guard(idx ? idx->ctx : nullptr, [&] {
        require(idx && queries && ms_per_batch && nq > 0 && reps > 0, "bad argument");
        require(norm == ZI_NORM_L2 || norm == ZI_NORM_L1, "norm must be l2 or l1");
        require(k >= 1 && k <= 256, "batch bench supports 1 <= k <= 256");
        zi_ctx* ctx = idx->ctx;
        zi::dbuf<uint8_t> dq;
        zi::dbuf<unsigned long long> dout, dstats;
        zi::dbuf<uint32_t> dcnt;
        dq.ensure(nq * idx->dims);
        dout.ensure(nq * k);
        dcnt.ensure(nq);
        dstats.ensure(4);
        ZI_CUDA(cudaMemcpyAsync(dq.p, queries, nq * idx->dims, cudaMemcpyHostToDevice, ctx->stream));
        zi::knn_batch_device(ctx, idx, dq.p, nq, k, norm, dout.p, dcnt.p, nullptr);  // warm-up
        ZI_CUDA(cudaMemsetAsync(dstats.p, 0, 4 * sizeof(unsigned long long), ctx->stream));
        cudaEvent_t e0, e1;
        ZI_CUDA(cudaEventCreate(&e0));
        ZI_CUDA(cudaEventCreate(&e1));
        float total = 0.f;
        for (int r = 0; r < reps; ++r) {
            ZI_CUDA(cudaEventRecord(e0, ctx->stream));
            zi::knn_batch_device(ctx, idx, dq.p, nq, k, norm, dout.p, dcnt.p, r == 0 ? dstats.p : nullptr);
            ZI_CUDA(cudaEventRecord(e1, ctx->stream));
            ZI_CUDA(cudaEventSynchronize(e1));
            float ms = 0.f;
            ZI_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            total += ms;
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        *ms_per_batch = total / reps;
        if (stats3)
            ZI_CUDA(cudaMemcpyAsync(stats3, dstats.p, 3 * sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
        if (packed_out)
            ZI_CUDA(cudaMemcpyAsync(packed_out, dout.p, nq * k * sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
        if (counts_out)
            ZI_CUDA(cudaMemcpyAsync(counts_out, dcnt.p, nq * sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
        ZI_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// ---------------------------------------------------------------- dictionary
zi_status zi_dictionary_collect(zi_ctx* ctx, const uint8_t* known, int32_t w, int32_t h, int32_t K, uint32_t* keys_out,
                                uint64_t cap, uint64_t* n_out) {
    return guard(ctx, [&] {
        require(ctx && known && n_out, "null argument");
        require(w > 0 && h > 0 && w <= 65535 && h <= 65535, "mask_image: bad dimensions");
        require(K >= 1, "patch size must be positive");
        zi::dbuf<uint8_t> dk;
        zi::dbuf<uint32_t> keys;
        dk.ensure(static_cast<size_t>(w) * h);
        ZI_CUDA(cudaMemcpyAsync(dk.p, known, static_cast<size_t>(w) * h, cudaMemcpyHostToDevice, ctx->stream));
        const uint64_t n = zi::collect_dictionary(ctx, dk.p, w, h, K, keys);
        *n_out = n;
        if (n == 0) throw zi::error(ZI_E_EMPTY_DICT, "no fully known patch window; inpainting impossible");
        if (keys_out) {
            require(cap >= n, "keys_out capacity below the dictionary size");
            ZI_CUDA(cudaMemcpyAsync(keys_out, keys.p, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
        }
        ZI_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// ---------------------------------------------------------------- multi-index
zi_status zi_multi_index_build(zi_ctx* ctx, const uint8_t* image, const uint8_t* known, int32_t w, int32_t h,
                               int32_t C, const zi_index_config* cfg, zi_multi_index** out) {
    return guard(ctx, [&] {
        require(out != nullptr, "null argument");
        zi_multi_index* mi = new_multi_index(ctx, image, known, w, h, C, cfg);
        try {
            zi::build_multi_index(mi);
        } catch (...) {
            delete mi;
            throw;
        }
        *out = mi;
    });
}

zi_status zi_multi_index_build_to(zi_ctx* ctx, const uint8_t* image, const uint8_t* known, int32_t w, int32_t h,
                                  int32_t C, const zi_index_config* cfg, uint32_t* keys_out, uint64_t keys_cap,
                                  uint64_t* n_out, zi_multi_index** out) {
    return guard(ctx, [&] {
        require(out != nullptr && keys_out != nullptr && n_out != nullptr, "null argument");
        zi_multi_index* mi = new_multi_index(ctx, image, known, w, h, C, cfg, true);
        try {
            mi->dict_out = keys_out;
            mi->dict_cap = keys_cap;
            zi::build_multi_index(mi);
            ZI_CUDA(cudaStreamSynchronize(ctx->stream));  // the kernels and (ev_copy) the dictionary copy
            mi->dict_out = nullptr;
            mi->image_on_copy = false;
        } catch (...) {
            cudaStreamSynchronize(ctx->copy_stream);  // no copy may still target the caller's buffers
            delete mi;
            throw;
        }
        *n_out = mi->n;
        *out = mi;
    });
}

// ---------------------------------------------------------------- one layout (build_index)
zi_status zi_index_build(zi_ctx* ctx, const uint8_t* image, int32_t w, int32_t h, int32_t C, const uint32_t* keys,
                         uint64_t n, const int32_t* layout_rc, int32_t m, const zi_index_config* cfg,
                         zi_patch_index** out) {
    return guard(ctx, [&] {
        require(ctx && image && keys && layout_rc && cfg && out, "null argument");
        require(w > 0 && h > 0 && (C == 1 || C == 3), "raster_image: bad dimensions");
        require(w <= 65535 && h <= 65535, "image side above the 16-bit patch_key range");
        zi::validate_config(*cfg, C);
        if (n == 0) throw zi::error(ZI_E_EMPTY_DICT, "build_index: empty dictionary");
        require(n < (1ull << 29), "build_index: dictionary above 2^29 patches");
        const int K = cfg->patch_size;
        require(m >= 1 && m <= K * K, "build_index: layout pixel count out of range");
        for (int p = 0; p < m; ++p)
            require(layout_rc[2 * p] >= 0 && layout_rc[2 * p] < K && layout_rc[2 * p + 1] >= 0 &&
                        layout_rc[2 * p + 1] < K,
                    "build_index: layout offset outside the patch");
        for (uint64_t i = 0; i < n; ++i) {
            const uint32_t x = keys[i] & 0xffffu, y = keys[i] >> 16;
            require(x + K <= static_cast<uint32_t>(w) && y + K <= static_cast<uint32_t>(h),
                    "build_index: dictionary window outside the image");
        }
        auto* pi = new zi_patch_index();
        try {
            pi->ctx = ctx;
            pi->cfg = *cfg;
            pi->w = w;
            pi->h = h;
            pi->C = C;
            pi->K = K;
            pi->m = m;
            pi->mc = m * C;
            pi->n = n;
            pi->rc.assign(layout_rc, layout_rc + 2 * m);
            std::vector<int32_t> off(m), loc(m), cols;
            for (int p = 0; p < m; ++p) {
                const int r = layout_rc[2 * p], c = layout_rc[2 * p + 1];
                off[p] = (r * w + c) * C;
                loc[p] = r * K + c;
                for (int ch = 0; ch < C; ++ch) cols.push_back((r * K + c) * C + ch);
            }
            const size_t npx = static_cast<size_t>(w) * h;
            pi->image.ensure(npx * C + 16);
            pi->dict.ensure(n);
            pi->off.ensure(m);
            pi->local.ensure(m);
            pi->cols.ensure(cols.size());
            ZI_CUDA(cudaMemcpyAsync(pi->image.p, image, npx * C, cudaMemcpyHostToDevice, ctx->stream));
            ZI_CUDA(cudaMemcpyAsync(pi->dict.p, keys, n * sizeof(uint32_t), cudaMemcpyHostToDevice, ctx->stream));
            ZI_CUDA(cudaMemcpyAsync(pi->off.p, off.data(), m * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
            ZI_CUDA(cudaMemcpyAsync(pi->local.p, loc.data(), m * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
            ZI_CUDA(cudaMemcpyAsync(pi->cols.p, cols.data(), cols.size() * sizeof(int32_t), cudaMemcpyHostToDevice,
                                    ctx->stream));
            ZI_CUDA(cudaStreamSynchronize(ctx->stream));  // pageable sources
            zi::build_patch_index(pi);
        } catch (...) {
            delete pi;
            throw;
        }
        *out = pi;
    });
}

zi_status zi_patch_index_destroy(zi_patch_index* pi) {
    return guard(pi ? pi->ctx : nullptr, [&] { delete pi; });
}

zi_status zi_patch_index_model(const zi_patch_index* pi, int32_t* dims, int32_t* mc, double* mean, double* components,
                               double* eigenvalues, double* lo, double* hi, double* build_seconds,
                               double* sort_seconds) {
    return guard(pi ? pi->ctx : nullptr, [&] {
        require(pi != nullptr, "null argument");
        if (dims) *dims = pi->dims;
        if (mc) *mc = pi->mc;
        auto put = [](double* dst, const std::vector<double>& v) {
            if (dst) std::memcpy(dst, v.data(), v.size() * sizeof(double));
        };
        put(mean, pi->h_mean);
        put(components, pi->h_comp);
        put(eigenvalues, pi->h_eig);
        put(lo, pi->h_lo);
        put(hi, pi->h_hi);
        if (build_seconds) *build_seconds = pi->build_ms * 1e-3;
        if (sort_seconds) *sort_seconds = pi->sort_ms * 1e-3;
    });
}

zi_status zi_patch_index_get_index(zi_patch_index* pi, zi_index** out) {
    return guard(pi ? pi->ctx : nullptr, [&] {
        require(pi && out, "null argument");
        *out = &pi->index;
    });
}

zi_status zi_make_query(zi_patch_index* pi, const uint8_t* target_values, const uint8_t* target_known, uint8_t* out) {
    return guard(pi ? pi->ctx : nullptr, [&] {
        require(pi && target_values && target_known && out, "null argument");
        zi::make_query(pi->ctx, target_values, target_known, pi->K, pi->C, pi->local.p, pi->m, pi->mean.p, pi->comp.p,
                       pi->minmax.p, pi->dims, out, pi->qbuf, pi->hstage);
    });
}

zi_status zi_multi_index_make_query(zi_multi_index* mi, int32_t layout, const uint8_t* target_values,
                                    const uint8_t* target_known, uint8_t* out) {
    return guard(mi ? mi->ctx : nullptr, [&] {
        require(mi && target_values && target_known && out, "null argument");
        require(layout >= 0 && layout < 8, "layout id out of range");
        require(mi->n > 0, "empty multi-index");
        const size_t mc = static_cast<size_t>(mi->mc), D = static_cast<size_t>(mi->dims);
        zi::make_query(mi->ctx, target_values, target_known, mi->K, mi->C, mi->layout_local.p + layout * mi->m, mi->m,
                       mi->pca_mean.p + layout * mc, mi->pca_comp.p + layout * mc * D, mi->minmax.p + layout * 2 * D,
                       mi->dims, out, mi->qscratch, mi->hstage);
        mi->qws_clean = false;
    });
}

zi_status zi_brute_force_scan(zi_ctx* ctx, const uint8_t* image, int32_t w, int32_t h, int32_t C, const uint32_t* keys,
                              uint64_t n, const uint8_t* target_values, const uint8_t* target_known, int32_t K,
                              int32_t norm, zi_best_patch* out) {
    return guard(ctx, [&] {
        require(ctx && image && target_values && target_known && out && (n == 0 || keys), "null argument");
        require(w > 0 && h > 0 && (C == 1 || C == 3), "raster_image: bad dimensions");
        require(K >= 1 && K <= 255, "patch size out of range");
        require(norm == ZI_NORM_L2 || norm == ZI_NORM_L1, "norm must be l2 or l1");
        for (uint64_t i = 0; i < n; ++i) {
            const uint32_t x = keys[i] & 0xffffu, y = keys[i] >> 16;
            require(x + K <= static_cast<uint32_t>(w) && y + K <= static_cast<uint32_t>(h),
                    "brute_force_best: dictionary window outside the image");
        }
        const size_t npx = static_cast<size_t>(w) * h;
        zi::dbuf<uint8_t> dimg, scratch;
        zi::dbuf<uint32_t> ddict;
        zi::hbuf<uint8_t> stage;
        dimg.ensure(npx * C + 16);
        ddict.ensure(n ? n : 1);
        ZI_CUDA(cudaMemcpyAsync(dimg.p, image, npx * C, cudaMemcpyHostToDevice, ctx->stream));
        if (n) ZI_CUDA(cudaMemcpyAsync(ddict.p, keys, n * sizeof(uint32_t), cudaMemcpyHostToDevice, ctx->stream));
        const uint64_t best =
            zi::brute_force_scan(ctx, dimg.p, w, C, K, ddict.p, n, target_values, target_known, norm, scratch, stage);
        out->key = static_cast<uint32_t>(best & 0xffffffffu);
        out->cost = static_cast<uint32_t>(best >> 32);
        out->error = norm == ZI_NORM_L2 ? std::sqrt(static_cast<double>(out->cost)) : static_cast<double>(out->cost);
        out->layout_id = 0;
        out->candidates = n;
        if (n == 0) {
            out->key = 0;
            out->cost = 0xffffffffu;
        }
    });
}

// ---------------------------------------------------------------- vector index (cfg5)
static zi_status vector_build(zi_ctx* ctx, const float* X, bool device_rows, uint64_t n, int32_t dim, int32_t dims,
                              zi_vector_index** out) {
    return guard(ctx, [&] {
        require(ctx && X && out, "null argument");
        require(n > 0, "vector index: empty input");
        require(dim >= 3 && dim <= 224, "vector index: dim must be in [3, 224]");
        require(dims >= 1 && dims <= 32, "vector index: dims must be in [1, 32]");
        require(n < (1ull << 29), "vector index: more than 2^29 rows");
        auto* vi = new zi_vector_index();
        vi->ctx = ctx;
        vi->n = n;
        vi->dim = dim;
        vi->dims = static_cast<int>(std::min<uint64_t>(static_cast<uint64_t>(dims), std::min<uint64_t>(dim, n)));
        try {
            cudaEvent_t e0, e1;
            ZI_CUDA(cudaEventCreate(&e0));
            ZI_CUDA(cudaEventCreate(&e1));
            if (device_rows) {
                vi->Xd = X;  // caller's device buffer: must outlive the build only
            } else {
                vi->X.ensure(n * dim);
                ZI_CUDA(cudaMemcpyAsync(vi->X.p, X, n * dim * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
                vi->Xd = vi->X.p;
            }
            ZI_CUDA(cudaEventRecord(e0, ctx->stream));
            zi::build_vector_index_device(vi);
            ZI_CUDA(cudaEventRecord(e1, ctx->stream));
            ZI_CUDA(cudaEventSynchronize(e1));
            float ms = 0.f;
            ZI_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            vi->build_ms = ms;
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
        } catch (...) {
            delete vi;
            throw;
        }
        *out = vi;
    });
}

zi_status zi_vector_index_build(zi_ctx* ctx, const float* X, uint64_t n, int32_t dim, int32_t dims,
                                zi_vector_index** out) {
    return vector_build(ctx, X, false, n, dim, dims, out);
}

zi_status zi_vector_index_build_device(zi_ctx* ctx, const float* d_X, uint64_t n, int32_t dim, int32_t dims,
                                       zi_vector_index** out) {
    return vector_build(ctx, d_X, true, n, dim, dims, out);
}

zi_status zi_vector_index_destroy(zi_vector_index* vi) {
    return guard(vi ? vi->ctx : nullptr, [&] { delete vi; });
}

zi_status zi_vector_index_model(zi_vector_index* vi, int32_t* dims, double* mean, double* components,
                                double* eigenvalues, double* lo, double* hi, double* build_ms) {
    return guard(vi ? vi->ctx : nullptr, [&] {
        require(vi != nullptr, "null argument");
        zi::vector_sync_host_model(vi);
        if (dims) *dims = vi->dims;
        if (mean) std::memcpy(mean, vi->h_mean.data(), vi->h_mean.size() * sizeof(double));
        if (components) std::memcpy(components, vi->h_comp.data(), vi->h_comp.size() * sizeof(double));
        if (eigenvalues) std::memcpy(eigenvalues, vi->h_eig.data(), vi->h_eig.size() * sizeof(double));
        if (lo) std::memcpy(lo, vi->h_lo.data(), vi->h_lo.size() * sizeof(double));
        if (hi) std::memcpy(hi, vi->h_hi.data(), vi->h_hi.size() * sizeof(double));
        if (build_ms) *build_ms = vi->build_ms;
    });
}

zi_status zi_vector_index_get_index(zi_vector_index* vi, zi_index** out) {
    return guard(vi ? vi->ctx : nullptr, [&] {
        require(vi && out, "null argument");
        *out = &vi->index;
    });
}

static uint8_t* vector_queries_to_device(zi_vector_index* vi, const float* Q, const uint8_t* known, uint64_t nq) {
    zi_ctx* ctx = vi->ctx;
    const size_t qb = nq * vi->dim * sizeof(float), kb = nq * vi->dim, ob = nq * vi->dims;
    uint8_t* b = vi->qbuf.ensure(qb + kb + ob + 64);
    ZI_CUDA(cudaMemcpyAsync(b, Q, qb, cudaMemcpyHostToDevice, ctx->stream));
    ZI_CUDA(cudaMemcpyAsync(b + qb, known, kb, cudaMemcpyHostToDevice, ctx->stream));
    zi::vector_make_queries(vi, reinterpret_cast<const float*>(b), b + qb, nq, b + qb + kb);
    return b + qb + kb;
}

zi_status zi_vector_make_queries(zi_vector_index* vi, const float* queries, const uint8_t* known, uint64_t nq,
                                 uint8_t* descriptors_out) {
    return guard(vi ? vi->ctx : nullptr, [&] {
        require(vi && (nq == 0 || (queries && known && descriptors_out)), "null argument");
        if (nq == 0) return;
        const uint8_t* d = vector_queries_to_device(vi, queries, known, nq);
        ZI_CUDA(cudaMemcpyAsync(descriptors_out, d, nq * vi->dims, cudaMemcpyDeviceToHost, vi->ctx->stream));
        ZI_CUDA(cudaStreamSynchronize(vi->ctx->stream));
    });
}

zi_status zi_vector_knn_batch(zi_vector_index* vi, const float* queries, const uint8_t* known, uint64_t nq,
                              uint32_t k, int32_t norm, uint64_t* packed_out, uint32_t* counts_out) {
    return guard(vi ? vi->ctx : nullptr, [&] {
        require(vi && (nq == 0 || (queries && known && packed_out && counts_out)), "null argument");
        require(norm == ZI_NORM_L2 || norm == ZI_NORM_L1, "norm must be l2 or l1");
        if (nq == 0) return;
        const uint8_t* d = vector_queries_to_device(vi, queries, known, nq);
        std::vector<uint8_t> h(nq * vi->dims);
        ZI_CUDA(cudaMemcpyAsync(h.data(), d, h.size(), cudaMemcpyDeviceToHost, vi->ctx->stream));
        ZI_CUDA(cudaStreamSynchronize(vi->ctx->stream));
        zi::knn_search_batch(&vi->index, h.data(), nq, k, norm, packed_out, counts_out);
    });
}

zi_status zi_multi_index_save(zi_multi_index* mi, const char* path) {
    return guard(mi ? mi->ctx : nullptr, [&] {
        require(mi && path, "null argument");
        require(!mi->shard, "ZIDX1 holds whole layout indices; save the unsharded multi_index");
        zi::save_multi_index(mi, path);
    });
}

zi_status zi_multi_index_load(zi_ctx* ctx, const char* path, const uint8_t* image, int32_t w, int32_t h, int32_t C,
                              zi_multi_index** out) {
    return guard(ctx, [&] {
        require(ctx && path && image && out, "null argument");
        require(w > 0 && h > 0 && (C == 1 || C == 3), "raster_image: bad dimensions");
        require(w <= 65535 && h <= 65535, "image side above the 16-bit patch_key range");
        const zi::zidx_header hd = zi::zidx_peek(path);
        zi_index_config cfg;
        zi_index_config_default(&cfg);
        cfg.patch_size = hd.K;
        cfg.coverage = hd.coverage;
        cfg.dims = hd.D;
        std::vector<uint8_t> known(static_cast<size_t>(w) * h, 1);  // the mask is not part of an index
        zi_multi_index* mi = new_multi_index(ctx, image, known.data(), w, h, C, &cfg);
        try {
            zi::load_multi_index_into(mi, path);
        } catch (...) {
            delete mi;
            throw;
        }
        *out = mi;
    });
}

zi_status zi_multi_index_rebuild(zi_multi_index* mi) {
    return guard(mi ? mi->ctx : nullptr, [&] {
        require(mi && !mi->loaded, "rebuild needs the build inputs; this index was loaded from a file");
        require(!mi->shard, "a shard is built by the zi_shard_* stages");
        zi::build_multi_index(mi);
    });
}

zi_status zi_multi_index_destroy(zi_multi_index* mi) {
    return guard(mi ? mi->ctx : nullptr, [&] {
        if (!mi) return;
        cudaStreamSynchronize(mi->ctx->stream);
        if (mi->ev0) cudaEventDestroy(mi->ev0);
        if (mi->ev1) cudaEventDestroy(mi->ev1);
        if (mi->hres) cudaFreeHost(mi->hres);
        delete mi;
    });
}

zi_status zi_multi_index_get_info(const zi_multi_index* mi, zi_multi_index_info* info) {
    return guard(mi ? mi->ctx : nullptr, [&] {
        info->n = mi->n;
        info->dims = mi->dims;
        info->m = mi->m;
        info->channels = mi->C;
        info->patch_size = mi->K;
        info->width = mi->w;
        info->height = mi->h;
        zi::finish_build_timing(const_cast<zi_multi_index*>(mi));
        info->build_seconds = mi->build_ms * 1e-3;
        info->eigen_seconds = mi->eigen_s;
        info->pca_on_device = mi->device_pca ? 1 : 0;
        info->coverage = mi->cfg.coverage;
        info->loaded = mi->loaded ? 1 : 0;
    });
}

zi_status zi_multi_index_dictionary(zi_multi_index* mi, uint32_t* keys_out) {
    return guard(mi ? mi->ctx : nullptr, [&] {
        ZI_CUDA(cudaMemcpyAsync(keys_out, mi->dict.p + mi->row_begin, mi->n * sizeof(uint32_t), cudaMemcpyDeviceToHost, mi->ctx->stream));
        ZI_CUDA(cudaStreamSynchronize(mi->ctx->stream));
    });
}

zi_status zi_multi_index_layout(zi_multi_index* mi, int32_t layout, int32_t* rc, double* mean, double* components,
                                double* eigenvalues, double* lo, double* hi) {
    return guard(mi ? mi->ctx : nullptr, [&] {
        require(layout >= 0 && layout < 8, "layout id must be in [0, 8)");
        zi::sync_host_model(mi);
        const auto& L = mi->L[layout];
        if (rc) std::memcpy(rc, L.rc.data(), L.rc.size() * sizeof(int32_t));
        if (mean) std::memcpy(mean, L.mean.data(), L.mean.size() * sizeof(double));
        if (components) std::memcpy(components, L.comp.data(), L.comp.size() * sizeof(double));
        if (eigenvalues) std::memcpy(eigenvalues, L.eig.data(), L.eig.size() * sizeof(double));
        if (lo) std::memcpy(lo, L.lo.data(), L.lo.size() * sizeof(double));
        if (hi) std::memcpy(hi, L.hi.data(), L.hi.size() * sizeof(double));
    });
}

zi_status zi_multi_index_layout_index(zi_multi_index* mi, int32_t layout, uint8_t* coords_out, uint32_t* keys_out) {
    return guard(mi ? mi->ctx : nullptr, [&] {
        require(layout >= 0 && layout < 8, "layout id must be in [0, 8)");
        export_index(&mi->L[layout].index, coords_out, keys_out);
    });
}

zi_status zi_multi_index_get_index(zi_multi_index* mi, int32_t layout, zi_index** out) {
    return guard(mi ? mi->ctx : nullptr, [&] {
        require(layout >= 0 && layout < 8, "layout id must be in [0, 8)");
        *out = &mi->L[layout].index;
    });
}

zi_status zi_multi_index_moments(zi_multi_index* mi, int64_t* s_out, int64_t* S_out) {
    return guard(mi ? mi->ctx : nullptr, [&] {
        require(!mi->loaded, "patch moments are not stored in an index file");
        zi::sync_host_model(mi);
        if (s_out) std::memcpy(s_out, mi->s.data(), mi->s.size() * sizeof(int64_t));
        if (S_out) std::memcpy(S_out, mi->S.data(), mi->S.size() * sizeof(int64_t));
    });
}

// ---------------------------------------------------------------- query
zi_status zi_query_best_patch(zi_multi_index* mi, const uint8_t* tv, const uint8_t* tk, uint32_t k, int32_t norm,
                              zi_best_patch* out, uint64_t* knn_out) {
    return guard(mi ? mi->ctx : nullptr, [&] {
        require(mi && tv && tk && out, "null argument");
        require(norm == ZI_NORM_L2 || norm == ZI_NORM_L1, "norm must be l2 or l1");
        const zi::query_result r = zi::query_best_patch(mi, tv, tk, k, norm, knn_out);
        out->key = static_cast<uint32_t>(r.best & 0xffffffffu);
        out->cost = static_cast<uint32_t>(r.best >> 32);
        out->error = norm == ZI_NORM_L2 ? std::sqrt(static_cast<double>(out->cost)) : static_cast<double>(out->cost);
        out->layout_id = r.lid;
        out->candidates = r.count;
    });
}

zi_status zi_brute_force_best(zi_multi_index* mi, const uint8_t* tv, const uint8_t* tk, int32_t norm, zi_best_patch* out) {
    return guard(mi ? mi->ctx : nullptr, [&] {
        require(mi && tv && tk && out, "null argument");
        require(norm == ZI_NORM_L2 || norm == ZI_NORM_L1, "norm must be l2 or l1");
        const uint64_t b = zi::brute_force_best(mi, tv, tk, norm);
        out->key = static_cast<uint32_t>(b & 0xffffffffu);
        out->cost = static_cast<uint32_t>(b >> 32);
        out->error = norm == ZI_NORM_L2 ? std::sqrt(static_cast<double>(out->cost)) : static_cast<double>(out->cost);
        out->layout_id = 0;
        out->candidates = mi->n;
    });
}

zi_status zi_refine_best(zi_multi_index* mi, const uint8_t* tv, const uint8_t* tk, const uint64_t* cands, uint32_t count,
                         int32_t norm, zi_best_patch* out) {
    return guard(mi ? mi->ctx : nullptr, [&] {
        require(mi && tv && tk && out && (cands || count == 0), "null argument");
        require(norm == ZI_NORM_L2 || norm == ZI_NORM_L1, "norm must be l2 or l1");
        const uint64_t b = zi::refine_candidates(mi, tv, tk, cands, count, norm);
        out->key = static_cast<uint32_t>(b & 0xffffffffu);
        out->cost = static_cast<uint32_t>(b >> 32);
        out->error = norm == ZI_NORM_L2 ? std::sqrt(static_cast<double>(out->cost)) : static_cast<double>(out->cost);
        out->layout_id = 0;
        out->candidates = count;
    });
}

// ---------------------------------------------------------------- range-partitioned shards
zi_status zi_shard_create(zi_ctx* ctx, const uint8_t* image, const uint8_t* known, int32_t w, int32_t h, int32_t C,
                          const zi_index_config* cfg, int32_t rank, int32_t world, zi_shard** out) {
    return guard(ctx, [&] {
        require(out != nullptr, "null argument");
        require(world >= 1 && world <= 64 && rank >= 0 && rank < world, "shard: rank / world out of range");
        zi_multi_index* mi = new_multi_index(ctx, image, known, w, h, C, cfg);
        try {
            *out = zi::shard_create(mi, rank, world);
        } catch (...) {
            delete mi;
            throw;
        }
    });
}

zi_status zi_shard_rebuild(zi_shard* sh) {
    if (!sh) return fail(ZI_E_INVALID, "null argument");
    return guard(zi::shard_multi_index(sh)->ctx, [&] { zi::shard_rebuild(sh); });
}

zi_status zi_shard_finish_local(zi_shard* sh) {
    if (!sh) return fail(ZI_E_INVALID, "null argument");
    return guard(zi::shard_multi_index(sh)->ctx, [&] { zi::shard_finish_local(sh); });
}

zi_status zi_shard_destroy(zi_shard* sh) {
    if (!sh) return ZI_OK;
    zi_multi_index* mi = zi::shard_multi_index(sh);
    return guard(mi->ctx, [&] {
        zi::shard_destroy(sh);
        zi_multi_index_destroy(mi);
    });
}

zi_status zi_shard_info(const zi_shard* sh, uint64_t* info) {
    return guard([&] {
        require(sh && info, "null argument");
        zi::shard_info(sh, info);
    });
}

zi_status zi_shard_moments(zi_shard* sh, int64_t* out) {
    return guard(sh ? zi::shard_multi_index(sh)->ctx : nullptr, [&] {
        require(sh && out, "null argument");
        zi::shard_moments(sh, out);
    });
}

zi_status zi_shard_fit_project(zi_shard* sh, const int64_t* moments, int64_t* lo, int64_t* hi) {
    return guard(sh ? zi::shard_multi_index(sh)->ctx : nullptr, [&] {
        require(sh && moments && lo && hi, "null argument");
        zi::shard_fit_project(sh, moments, lo, hi);
    });
}

zi_status zi_shard_refine_ranges(zi_shard* sh, const int64_t* lo, const int64_t* hi, int64_t* lo_out, int64_t* hi_out) {
    return guard(sh ? zi::shard_multi_index(sh)->ctx : nullptr, [&] {
        require(sh && lo && hi && lo_out && hi_out, "null argument");
        zi::shard_refine_ranges(sh, lo, hi, lo_out, hi_out);
    });
}

zi_status zi_shard_quantize_sort(zi_shard* sh, const int64_t* lo, const int64_t* hi, uint32_t S, uint32_t* samples) {
    return guard(sh ? zi::shard_multi_index(sh)->ctx : nullptr, [&] {
        require(sh && lo && hi && (samples || S == 0), "null argument");
        require(S <= 65536, "shard: at most 65536 samples per layout");
        zi::shard_quantize_sort(sh, lo, hi, S, samples);
    });
}

zi_status zi_shard_splitters(const uint32_t* samples, uint64_t count, int32_t words, int32_t world, uint32_t* out) {
    return guard([&] {
        require((samples || count == 0) && (out || world == 1), "null argument");
        require(words >= 1 && words <= 8 && world >= 1 && world <= 64, "shard: words / world out of range");
        zi::shard_splitters(samples, count, words, world, out);
    });
}

zi_status zi_shard_partition(zi_shard* sh, const uint32_t* splitters, uint64_t* counts, const uint32_t** d_send) {
    return guard(sh ? zi::shard_multi_index(sh)->ctx : nullptr, [&] {
        require(sh && counts && d_send, "null argument");
        zi::shard_partition(sh, splitters, counts, d_send);
    });
}

zi_status zi_shard_rebalance_plan(const uint64_t* all_counts, int32_t world, uint64_t n_total, int32_t me,
                                  uint64_t* send_counts, uint64_t* send_starts) {
    return guard([&] {
        require(all_counts && send_counts && send_starts, "null argument");
        require(world >= 1 && world <= 64 && me >= 0 && me < world, "shard: rank / world out of range");
        zi::shard_rebalance_plan(all_counts, world, n_total, me, send_counts, send_starts);
    });
}

zi_status zi_shard_receive(zi_shard* sh, const uint32_t* d_recv, const uint64_t* all_counts, uint64_t* counts2,
                           const uint32_t** d_send2) {
    return guard(sh ? zi::shard_multi_index(sh)->ctx : nullptr, [&] {
        require(sh && all_counts && counts2 && d_send2, "null argument");
        zi::shard_receive(sh, d_recv, all_counts, counts2, d_send2);
    });
}

zi_status zi_shard_finish(zi_shard* sh, const uint32_t* d_recv2, const uint64_t* all_counts2) {
    return guard(sh ? zi::shard_multi_index(sh)->ctx : nullptr, [&] {
        require(sh && all_counts2, "null argument");
        zi::shard_finish(sh, d_recv2, all_counts2);
    });
}

zi_status zi_shard_multi_index(zi_shard* sh, zi_multi_index** out) {
    return guard([&] {
        require(sh && out, "null argument");
        *out = zi::shard_multi_index(sh);
    });
}

// ---------------------------------------------------------------- inpaint
static void fill_stats_defaults(zi_run_stats* st) {
    std::memset(st, 0, sizeof(*st));
    st->mean_ae = std::numeric_limits<double>::quiet_NaN();
    st->confidence_low = 1.0;
}

zi_status zi_inpaint(zi_ctx* ctx, const uint8_t* image, const uint8_t* known, int32_t w, int32_t h, int32_t C,
                     const zi_index_config* cfg, const zi_inpaint_config* icfg, uint8_t* image_out,
                     zi_iteration_record* records, uint64_t cap, uint64_t* n_records, zi_run_stats* stats) {
    return guard(ctx, [&] {
        require(ctx && image && known && cfg && icfg && image_out && n_records && stats, "null argument");
        require(w > 0 && h > 0 && (C == 1 || C == 3), "raster_image: bad dimensions");
        zi::validate_config(*cfg, C);
        fill_stats_defaults(stats);
        *n_records = 0;
        uint64_t unknown = 0;
        for (size_t i = 0; i < static_cast<size_t>(w) * h; ++i) unknown += known[i] == 0;
        if (unknown == 0) {  // engine.cpp:449-453
            std::memcpy(image_out, image, static_cast<size_t>(w) * h * C);
            return;
        }
        zi_multi_index* mi = new_multi_index(ctx, image, known, w, h, C, cfg);
        try {
            const auto t0 = std::chrono::steady_clock::now();
            if (icfg->brute_force) {  // dictionary only (engine.cpp:466-473)
                mi->n = zi::collect_dictionary(ctx, mi->known.p, w, h, mi->K, mi->dict);
                if (mi->n == 0) throw zi::error(ZI_E_EMPTY_DICT, "no fully known patch window; inpainting impossible");
            } else {
                zi::build_multi_index(mi);
            }
            stats->build_wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            stats->dictionary_size = mi->n;
            zi::run_inpaint(mi, image, known, *cfg, *icfg, image_out, records, cap, n_records, stats);
            stats->dictionary_size = mi->n;
        } catch (...) {
            delete mi;
            throw;
        }
        delete mi;
    });
}

zi_status zi_inpaint_with_index(zi_multi_index* mi, const uint8_t* image, const uint8_t* known,
                                const zi_index_config* cfg, const zi_inpaint_config* icfg, uint8_t* image_out,
                                zi_iteration_record* records, uint64_t cap, uint64_t* n_records, zi_run_stats* stats) {
    return guard(mi ? mi->ctx : nullptr, [&] {
        require(mi && image && known && cfg && icfg && image_out && n_records && stats, "null argument");
        require(!mi->shard, "the fill loop needs the whole index (sharding.ShardedMultiIndex.query_best_patch merges shards)");
        fill_stats_defaults(stats);
        *n_records = 0;
        uint64_t unknown = 0;
        for (size_t i = 0; i < static_cast<size_t>(mi->w) * mi->h; ++i) unknown += known[i] == 0;
        if (unknown == 0) {
            std::memcpy(image_out, image, static_cast<size_t>(mi->w) * mi->h * mi->C);
            return;
        }
        // query-side knobs from cfg; build-side parameters pinned by the index (engine.cpp:498-505)
        zi_index_config eff = *cfg;
        eff.patch_size = mi->cfg.patch_size;
        eff.coverage = mi->cfg.coverage;
        eff.dims = mi->cfg.dims;
        require(eff.norm == ZI_NORM_L2 || eff.norm == ZI_NORM_L1, "norm must be l2 or l1");
        ZI_CUDA(cudaMemcpyAsync(mi->image.p, image, static_cast<size_t>(mi->w) * mi->h * mi->C, cudaMemcpyHostToDevice,
                                mi->ctx->stream));
        stats->dictionary_size = mi->n;
        zi::run_inpaint(mi, image, known, eff, *icfg, image_out, records, cap, n_records, stats);
    });
}

}  // extern "C"
