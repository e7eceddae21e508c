// ref_shim.cpp -- C ABI over the reference's OWN compiled sources (TEST INFRASTRUCTURE ONLY).
//
// `make -C oracle ref` (oracle/Makefile) compiles this file together with the unmodified reference sources
//   /root/reference/proj/src/{zcurve,pool,layouts,image}.cpp
// (the Eigen-free part of the reference) into oracle/_ref/libzref.so.
// No reference source is copied into this repository; this shim only calls it.
#include <cstdint>
#include <cstring>
#include <memory>
#include <thread>
#include <vector>

#include "zinpaint/image.hpp"
#include "zinpaint/layouts.hpp"
#include "zinpaint/morton.hpp"
#include "zinpaint/pool.hpp"
#include "zinpaint/zcurve.hpp"

using namespace zinpaint;

namespace {
std::vector<patch_key> unpack_keys(const uint32_t* keys, int64_t n) {
    std::vector<patch_key> out(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i)
        out[i] = {static_cast<uint16_t>(keys[i] & 0xffff), static_cast<uint16_t>(keys[i] >> 16)};
    return out;
}
}  // namespace

extern "C" {

int zr_less_msb(int a, int b) {
    return less_most_significant_bit(static_cast<uint8_t>(a), static_cast<uint8_t>(b)) ? 1 : 0;
}

int zr_morton_less(const uint8_t* a, const uint8_t* b, int dims) {
    return morton_less(a, b, static_cast<size_t>(dims)) ? 1 : 0;
}

// build_subset_layouts (proj/src/layouts.cpp:13-60); rc_out 8*m*2; returns m
int zr_layouts(int K, double coverage, int* rc_out) {
    try {
        const auto layouts = build_subset_layouts(K, coverage);
        const int m = static_cast<int>(layouts[0].pixels.size());
        for (int l = 0; l < 8; ++l)
            for (int p = 0; p < m; ++p) {
                rc_out[(l * m + p) * 2] = layouts[l].pixels[p].first;
                rc_out[(l * m + p) * 2 + 1] = layouts[l].pixels[p].second;
            }
        return m;
    } catch (...) {
        return -1;
    }
}

// zcurve_index::from_descriptors (proj/src/zcurve.cpp:108-138)
void* zr_index_create(const uint8_t* coords, const uint32_t* keys, int64_t n, int dims) {
    try {
        std::vector<uint8_t> c(coords, coords + static_cast<size_t>(n) * dims);
        auto* idx = new zcurve_index(
            zcurve_index::from_descriptors(std::move(c), unpack_keys(keys, n), static_cast<uint32_t>(dims), 0));
        return idx;
    } catch (...) {
        return nullptr;
    }
}

void zr_index_free(void* h) { delete static_cast<zcurve_index*>(h); }

void zr_index_export(void* h, uint8_t* coords_out, uint32_t* keys_out) {
    const auto* idx = static_cast<zcurve_index*>(h);
    std::memcpy(coords_out, idx->coords().data(), idx->coords().size());
    for (size_t i = 0; i < idx->size(); ++i) keys_out[i] = idx->key_at(i).packed();
}

// knn_search (proj/src/zcurve.cpp:429-452); out packed (dist<<32|key) ascending; returns count
int64_t zr_index_knn(void* h, const uint8_t* query, int k, int mu, int nu, int norm, int workers,
                     uint64_t* out) {
    const auto* idx = static_cast<zcurve_index*>(h);
    search_params sp;
    sp.k = static_cast<uint32_t>(k);
    sp.mu = static_cast<uint32_t>(mu);
    sp.nu = static_cast<uint32_t>(nu);
    sp.norm = norm == 0 ? norm_kind::l2 : norm_kind::l1;
    std::unique_ptr<priority_pool> pool;
    if (workers > 1) {
        pool = std::make_unique<priority_pool>(static_cast<unsigned>(workers - 1));
        sp.pool = pool.get();
    }
    const auto found = knn_search(*idx, query, sp);
    for (size_t i = 0; i < found.size(); ++i) out[i] = pack_candidate(found[i].distance, found[i].key);
    return static_cast<int64_t>(found.size());
}

// batch of queries on one index, sequential traversal each (timing helper for the CPU arm)
int64_t zr_index_knn_batch(void* h, const uint8_t* queries, int64_t nq, int k, int mu, int nu, int norm,
                           int workers, uint64_t* out) {
    const auto* idx = static_cast<zcurve_index*>(h);
    search_params sp;
    sp.k = static_cast<uint32_t>(k);
    sp.mu = static_cast<uint32_t>(mu);
    sp.nu = static_cast<uint32_t>(nu);
    sp.norm = norm == 0 ? norm_kind::l2 : norm_kind::l1;
    std::unique_ptr<priority_pool> pool;
    if (workers > 1) {
        pool = std::make_unique<priority_pool>(static_cast<unsigned>(workers - 1));
        sp.pool = pool.get();
    }
    int64_t total = 0;
    knn_list list(sp.k);
    for (int64_t q = 0; q < nq; ++q) {
        knn_search(*idx, queries + q * idx->dims(), sp, list);
        const auto found = list.sorted();
        for (size_t i = 0; i < found.size(); ++i) out[q * k + static_cast<int64_t>(i)] = pack_candidate(found[i].distance, found[i].key);
        total += static_cast<int64_t>(found.size());
    }
    return total;
}

// the same over `threads` host threads, queries split into contiguous blocks (each query is a
// sequential traversal, as above; the result does not depend on the split)
int64_t zr_index_knn_batch_mt(void* h, const uint8_t* queries, int64_t nq, int k, int mu, int nu, int norm,
                              int threads, uint64_t* out, uint32_t* counts) {
    const auto* idx = static_cast<zcurve_index*>(h);
    search_params sp;
    sp.k = static_cast<uint32_t>(k);
    sp.mu = static_cast<uint32_t>(mu);
    sp.nu = static_cast<uint32_t>(nu);
    sp.norm = norm == 0 ? norm_kind::l2 : norm_kind::l1;
    const int T = threads < 1 ? 1 : threads;
    std::vector<int64_t> tot(T, 0);
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
        th.emplace_back([&, t] {
            knn_list list(sp.k);
            for (int64_t q = nq * t / T; q < nq * (t + 1) / T; ++q) {
                list.reset(sp.k);
                knn_search(*idx, queries + q * idx->dims(), sp, list);
                const auto found = list.sorted();
                for (size_t i = 0; i < found.size(); ++i)
                    out[q * k + static_cast<int64_t>(i)] = pack_candidate(found[i].distance, found[i].key);
                if (counts) counts[q] = static_cast<uint32_t>(found.size());
                tot[t] += static_cast<int64_t>(found.size());
            }
        });
    for (auto& x : th) x.join();
    int64_t total = 0;
    for (auto v : tot) total += v;
    return total;
}

// k-NN hook for the restated fill loop (zoracle.h zo_knn_fn): the reference's knn_search over its
// own zcurve_index per layout, on a priority_pool of `workers - 1` background threads like
// run_loop's (engine.cpp:454-458); mu / nu as in index_config.
struct zr_hook {
    zcurve_index* idx[8];
    std::unique_ptr<priority_pool> pool;
    search_params sp;
};

void* zr_hook_create(void* const* idx8, int workers, int mu, int nu) {
    auto* h = new zr_hook();
    for (int l = 0; l < 8; ++l) h->idx[l] = static_cast<zcurve_index*>(idx8[l]);
    if (workers > 1) h->pool = std::make_unique<priority_pool>(static_cast<unsigned>(workers - 1));
    h->sp.mu = static_cast<uint32_t>(mu);
    h->sp.nu = static_cast<uint32_t>(nu);
    h->sp.pool = h->pool.get();
    return h;
}

void zr_hook_free(void* h) { delete static_cast<zr_hook*>(h); }

int64_t zr_hook_knn(void* user, int layout, const uint8_t* query, int64_t k, int norm, uint64_t* out) {
    auto* h = static_cast<zr_hook*>(user);
    search_params sp = h->sp;
    sp.k = static_cast<uint32_t>(k);
    sp.norm = norm == 0 ? norm_kind::l2 : norm_kind::l1;
    const auto found = knn_search(*h->idx[layout], query, sp);
    for (size_t i = 0; i < found.size(); ++i) out[i] = pack_candidate(found[i].distance, found[i].key);
    return static_cast<int64_t>(found.size());
}

// extract_patch_clamped (proj/src/image.cpp:44-47)
void zr_extract_patch_clamped(const uint8_t* img, const uint8_t* known, int w, int h, int C, int cx,
                              int cy, int K, uint8_t* tv, uint8_t* tk) {
    raster_image im(w, h, C);
    std::memcpy(im.data.data(), img, im.data.size());
    mask_image mk(w, h);
    std::memcpy(mk.known.data(), known, mk.known.size());
    const auto v = extract_patch_clamped(im, mk, {cx, cy}, K);
    std::memcpy(tv, v.values.data(), v.values.size());
    std::memcpy(tk, v.known.data(), v.known.size());
}

// compute_fillfront (proj/src/image.cpp:49-61); xy_out 2 ints per pixel; returns count
int64_t zr_fillfront(const uint8_t* known, int w, int h, int* xy_out) {
    mask_image mk(w, h);
    std::memcpy(mk.known.data(), known, mk.known.size());
    const auto f = compute_fillfront(mk);
    for (size_t i = 0; i < f.size(); ++i) {
        xy_out[2 * i] = f[i].x;
        xy_out[2 * i + 1] = f[i].y;
    }
    return static_cast<int64_t>(f.size());
}

}  // extern "C"
