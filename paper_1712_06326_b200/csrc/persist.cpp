// persist.cpp -- ZIDX1 index persistence (proj/src/io_index.cpp:41-154; format documented at
// proj/include/zinpaint/io_index.hpp:10-17).
//
// One block per layout index, eight blocks back to back (layout 0 first), little-endian:
//   "ZIDX1" | u32 K | f64 coverage | u32 D | u32 layout id | u64 count | u32 channels
//   mean (m f64) | components (D rows of m f64) | eigenvalues (D f64) | lo (D f64) | hi (D f64)
//   count entries of (D coordinate bytes, u32 x, u32 y), in index (Morton) order
// with m = subset_pixel_count(K, coverage) * channels.  Loading re-sorts every block's entries
// on the device (the from_descriptors path, io_index.cpp:120) and recovers the dictionary from
// layout 0's keys (io_index.cpp:149-151); the PCA models and quantiser ranges are uploaded as
// stored, so a loaded index answers queries exactly like the one that was saved.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "zi_internal.h"

namespace zi {

namespace {

constexpr char kMagic[5] = {'Z', 'I', 'D', 'X', '1'};

struct file_closer {
    void operator()(std::FILE* f) const {
        if (f) std::fclose(f);
    }
};
using file_ptr = std::unique_ptr<std::FILE, file_closer>;

// same order-preserving map as common.cuh's double_to_ordered (device min/max slots)
unsigned long long double_to_ordered_host(double x) {
    unsigned long long b;
    std::memcpy(&b, &x, sizeof(b));
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

template <typename T>
void put(std::vector<uint8_t>& b, T v) {
    const size_t o = b.size();
    b.resize(o + sizeof(T));
    std::memcpy(b.data() + o, &v, sizeof(T));
}
void put_f64s(std::vector<uint8_t>& b, const double* v, size_t n) {
    const size_t o = b.size();
    b.resize(o + n * sizeof(double));
    std::memcpy(b.data() + o, v, n * sizeof(double));
}

struct reader {
    std::FILE* f;
    void read(void* dst, size_t bytes) {
        if (bytes && std::fread(dst, 1, bytes, f) != bytes) throw error(ZI_E_RUNTIME, "index file: truncated");
    }
    template <typename T>
    T pod() {
        T v{};
        read(&v, sizeof(T));
        return v;
    }
};

struct block {
    uint32_t K = 0, D = 0, layout = 0, C = 0;
    double coverage = 0.0;
    uint64_t count = 0;
    std::vector<double> mean, comp, eig, lo, hi;
    std::vector<uint8_t> coords;
    std::vector<uint32_t> keys;  // packed y<<16 | x
};

block read_block(reader& r) {
    char magic[5];
    r.read(magic, sizeof(magic));
    if (std::memcmp(magic, kMagic, sizeof(kMagic)) != 0) throw error(ZI_E_RUNTIME, "index file: bad magic");
    block b;
    b.K = r.pod<uint32_t>();
    b.coverage = r.pod<double>();
    b.D = r.pod<uint32_t>();
    b.layout = r.pod<uint32_t>();
    b.count = r.pod<uint64_t>();
    b.C = r.pod<uint32_t>();
    if (b.layout >= 8 || b.D == 0 || b.D > 32 || (b.C != 1 && b.C != 3))
        throw error(ZI_E_RUNTIME, "index file: bad header");
    if (b.K < 1 || b.K > 255 || !(b.coverage > 0.0 && b.coverage <= 1.0))
        throw error(ZI_E_RUNTIME, "index file: bad header");
    const size_t m = static_cast<size_t>(subset_pixel_count(static_cast<int>(b.K), b.coverage)) * b.C;
    b.mean.resize(m);
    r.read(b.mean.data(), m * sizeof(double));
    b.comp.resize(static_cast<size_t>(b.D) * m);
    r.read(b.comp.data(), b.comp.size() * sizeof(double));
    b.eig.resize(b.D);
    b.lo.resize(b.D);
    b.hi.resize(b.D);
    r.read(b.eig.data(), b.D * sizeof(double));
    r.read(b.lo.data(), b.D * sizeof(double));
    r.read(b.hi.data(), b.D * sizeof(double));
    if (b.count > (1ull << 32)) throw error(ZI_E_RUNTIME, "index file: bad header");
    b.coords.resize(b.count * b.D);
    b.keys.resize(b.count);
    const size_t entry = b.D + 8;
    std::vector<uint8_t> buf(std::min<uint64_t>(b.count, 1u << 16) * entry);
    for (uint64_t i0 = 0; i0 < b.count; i0 += 1u << 16) {
        const uint64_t c = std::min<uint64_t>(b.count - i0, 1u << 16);
        r.read(buf.data(), c * entry);
        for (uint64_t i = 0; i < c; ++i) {
            const uint8_t* e = buf.data() + i * entry;
            std::memcpy(b.coords.data() + (i0 + i) * b.D, e, b.D);
            uint32_t x, y;
            std::memcpy(&x, e + b.D, 4);
            std::memcpy(&y, e + b.D + 4, 4);
            if (x > 0xffff || y > 0xffff) throw error(ZI_E_RUNTIME, "index file: key out of range");
            b.keys[i0 + i] = (y << 16) | x;
        }
    }
    return b;
}

// coords (n x D, any order) + packed keys -> a device z-curve index sorted by (Morton, key)
void index_from_host(zi_ctx* ctx, const uint8_t* coords, const uint32_t* keys, uint64_t n, int D, uint32_t layout,
                     zi_index* idx) {
    idx->ctx = ctx;
    idx->layout_id = layout;
    if (n == 0) {
        finalize_index(ctx, nullptr, nullptr, 0, 0, 0, D, nullptr, idx);
        return;
    }
    const int W = (D + 3) / 4;
    dbuf<uint8_t> dc;
    dbuf<uint32_t> recs;
    dc.ensure(n * D);
    recs.ensure(static_cast<size_t>(W + 1) * n + n);
    uint32_t* keys_in = recs.p + static_cast<size_t>(W + 1) * n;
    ZI_CUDA(cudaMemcpyAsync(dc.p, coords, n * D, cudaMemcpyHostToDevice, ctx->stream));
    ZI_CUDA(cudaMemcpyAsync(keys_in, keys, n * sizeof(uint32_t), cudaMemcpyHostToDevice, ctx->stream));
    bool ascending = true;
    for (uint64_t i = 1; i < n && ascending; ++i) ascending = keys[i - 1] < keys[i];
    uint32_t* keyw = recs.p;
    uint32_t* val = recs.p + static_cast<size_t>(W) * n;
    interleave_coords(ctx, dc.p, keys_in, n, D, keyw, val);
    uint32_t* sorted[10];
    morton_sort_records(ctx, keyw, val, n, 1, D, false, sorted, ascending);
    finalize_index(ctx, sorted[0], sorted[W], n, 0, n, D, nullptr, idx);
    ZI_CUDA(cudaStreamSynchronize(ctx->stream));  // dc / recs are freed (stream-ordered) on return
}

}  // namespace

void save_multi_index(zi_multi_index* mi, const char* path) {
    if (mi->n == 0) throw error(ZI_E_INVALID, "index file: empty multi-index");
    sync_host_model(mi);
    if (mi->L[0].mean.empty()) throw error(ZI_E_RUNTIME, "index file: PCA model unavailable");
    file_ptr f(std::fopen(path, "wb"));
    if (!f) throw error(ZI_E_RUNTIME, std::string("cannot write index file: ") + path);
    const uint32_t D = static_cast<uint32_t>(mi->dims);
    const uint64_t n = mi->n;
    std::vector<uint32_t> keys(n);
    for (int l = 0; l < 8; ++l) {
        const zi_layout_state& L = mi->L[l];
        std::vector<uint8_t> b;
        b.reserve(64 + (L.mean.size() * (D + 1) + 3 * D) * 8);
        for (char c : kMagic) b.push_back(static_cast<uint8_t>(c));
        put<uint32_t>(b, static_cast<uint32_t>(mi->K));
        put<double>(b, mi->cfg.coverage);
        put<uint32_t>(b, D);
        put<uint32_t>(b, static_cast<uint32_t>(l));
        put<uint64_t>(b, n);
        put<uint32_t>(b, static_cast<uint32_t>(mi->C));
        put_f64s(b, L.mean.data(), L.mean.size());
        put_f64s(b, L.comp.data(), L.comp.size());  // D rows of m (component d contiguous)
        put_f64s(b, L.eig.data(), D);
        put_f64s(b, L.lo.data(), D);
        put_f64s(b, L.hi.data(), D);
        if (std::fwrite(b.data(), 1, b.size(), f.get()) != b.size())
            throw error(ZI_E_RUNTIME, "index file: write failed");
        // entries in index (Morton) order
        zi_index* idx = const_cast<zi_index*>(&L.index);
        std::vector<uint32_t> planes(static_cast<size_t>(idx->planes_n) * n);
        ZI_CUDA(cudaMemcpyAsync(planes.data(), idx->planes.p, planes.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                                mi->ctx->stream));
        ZI_CUDA(cudaMemcpyAsync(keys.data(), idx->keys.p, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, mi->ctx->stream));
        ZI_CUDA(cudaStreamSynchronize(mi->ctx->stream));
        const size_t entry = D + 8;
        std::vector<uint8_t> eb(std::min<uint64_t>(n, 1u << 16) * entry);
        for (uint64_t i0 = 0; i0 < n; i0 += 1u << 16) {
            const uint64_t c = std::min<uint64_t>(n - i0, 1u << 16);
            for (uint64_t i = 0; i < c; ++i) {
                uint8_t* e = eb.data() + i * entry;
                for (uint32_t d = 0; d < D; ++d)
                    e[d] = static_cast<uint8_t>((planes[static_cast<size_t>(d >> 2) * n + i0 + i] >> ((d & 3) * 8)) & 0xff);
                const uint32_t key = keys[i0 + i], x = key & 0xffffu, y = key >> 16;
                std::memcpy(e + D, &x, 4);
                std::memcpy(e + D + 4, &y, 4);
            }
            if (std::fwrite(eb.data(), 1, c * entry, f.get()) != c * entry)
                throw error(ZI_E_RUNTIME, "index file: write failed");
        }
    }
    if (std::fflush(f.get()) != 0) throw error(ZI_E_RUNTIME, "index file: write failed");
}

zidx_header zidx_peek(const char* path) {
    file_ptr f(std::fopen(path, "rb"));
    if (!f) throw error(ZI_E_RUNTIME, std::string("cannot open index file: ") + path);
    reader r{f.get()};
    char magic[5];
    r.read(magic, sizeof(magic));
    if (std::memcmp(magic, kMagic, sizeof(kMagic)) != 0) throw error(ZI_E_RUNTIME, "index file: bad magic");
    zidx_header h;
    h.K = static_cast<int>(r.pod<uint32_t>());
    h.coverage = r.pod<double>();
    h.D = static_cast<int>(r.pod<uint32_t>());
    (void)r.pod<uint32_t>();
    h.count = r.pod<uint64_t>();
    h.C = static_cast<int>(r.pod<uint32_t>());
    if (h.D <= 0 || h.D > 32 || (h.C != 1 && h.C != 3) || h.K < 1 || h.K > 255 || !(h.coverage > 0.0 && h.coverage <= 1.0))
        throw error(ZI_E_RUNTIME, "index file: bad header");
    return h;
}

void load_multi_index_into(zi_multi_index* mi, const char* path) {
    file_ptr f(std::fopen(path, "rb"));
    if (!f) throw error(ZI_E_RUNTIME, std::string("cannot open index file: ") + path);
    reader r{f.get()};
    std::vector<block> blocks;
    blocks.reserve(8);
    for (int i = 0; i < 8; ++i) {
        blocks.push_back(read_block(r));
        const block& b = blocks.back();
        const block& b0 = blocks.front();
        if (b.K != b0.K || b.coverage != b0.coverage || b.D != b0.D || b.C != b0.C || b.count != b0.count)
            throw error(ZI_E_RUNTIME, "index file: blocks disagree on build parameters");
    }
    int seen = 0;
    for (const block& b : blocks) seen |= 1 << b.layout;
    if (seen != 0xff) throw error(ZI_E_RUNTIME, "index file: layout ids are not 0..7");
    const block& b0 = blocks.front();
    if (static_cast<int>(b0.C) != mi->C) throw error(ZI_E_INVALID, "index file: channel count differs from the image");
    if (b0.count == 0) throw error(ZI_E_EMPTY_DICT, "index file: empty dictionary");
    mi->cfg.patch_size = static_cast<int32_t>(b0.K);
    mi->cfg.coverage = b0.coverage;
    mi->cfg.dims = static_cast<int32_t>(b0.D);
    mi->K = static_cast<int32_t>(b0.K);
    mi->F = mi->K * mi->K * mi->C;
    mi->n = b0.count;
    mi->dims = static_cast<int32_t>(b0.D);
    zi_ctx* ctx = mi->ctx;
    const int D = mi->dims, mc = mi->mc;  // mc from the layouts the caller uploaded for (K, coverage)
    if (static_cast<size_t>(mc) != b0.mean.size()) throw error(ZI_E_RUNTIME, "index file: bad header");
    // host model, device models, quantiser ranges
    std::vector<double> hmean(static_cast<size_t>(8) * mc), hcomp(static_cast<size_t>(8) * mc * D);
    std::vector<unsigned long long> hmm(static_cast<size_t>(8) * 2 * D);
    for (const block& b : blocks) {
        zi_layout_state& L = mi->L[b.layout];
        L.mean = b.mean;
        L.comp = b.comp;
        L.eig = b.eig;
        L.lo = b.lo;
        L.hi = b.hi;
        std::copy(b.mean.begin(), b.mean.end(), hmean.begin() + static_cast<size_t>(b.layout) * mc);
        for (int j = 0; j < mc; ++j)
            for (int d = 0; d < D; ++d)
                hcomp[(static_cast<size_t>(b.layout) * mc + j) * D + d] = b.comp[static_cast<size_t>(d) * mc + j];
        for (int d = 0; d < D; ++d) {
            hmm[static_cast<size_t>(b.layout) * 2 * D + d] = double_to_ordered_host(b.lo[d]);
            hmm[static_cast<size_t>(b.layout) * 2 * D + D + d] = double_to_ordered_host(b.hi[d]);
        }
    }
    mi->pca_mean.ensure(hmean.size());
    mi->pca_comp.ensure(hcomp.size());
    mi->minmax.ensure(hmm.size());
    ZI_CUDA(cudaMemcpyAsync(mi->pca_mean.p, hmean.data(), hmean.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    ZI_CUDA(cudaMemcpyAsync(mi->pca_comp.p, hcomp.data(), hcomp.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    ZI_CUDA(cudaMemcpyAsync(mi->minmax.p, hmm.data(), hmm.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice,
                            ctx->stream));
    ZI_CUDA(cudaStreamSynchronize(ctx->stream));  // the host vectors above are pageable locals
    mi->host_model = true;
    mi->host_lohi = true;
    mi->loaded = true;
    // the eight indices (re-sorted on the device) and the dictionary = sorted layout-0 keys
    for (const block& b : blocks)
        index_from_host(ctx, b.coords.data(), b.keys.data(), b.count, D, b.layout, &mi->L[b.layout].index);
    std::vector<uint32_t> dict;
    for (const block& b : blocks)
        if (b.layout == 0) dict = b.keys;
    std::sort(dict.begin(), dict.end());
    mi->dict.ensure(dict.size());
    ZI_CUDA(cudaMemcpyAsync(mi->dict.p, dict.data(), dict.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, ctx->stream));
    ZI_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace zi
