// dropin.cpp -- the reference's C++ API (include/zinpaint_b200.hpp) over the zi_* C ABI.
//
// Device work goes through the C ABI (api.cu) on one process-wide context; status codes come
// back as the reference's exception types.  The host-only pieces restate the reference:
//   types / Morton order / splits / distances / knn_list   proj/src/zcurve.cpp:16-106
//   subinterval, leaf_scan                                 proj/src/zcurve.cpp:140-179, :453-457
//   image windows and the fill front                       proj/src/image.cpp:7-61
//   costs, confidence, priority, target / layout choice,
//   paste, acceleration error                              proj/src/engine.cpp:16-276
//   priority_pool                                          proj/include/zinpaint/pool.hpp
// Built with -ffp-contract=off: priorities and the host projection are compared exactly.
#include "zinpaint_b200.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>

namespace zinpaint {

// ------------------------------------------------------------------ runtime
namespace {
std::mutex g_ctx_mx;
zi_ctx* g_ctx = nullptr;
int g_device = -1;

int device_from_env() {
    const char* e = std::getenv("ZI_DEVICE");
    return e ? std::atoi(e) : 0;
}

std::vector<std::uint32_t> pack_keys(const std::vector<patch_key>& keys) {
    std::vector<std::uint32_t> out(keys.size());
    for (std::size_t i = 0; i < keys.size(); ++i) out[i] = keys[i].packed();
    return out;
}

patch_key unpack_key(std::uint32_t k) {
    return patch_key{static_cast<std::uint16_t>(k & 0xffffu), static_cast<std::uint16_t>(k >> 16)};
}

zi_index_config to_c(const index_config& c) {
    zi_index_config z;
    z.patch_size = c.patch_size;
    z.coverage = c.coverage;
    z.dims = c.dims;
    z.knn = c.knn;
    z.mu = c.mu;
    z.nu = c.nu;
    z.norm = c.norm == norm_kind::l2 ? ZI_NORM_L2 : ZI_NORM_L1;
    return z;
}

int to_c(norm_kind n) { return n == norm_kind::l2 ? ZI_NORM_L2 : ZI_NORM_L1; }

// 8-bit value of bit position of the top set bit (-1 for 0)
int top_bit(unsigned v) {
    int b = -1;
    while (v) {
        ++b;
        v >>= 1;
    }
    return b;
}

// ceil(sqrt(n)) exactly (the leaf crop radius of an L2 list, zcurve.cpp:16-21)
std::uint32_t isqrt_up(std::uint32_t n) {
    std::uint64_t s = static_cast<std::uint64_t>(std::sqrt(static_cast<double>(n)));
    while (s > 0 && s * s >= n) --s;
    while (s * s < n) ++s;
    return static_cast<std::uint32_t>(s);
}
}  // namespace

void set_device(int device) {
    std::lock_guard<std::mutex> lk(g_ctx_mx);
    if (!g_ctx) g_device = device;
}

zi_ctx* default_context() {
    std::lock_guard<std::mutex> lk(g_ctx_mx);
    if (!g_ctx) {
        const int dev = g_device >= 0 ? g_device : device_from_env();
        zi_ctx* c = nullptr;
        const zi_status s = zi_ctx_create(dev, &c);
        if (s != ZI_OK) throw device_error(std::string("zinpaint_b200: no CUDA context: ") + zi_last_error());
        g_ctx = c;  // process lifetime
    }
    return g_ctx;
}

void check_status(zi_status s) {
    if (s == ZI_OK) return;
    const std::string msg = zi_last_error();
    switch (s) {
        case ZI_E_INVALID: throw std::invalid_argument(msg);
        case ZI_E_EMPTY_DICT: throw empty_dictionary_error(msg);
        case ZI_E_RANGE: throw std::out_of_range(msg);
        case ZI_E_RUNTIME: throw std::runtime_error(msg);
        default: throw device_error(msg);
    }
}

// ------------------------------------------------------------------ image.hpp
raster_image::raster_image(int w, int h, int ch, std::uint8_t fill) : width(w), height(h), channels(ch) {
    if (w <= 0 || h <= 0 || (ch != 1 && ch != 3)) throw std::invalid_argument("raster_image: bad dimensions");
    data.assign(static_cast<std::size_t>(w) * h * ch, fill);
}

mask_image::mask_image(int w, int h, bool all_known) : width(w), height(h) {
    if (w <= 0 || h <= 0) throw std::invalid_argument("mask_image: bad dimensions");
    known.assign(static_cast<std::size_t>(w) * h, all_known ? 1 : 0);
}

std::size_t mask_image::count_unknown() const {
    return static_cast<std::size_t>(std::count(known.begin(), known.end(), std::uint8_t{0}));
}

int patch_view::known_count() const {
    return static_cast<int>(known.size() - static_cast<std::size_t>(std::count(known.begin(), known.end(), 0)));
}

namespace {
patch_view window(const raster_image& image, const mask_image& mask, pixel_coord c, int k, bool clamp) {
    if (k < 3 || k % 2 == 0) throw std::invalid_argument("extract_patch: K must be odd and >= 3");
    const int r = (k - 1) / 2;
    if (!clamp && (c.x < r || c.y < r || c.x + r >= image.width || c.y + r >= image.height))
        throw std::out_of_range("extract_patch: window outside the image");
    patch_view v;
    v.k = k;
    v.channels = image.channels;
    v.values.assign(static_cast<std::size_t>(k) * k * image.channels, 0);
    v.known.assign(static_cast<std::size_t>(k) * k, 0);
    for (int dy = 0; dy < k; ++dy)
        for (int dx = 0; dx < k; ++dx) {
            const int x = c.x - r + dx, y = c.y - r + dy;
            if (!image.in_bounds(x, y) || !mask.is_known(x, y)) continue;
            const std::size_t local = static_cast<std::size_t>(dy) * k + dx;
            v.known[local] = 1;
            std::memcpy(v.values.data() + local * image.channels, image.pixel(x, y), image.channels);
        }
    return v;
}
}  // namespace

patch_view extract_patch(const raster_image& image, const mask_image& mask, pixel_coord center, int k) {
    return window(image, mask, center, k, false);
}

patch_view extract_patch_clamped(const raster_image& image, const mask_image& mask, pixel_coord center, int k) {
    return window(image, mask, center, k, true);
}

bool is_fillfront_pixel(const mask_image& mask, int x, int y) {
    if (!mask.is_known(x, y)) return false;
    return (x > 0 && !mask.is_known(x - 1, y)) || (x + 1 < mask.width && !mask.is_known(x + 1, y)) ||
           (y > 0 && !mask.is_known(x, y - 1)) || (y + 1 < mask.height && !mask.is_known(x, y + 1));
}

std::vector<pixel_coord> compute_fillfront(const mask_image& mask) {
    std::vector<pixel_coord> out;
    for (int y = 0; y < mask.height; ++y)
        for (int x = 0; x < mask.width; ++x)
            if (is_fillfront_pixel(mask, x, y)) out.push_back({x, y});
    return out;
}

// ------------------------------------------------------------------ layouts.hpp
int subset_pixel_count(int patch_size, double coverage) { return zi_subset_pixel_count(patch_size, coverage); }

std::array<subset_layout, 8> build_subset_layouts(int patch_size, double coverage) {
    int32_t m = 0;
    check_status(zi_subset_layouts(patch_size, coverage, nullptr, &m));
    std::vector<int32_t> rc(static_cast<std::size_t>(8) * m * 2);
    int32_t anchors[16];
    check_status(zi_subset_layouts(patch_size, coverage, rc.data(), &m));
    check_status(zi_subset_layout_anchors(patch_size, anchors));
    std::array<subset_layout, 8> out;
    for (int l = 0; l < 8; ++l) {
        auto& L = out[l];
        L.id = static_cast<std::uint32_t>(l);
        L.patch_size = patch_size;
        L.anchor = {anchors[2 * l], anchors[2 * l + 1]};
        L.pixels.resize(m);
        for (int p = 0; p < m; ++p)
            L.pixels[p] = {rc[(static_cast<std::size_t>(l) * m + p) * 2], rc[(static_cast<std::size_t>(l) * m + p) * 2 + 1]};
    }
    return out;
}

// ------------------------------------------------------------------ pool.hpp
priority_pool::priority_pool(unsigned background_threads) {
    for (unsigned i = 0; i < background_threads; ++i)
        threads_.emplace_back([this] {
            std::unique_lock<std::mutex> lk(mx_);
            for (;;) {
                wake_.wait(lk, [this] { return stop_ || !queue_.empty(); });
                if (stop_ && queue_.empty()) return;
                run_next(lk);
            }
        });
}

priority_pool::~priority_pool() {
    {
        std::lock_guard<std::mutex> lk(mx_);
        stop_ = true;
    }
    wake_.notify_all();
    for (auto& t : threads_) t.join();
}

void priority_pool::submit(std::uint64_t priority, std::function<void()> fn) {
    {
        std::lock_guard<std::mutex> lk(mx_);
        queue_.push(job{priority, seq_++, std::move(fn)});
    }
    wake_.notify_one();
}

// pops and runs one job (lock held on entry and exit, released while the job runs)
bool priority_pool::run_next(std::unique_lock<std::mutex>& lk) {
    if (queue_.empty()) return false;
    job j = queue_.top();
    queue_.pop();
    ++running_;
    lk.unlock();
    try {
        j.fn();
    } catch (...) {
    }
    lk.lock();
    --running_;
    if (queue_.empty() && running_ == 0) idle_.notify_all();
    return true;
}

void priority_pool::help_until_idle() {
    std::unique_lock<std::mutex> lk(mx_);
    for (;;) {
        if (run_next(lk)) continue;
        if (running_ == 0) return;
        idle_.wait(lk, [this] { return !queue_.empty() || running_ == 0; });
    }
}

// ------------------------------------------------------------------ pca.hpp
void pca_model::project(const double* x, double* y) const {
    const long in = mean.size(), D = components.cols();
    for (long d = 0; d < D; ++d) {
        double acc = 0.0;
        for (long j = 0; j < in; ++j) acc = std::fma(components(j, d), x[j] - mean[j], acc);
        y[d] = acc;
    }
}

// ------------------------------------------------------------------ zcurve.hpp
split_point find_split(const hyper_cube& range) {
    int best = -1;
    std::uint32_t dim = 0;
    for (std::uint32_t d = 0; d < range.dims; ++d) {
        const int b = top_bit(static_cast<unsigned>(range.first[d] ^ range.last[d]));
        if (b > best) {  // equal levels keep the earlier dimension
            best = b;
            dim = d;
        }
    }
    const unsigned low = (1u << best) - 1u;                     // bits below the split level
    const unsigned clear = ~((low << 1) | 1u) & 0xffu;          // clears the split level and below
    return {dim, static_cast<std::uint8_t>((range.first[dim] & clear) | low)};
}

std::uint32_t region_distance(const std::uint8_t* q, const hyper_cube& range, norm_kind norm) {
    std::uint32_t acc = 0;
    for (std::uint32_t d = 0; d < range.dims; ++d) {
        const std::uint32_t g = q[d] < range.first[d] ? range.first[d] - q[d]
                                : q[d] > range.last[d] ? q[d] - range.last[d]
                                                       : 0u;
        acc += norm == norm_kind::l2 ? g * g : g;
    }
    return acc;
}

std::uint32_t point_distance(const std::uint8_t* a, const std::uint8_t* b, std::uint32_t dims, norm_kind norm) {
    std::uint32_t acc = 0;
    for (std::uint32_t d = 0; d < dims; ++d) {
        const std::int32_t diff = static_cast<std::int32_t>(a[d]) - static_cast<std::int32_t>(b[d]);
        acc += norm == norm_kind::l2 ? static_cast<std::uint32_t>(diff * diff)
                                     : static_cast<std::uint32_t>(diff < 0 ? -diff : diff);
    }
    return acc;
}

void knn_list::reset(std::uint32_t capacity) {
    std::lock_guard<std::mutex> lk(mx_);
    capacity_ = std::max<std::uint32_t>(capacity, 1);
    heap_.clear();
    heap_.reserve(capacity_);
    bound_.store(~0ull, std::memory_order_release);
    size_.store(0, std::memory_order_release);
}

bool knn_list::insert(std::uint64_t c) {
    if (c >= bound()) return false;
    std::lock_guard<std::mutex> lk(mx_);
    if (heap_.size() < capacity_) {
        heap_.push_back(c);
        std::push_heap(heap_.begin(), heap_.end());
        size_.store(heap_.size(), std::memory_order_release);
        if (heap_.size() == capacity_) bound_.store(heap_.front(), std::memory_order_release);
        return true;
    }
    if (c >= heap_.front()) return false;
    std::pop_heap(heap_.begin(), heap_.end());
    heap_.back() = c;
    std::push_heap(heap_.begin(), heap_.end());
    bound_.store(heap_.front(), std::memory_order_release);
    return true;
}

std::vector<knn_entry> knn_list::sorted() const {
    std::vector<std::uint64_t> v;
    {
        std::lock_guard<std::mutex> lk(mx_);
        v = heap_;
    }
    std::sort(v.begin(), v.end());
    std::vector<knn_entry> out(v.size());
    for (std::size_t i = 0; i < v.size(); ++i) out[i] = {packed_distance(v[i]), packed_key(v[i])};
    return out;
}

namespace detail {
struct zindex_state {
    zi_index* idx = nullptr;
    bool owned = false;
    std::shared_ptr<void> owner;  // keeps a borrowed index's parent alive
    std::mutex mx;
    std::atomic<bool> ready{false};
    std::vector<std::uint8_t> coords;
    std::vector<patch_key> keys;
    ~zindex_state() {
        if (owned && idx) zi_index_destroy(idx);
    }
    void fill(std::size_t n, std::uint32_t dims) {
        if (ready.load(std::memory_order_acquire)) return;
        std::lock_guard<std::mutex> lk(mx);
        if (ready.load(std::memory_order_relaxed)) return;
        std::vector<std::uint32_t> k(n);
        coords.assign(n * dims, 0);
        if (n) check_status(zi_index_export(idx, coords.data(), k.data()));
        keys.resize(n);
        for (std::size_t i = 0; i < n; ++i) keys[i] = unpack_key(k[i]);
        ready.store(true, std::memory_order_release);
    }
};
}  // namespace detail

namespace {
const std::vector<std::uint8_t> kNoCoords;
const std::vector<patch_key> kNoKeys;
}  // namespace

zcurve_index zcurve_index::from_descriptors(std::vector<std::uint8_t> coords, std::vector<patch_key> keys,
                                            std::uint32_t dims, std::uint32_t layout_id) {
    if (dims == 0 || dims > hyper_cube::max_dims) throw std::invalid_argument("zcurve_index: dims must be in [1, 32]");
    if (coords.size() != keys.size() * dims) throw std::invalid_argument("zcurve_index: coords/keys size mismatch");
    zcurve_index out;
    out.dims_ = dims;
    out.layout_id_ = layout_id;
    out.size_ = keys.size();
    if (keys.empty()) return out;
    const auto packed = pack_keys(keys);
    auto st = std::make_shared<detail::zindex_state>();
    check_status(zi_index_from_descriptors(default_context(), coords.data(), packed.data(), keys.size(), dims,
                                           layout_id, &st->idx));
    st->owned = true;
    out.state_ = std::move(st);
    return out;
}

zcurve_index zcurve_index::from_device(zi_index* idx, std::uint32_t layout_id, std::shared_ptr<void> owner) {
    zcurve_index out;
    std::uint64_t n = 0;
    std::uint32_t dims = 0;
    check_status(zi_index_size(idx, &n, &dims));
    out.dims_ = dims;
    out.layout_id_ = layout_id;
    out.size_ = static_cast<std::size_t>(n);
    auto st = std::make_shared<detail::zindex_state>();
    st->idx = idx;
    st->owner = std::move(owner);
    out.state_ = std::move(st);
    return out;
}

zi_index* zcurve_index::device_index() const { return state_ ? state_->idx : nullptr; }

const std::vector<std::uint8_t>& zcurve_index::coords() const {
    if (!state_) return kNoCoords;
    state_->fill(size_, dims_);
    return state_->coords;
}

const std::vector<patch_key>& zcurve_index::keys() const {
    if (!state_) return kNoKeys;
    state_->fill(size_, dims_);
    return state_->keys;
}

// Entries of `parent` inside the z-window of the region corners (zcurve.cpp:140-179): the first
// entry not below the min corner, the last entry not above the max corner; a hint takes that
// side from the parent unchanged.
interval zcurve_index::subinterval(const hyper_cube& range, interval parent, boundary_hint hint) const {
    if (parent.empty()) return parent;
    const std::uint8_t* lo_c = range.first.data();
    const std::uint8_t* hi_c = range.last.data();
    std::int64_t first = parent.first, last = parent.last;
    if (hint != boundary_hint::lower) {
        std::int64_t a = parent.first, b = parent.last + 1;
        if (!morton_less(coords_at(static_cast<std::size_t>(a)), lo_c, dims_)) b = a;
        while (a < b) {
            const std::int64_t mid = a + (b - a) / 2;
            if (morton_less(coords_at(static_cast<std::size_t>(mid)), lo_c, dims_)) a = mid + 1;
            else b = mid;
        }
        first = a;
    }
    if (hint != boundary_hint::upper) {
        std::int64_t a = first, b = parent.last + 1;
        if (a <= parent.last && !morton_less(hi_c, coords_at(static_cast<std::size_t>(parent.last)), dims_)) a = b;
        while (a < b) {
            const std::int64_t mid = a + (b - a) / 2;
            if (morton_less(hi_c, coords_at(static_cast<std::size_t>(mid)), dims_)) b = mid;
            else a = mid + 1;
        }
        last = a - 1;
    }
    return {first, last};
}

void knn_search(const zcurve_index& index, const std::uint8_t* query, const search_params& params, knn_list& out) {
    out.reset(params.k);
    if (index.empty()) return;
    const std::uint32_t k = std::max<std::uint32_t>(params.k, 1);
    std::vector<std::uint64_t> found(std::min<std::size_t>(k, index.size()));
    std::uint32_t count = 0;
    check_status(zi_knn_search(index.device_index(), query, k, params.mu, to_c(params.norm), found.data(), &count));
    for (std::uint32_t i = 0; i < count; ++i) out.insert(found[i]);
}

std::vector<knn_entry> knn_search(const zcurve_index& index, const std::uint8_t* query, const search_params& params) {
    knn_list list(params.k);
    knn_search(index, query, params, list);
    return list.sorted();
}

bool leaf_scan(const zcurve_index& index, interval iv, const std::uint8_t* query, norm_kind norm, knn_list& list,
               hyper_cube& range) {
    if (iv.empty()) return false;
    bool improved = false;
    for (std::int64_t i = iv.first; i <= iv.last; ++i) {
        const std::size_t e = static_cast<std::size_t>(i);
        improved |= list.insert(pack_candidate(point_distance(query, index.coords_at(e), index.dims(), norm),
                                               index.key_at(e)));
    }
    if (improved && list.full()) {
        // crop to query +- ceil(k-th distance): nothing outside can still enter the list
        const std::uint32_t kth = packed_distance(list.bound());
        const std::uint32_t rad = norm == norm_kind::l2 ? isqrt_up(kth) : kth;
        for (std::uint32_t d = 0; d < range.dims; ++d) {
            const std::uint32_t q = query[d];
            const std::uint8_t lo = static_cast<std::uint8_t>(q > rad ? q - rad : 0);
            const std::uint8_t hi = static_cast<std::uint8_t>(std::min<std::uint32_t>(255u, q + rad));
            std::uint8_t f = std::max(range.first[d], lo), l = std::min(range.last[d], hi);
            if (f > l) f = l = hi < range.first[d] ? range.first[d] : range.last[d];
            range.first[d] = f;
            range.last[d] = l;
        }
    }
    return improved;
}

// ------------------------------------------------------------------ builder.hpp
void index_config::validate(int channels) const {
    const zi_index_config c = to_c(*this);
    check_status(zi_index_config_validate(&c, channels));
}

std::uint8_t quantizer::quantize(int dim, double y) const {
    const double l = lo[static_cast<std::size_t>(dim)], h = hi[static_cast<std::size_t>(dim)];
    if (!(h > l)) return 0;
    const double c = std::clamp(y, l, h);
    return static_cast<std::uint8_t>(std::llround(255.0 * (c - l) / (h - l)));
}

void quantizer::quantize_vector(const double* y, std::uint8_t* out) const {
    for (std::size_t d = 0; d < lo.size(); ++d) out[d] = quantize(static_cast<int>(d), y[d]);
}

void project_quantize(const pca_model& model, const quantizer& q, const double* x, std::uint8_t* out) {
    std::vector<double> y(static_cast<std::size_t>(model.dims()));
    model.project(x, y.data());
    q.quantize_vector(y.data(), out);
}

std::vector<patch_key> collect_dictionary(const raster_image& image, const mask_image& mask, int patch_size) {
    if (image.width != mask.width || image.height != mask.height)
        throw std::invalid_argument("collect_dictionary: image/mask dimensions differ");
    std::vector<std::uint32_t> keys(static_cast<std::size_t>(mask.width) * mask.height);
    std::uint64_t n = 0;
    check_status(zi_dictionary_collect(default_context(), mask.known.data(), mask.width, mask.height, patch_size,
                                       keys.data(), keys.size(), &n));
    std::vector<patch_key> out(static_cast<std::size_t>(n));
    for (std::size_t i = 0; i < out.size(); ++i) out[i] = unpack_key(keys[i]);
    return out;
}

namespace detail {
struct mindex_state {
    zi_multi_index* mi = nullptr;
    std::string path;  // loaded from a ZIDX1 file: bound to an image at first use
    int channels = 1;
    std::mutex mx;
    ~mindex_state() {
        if (mi) zi_multi_index_destroy(mi);
    }
    zi_multi_index* bind(const raster_image& image) {
        std::lock_guard<std::mutex> lk(mx);
        if (!mi) {
            if (image.channels != channels)
                throw std::invalid_argument("multi_index: image channels differ from the index's");
            check_status(zi_multi_index_load(default_context(), path.c_str(), image.data.data(), image.width,
                                             image.height, image.channels, &mi));
        }
        return mi;
    }
};

struct pindex_state {
    zi_patch_index* pi = nullptr;              // standalone build_index
    std::shared_ptr<mindex_state> parent;      // or layout `layout` of a multi-index
    int layout = 0;
    ~pindex_state() {
        if (pi) zi_patch_index_destroy(pi);
    }
};
}  // namespace detail

void patch_index::make_query(const patch_view& target, std::uint8_t* out) const {
    if (!b200) throw std::invalid_argument("patch_index::make_query: index has no device model");
    if (target.channels != channels || target.k != layout.patch_size)
        throw std::invalid_argument("patch_index::make_query: target shape differs from the index's");
    if (b200->pi) {
        check_status(zi_make_query(b200->pi, target.values.data(), target.known.data(), out));
        return;
    }
    zi_multi_index* mi = b200->parent ? b200->parent->mi : nullptr;
    if (!mi) throw std::invalid_argument("patch_index::make_query: multi-index not bound to an image yet");
    check_status(zi_multi_index_make_query(mi, b200->layout, target.values.data(), target.known.data(), out));
}

namespace {
void fill_pca(pca_model& p, int mc, int D, const std::vector<double>& mean, const std::vector<double>& comp_rows,
              const std::vector<double>& eig) {
    p.mean = Eigen::VectorXd(mc);
    p.components = Eigen::MatrixXd(mc, D);
    p.eigenvalues = Eigen::VectorXd(D);
    std::copy(mean.begin(), mean.end(), p.mean.data());
    std::copy(comp_rows.begin(), comp_rows.end(), p.components.data());  // column d = row d of comp_rows
    std::copy(eig.begin(), eig.end(), p.eigenvalues.data());
}
}  // namespace

patch_index build_index(const raster_image& image, const std::vector<patch_key>& dictionary,
                        const subset_layout& layout, const index_config& cfg) {
    cfg.validate(image.channels);
    if (dictionary.empty()) throw empty_dictionary_error("build_index: empty dictionary");
    const int m = static_cast<int>(layout.pixels.size());
    std::vector<int32_t> rc(static_cast<std::size_t>(2) * m);
    for (int p = 0; p < m; ++p) {
        rc[2 * p] = layout.pixels[p].first;
        rc[2 * p + 1] = layout.pixels[p].second;
    }
    const auto keys = pack_keys(dictionary);
    const zi_index_config c = to_c(cfg);
    auto st = std::make_shared<detail::pindex_state>();
    check_status(zi_index_build(default_context(), image.data.data(), image.width, image.height, image.channels,
                                keys.data(), keys.size(), rc.data(), m, &c, &st->pi));
    int32_t D = 0, mc = 0;
    check_status(zi_patch_index_model(st->pi, &D, &mc, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr));
    std::vector<double> mean(mc), comp(static_cast<std::size_t>(D) * mc), eig(D), lo(D), hi(D);
    patch_index out;
    check_status(zi_patch_index_model(st->pi, nullptr, nullptr, mean.data(), comp.data(), eig.data(), lo.data(),
                                      hi.data(), &out.build_seconds, &out.sort_seconds));
    out.layout = layout;
    out.layout.patch_size = cfg.patch_size;
    fill_pca(out.pca, mc, D, mean, comp, eig);
    out.quant.lo = lo;
    out.quant.hi = hi;
    out.channels = image.channels;
    zi_index* idx = nullptr;
    check_status(zi_patch_index_get_index(st->pi, &idx));
    out.index = zcurve_index::from_device(idx, layout.id, st);
    out.b200 = st;
    return out;
}

patch_index build_index(const raster_image& image, const mask_image& mask, const subset_layout& layout,
                        const index_config& cfg) {
    return build_index(image, collect_dictionary(image, mask, cfg.patch_size), layout, cfg);
}

namespace {
// host mirror of a device multi-index: dictionary, layouts, PCA models, quantisers, index views
multi_index mirror_of(const std::shared_ptr<detail::mindex_state>& st, const index_config& cfg, int channels) {
    zi_multi_index* h = st->mi;
    zi_multi_index_info info;
    check_status(zi_multi_index_get_info(h, &info));
    multi_index out;
    out.cfg = cfg;
    out.channels = channels;
    out.b200 = st;
    std::vector<std::uint32_t> dict(static_cast<std::size_t>(info.n));
    check_status(zi_multi_index_dictionary(h, dict.data()));
    out.dictionary.resize(dict.size());
    for (std::size_t i = 0; i < dict.size(); ++i) out.dictionary[i] = unpack_key(dict[i]);
    int32_t anchors[16];
    check_status(zi_subset_layout_anchors(info.patch_size, anchors));
    const int m = info.m, mc = info.m * channels, D = info.dims;
    out.indices.resize(8);
    for (int l = 0; l < 8; ++l) {
        std::vector<int32_t> rc(static_cast<std::size_t>(2) * m);
        std::vector<double> mean(mc), comp(static_cast<std::size_t>(D) * mc), eig(D), lo(D), hi(D);
        check_status(zi_multi_index_layout(h, l, rc.data(), mean.data(), comp.data(), eig.data(), lo.data(), hi.data()));
        patch_index& p = out.indices[l];
        p.layout.id = static_cast<std::uint32_t>(l);
        p.layout.patch_size = info.patch_size;
        p.layout.anchor = {anchors[2 * l], anchors[2 * l + 1]};
        p.layout.pixels.resize(m);
        for (int q = 0; q < m; ++q) p.layout.pixels[q] = {rc[2 * q], rc[2 * q + 1]};
        fill_pca(p.pca, mc, D, mean, comp, eig);
        p.quant.lo = lo;
        p.quant.hi = hi;
        p.channels = channels;
        p.build_seconds = info.build_seconds / 8.0;  // the eight layouts are built together
        zi_index* idx = nullptr;
        check_status(zi_multi_index_get_index(h, l, &idx));
        p.index = zcurve_index::from_device(idx, static_cast<std::uint32_t>(l), st);
        auto ps = std::make_shared<detail::pindex_state>();
        ps->parent = st;
        ps->layout = l;
        p.b200 = ps;
    }
    return out;
}
}  // namespace

multi_index multi_index::build(const raster_image& image, const mask_image& mask, const index_config& cfg,
                               priority_pool* /*pool*/) {
    if (image.width != mask.width || image.height != mask.height)
        throw std::invalid_argument("multi_index: image/mask dimensions differ");
    const zi_index_config c = to_c(cfg);
    auto st = std::make_shared<detail::mindex_state>();
    st->channels = image.channels;
    check_status(zi_multi_index_build(default_context(), image.data.data(), mask.known.data(), image.width,
                                      image.height, image.channels, &c, &st->mi));
    return mirror_of(st, cfg, image.channels);
}

// ------------------------------------------------------------------ engine.hpp
std::uint32_t masked_cost(const patch_view& target, const patch_view& candidate, norm_kind norm) {
    std::uint32_t acc = 0;
    const int C = target.channels;
    for (std::size_t i = 0; i < target.known.size(); ++i) {
        if (!target.known[i]) continue;
        for (int c = 0; c < C; ++c) {
            const std::int32_t d = static_cast<std::int32_t>(target.values[i * C + c]) - candidate.values[i * C + c];
            acc += norm == norm_kind::l2 ? static_cast<std::uint32_t>(d * d) : static_cast<std::uint32_t>(d < 0 ? -d : d);
        }
    }
    return acc;
}

std::uint32_t masked_cost_at(const raster_image& image, const patch_view& target,
                             const std::vector<std::uint16_t>& known_locals, patch_key source, norm_kind norm) {
    std::uint32_t acc = 0;
    const int C = image.channels, k = target.k;
    for (const std::uint16_t local : known_locals) {
        const std::uint8_t* s = image.pixel(source.x + local % k, source.y + local / k);
        const std::uint8_t* t = target.values.data() + static_cast<std::size_t>(local) * C;
        for (int c = 0; c < C; ++c) {
            const std::int32_t d = static_cast<std::int32_t>(t[c]) - s[c];
            acc += norm == norm_kind::l2 ? static_cast<std::uint32_t>(d * d) : static_cast<std::uint32_t>(d < 0 ? -d : d);
        }
    }
    return acc;
}

double cost_to_error(std::uint32_t cost, norm_kind norm) {
    return norm == norm_kind::l2 ? std::sqrt(static_cast<double>(cost)) : static_cast<double>(cost);
}

double confidence_term(const mask_image& mask, const std::vector<double>& confidence, pixel_coord center,
                       int patch_size) {
    const int r = (patch_size - 1) / 2;
    double sum = 0.0;
    for (int y = center.y - r; y <= center.y + r; ++y)
        for (int x = center.x - r; x <= center.x + r; ++x)
            if (mask.in_bounds(x, y) && mask.is_known(x, y)) sum += confidence[mask.idx(x, y)];
    return sum / (static_cast<double>(patch_size) * patch_size);
}

double compute_priority(const raster_image& image, const mask_image& mask, const std::vector<double>& confidence,
                        pixel_coord center, int patch_size) {
    const int r = (patch_size - 1) / 2;
    const double cterm = confidence_term(mask, confidence, center, patch_size);
    auto inten = [&](int x, int y) {
        const std::uint8_t* p = image.pixel(x, y);
        int s = 0;
        for (int c = 0; c < image.channels; ++c) s += p[c];
        return static_cast<double>(s) / image.channels;
    };
    // strongest central-difference gradient over interior pixels whose stencil is known
    double best = -1.0, bgx = 0.0, bgy = 0.0;
    for (int y = center.y - r; y <= center.y + r; ++y)
        for (int x = center.x - r; x <= center.x + r; ++x) {
            if (x < 1 || y < 1 || x + 1 >= image.width || y + 1 >= image.height) continue;
            if (!mask.is_known(x, y) || !mask.is_known(x - 1, y) || !mask.is_known(x + 1, y) ||
                !mask.is_known(x, y - 1) || !mask.is_known(x, y + 1))
                continue;
            const double gx = (inten(x + 1, y) - inten(x - 1, y)) / 2.0;
            const double gy = (inten(x, y + 1) - inten(x, y - 1)) / 2.0;
            const double sq = gx * gx + gy * gy;
            if (sq > best) {
                best = sq;
                bgx = gx;
                bgy = gy;
            }
        }
    // front normal: central differences of the clamped unknown indicator
    auto unk = [&](int x, int y) {
        return mask.is_known(std::clamp(x, 0, mask.width - 1), std::clamp(y, 0, mask.height - 1)) ? 0.0 : 1.0;
    };
    const double nx = (unk(center.x + 1, center.y) - unk(center.x - 1, center.y)) / 2.0;
    const double ny = (unk(center.x, center.y + 1) - unk(center.x, center.y - 1)) / 2.0;
    const double nl = std::hypot(nx, ny);
    double data = 1e-3;
    if (best > 0.0 && nl > 0.0) data = std::abs(-bgy * nx / nl + bgx * ny / nl) / 255.0 + 1e-3;
    return cterm * data;
}

pixel_coord select_target(const std::vector<pixel_coord>& fillfront, const std::vector<double>& priorities) {
    std::size_t best = 0;
    for (std::size_t i = 1; i < fillfront.size(); ++i) {
        const bool earlier = fillfront[i].y < fillfront[best].y ||
                             (fillfront[i].y == fillfront[best].y && fillfront[i].x < fillfront[best].x);
        if (priorities[i] > priorities[best] || (priorities[i] == priorities[best] && earlier)) best = i;
    }
    return fillfront[best];
}

std::uint32_t select_index(const patch_view& target, const std::array<subset_layout, 8>& layouts) {
    std::uint32_t id = 0;
    std::size_t most = 0;
    for (const auto& L : layouts) {
        std::size_t ov = 0;
        for (const auto& px : L.pixels) ov += target.known[static_cast<std::size_t>(px.first) * target.k + px.second] != 0;
        if (ov > most) {
            most = ov;
            id = L.id;
        }
    }
    return id;
}

best_patch query_best_patch(const raster_image& image, const patch_view& target, const multi_index& mi,
                            const index_config& cfg, priority_pool* /*pool*/) {
    if (!mi.b200)
        throw std::invalid_argument("query_best_patch: multi_index was not built by multi_index::build or loaded");
    if (target.k != mi.cfg.patch_size || target.channels != mi.channels)
        throw std::invalid_argument("query_best_patch: target shape differs from the index's");
    zi_multi_index* h = mi.b200->bind(image);
    zi_best_patch bp;
    check_status(zi_query_best_patch(h, target.values.data(), target.known.data(),
                                     static_cast<std::uint32_t>(std::max(cfg.knn, 1)), to_c(cfg.norm), &bp, nullptr));
    best_patch out;
    out.key = unpack_key(bp.key);
    out.cost = bp.cost;
    out.error = bp.error;
    out.layout_id = bp.layout_id;
    out.candidates = static_cast<std::size_t>(bp.candidates);
    return out;
}

best_patch query_best_patch(const raster_image& image, const patch_view& target, const multi_index& mi,
                            priority_pool* pool) {
    return query_best_patch(image, target, mi, mi.cfg, pool);
}

best_patch brute_force_best(const raster_image& image, const patch_view& target,
                            const std::vector<patch_key>& dictionary, norm_kind norm) {
    best_patch out;
    out.candidates = dictionary.size();
    if (dictionary.empty()) return out;
    if (target.channels != image.channels) throw std::invalid_argument("brute_force_best: channel count differs");
    const auto keys = pack_keys(dictionary);
    zi_best_patch bp;
    check_status(zi_brute_force_scan(default_context(), image.data.data(), image.width, image.height, image.channels,
                                     keys.data(), keys.size(), target.values.data(), target.known.data(), target.k,
                                     to_c(norm), &bp));
    out.key = unpack_key(bp.key);
    out.cost = bp.cost;
    out.error = cost_to_error(bp.cost, norm);
    return out;
}

paste_result paste(raster_image& image, mask_image& mask, std::vector<double>& confidence, pixel_coord center,
                   patch_key source, int patch_size) {
    const int r = (patch_size - 1) / 2;
    paste_result res;
    res.center_confidence = confidence_term(mask, confidence, center, patch_size);
    for (int dy = 0; dy < patch_size; ++dy)
        for (int dx = 0; dx < patch_size; ++dx) {
            const int x = center.x - r + dx, y = center.y - r + dy;
            if (!image.in_bounds(x, y) || mask.is_known(x, y)) continue;
            std::memcpy(image.pixel(x, y), image.pixel(source.x + dx, source.y + dy), image.channels);
            mask.set_known(x, y, true);
            confidence[mask.idx(x, y)] = res.center_confidence;
            ++res.filled;
        }
    return res;
}

namespace {
inpaint_result finish_run(const raster_image& image, std::vector<std::uint8_t>&& out_px,
                          const std::vector<zi_iteration_record>& recs, std::uint64_t nrec, const zi_run_stats& st) {
    inpaint_result res;
    res.image.width = image.width;
    res.image.height = image.height;
    res.image.channels = image.channels;
    res.image.data = std::move(out_px);
    res.records.resize(static_cast<std::size_t>(nrec));
    for (std::size_t i = 0; i < res.records.size(); ++i) {
        const auto& z = recs[i];
        auto& r = res.records[i];
        r.iteration = static_cast<std::size_t>(z.iteration);
        r.target = {z.target_x, z.target_y};
        r.layout_id = z.layout_id;
        r.source = unpack_key(z.source_key);
        r.z_error = z.z_error;
        if (!std::isnan(z.bf_error)) r.bf_error = z.bf_error;
        r.candidates = static_cast<std::size_t>(z.candidates);
        r.elapsed_seconds = z.elapsed_seconds;
    }
    res.stats.dictionary_size = static_cast<std::size_t>(st.dictionary_size);
    res.stats.sort_seconds = st.sort_seconds;
    res.stats.build_wall_seconds = st.build_wall_seconds;
    res.stats.inpaint_seconds = st.inpaint_seconds;
    res.stats.iterations = static_cast<std::size_t>(st.iterations);
    if (!std::isnan(st.mean_ae)) res.stats.mean_acceleration_error = st.mean_ae;
    res.stats.ae_excluded = static_cast<std::size_t>(st.ae_excluded);
    res.stats.confidence_low = st.confidence_low;
    res.stats.confidence_high = st.confidence_high;
    return res;
}

zi_inpaint_config to_c(const inpaint_config& cfg) {
    zi_inpaint_config z;
    z.workers = cfg.workers;
    z.oracle = cfg.oracle ? 1 : 0;
    z.oracle_stride = cfg.oracle_stride;
    z.brute_force = cfg.brute_force ? 1 : 0;
    return z;
}
}  // namespace

inpaint_result inpaint(const raster_image& image, const mask_image& mask, const inpaint_config& cfg) {
    if (image.width != mask.width || image.height != mask.height)
        throw std::invalid_argument("inpaint: image/mask dimensions differ");
    cfg.index.validate(image.channels);
    if (mask.count_unknown() == 0) {
        inpaint_result res;
        res.image = image;
        return res;
    }
    const zi_index_config c = to_c(cfg.index);
    const zi_inpaint_config ic = to_c(cfg);
    std::vector<std::uint8_t> out(image.data.size());
    std::vector<zi_iteration_record> recs(mask.count_unknown() + 1);
    std::uint64_t n = 0;
    zi_run_stats st;
    check_status(zi_inpaint(default_context(), image.data.data(), mask.known.data(), image.width, image.height,
                            image.channels, &c, &ic, out.data(), recs.data(), recs.size(), &n, &st));
    inpaint_result res = finish_run(image, std::move(out), recs, n, st);
    if (!cfg.brute_force) res.stats.index_build_seconds.assign(8, st.build_wall_seconds / 8.0);
    return res;
}

inpaint_result inpaint(const raster_image& image, const mask_image& mask, const multi_index& mi,
                       const inpaint_config& cfg) {
    if (image.width != mask.width || image.height != mask.height)
        throw std::invalid_argument("inpaint: image/mask dimensions differ");
    if (mask.count_unknown() == 0) {
        inpaint_result res;
        res.image = image;
        return res;
    }
    if (!mi.b200) throw std::invalid_argument("inpaint: multi_index was not built by multi_index::build or loaded");
    zi_multi_index* h = mi.b200->bind(image);
    const zi_index_config c = to_c(cfg.index);
    const zi_inpaint_config ic = to_c(cfg);
    std::vector<std::uint8_t> out(image.data.size());
    std::vector<zi_iteration_record> recs(mask.count_unknown() + 1);
    std::uint64_t n = 0;
    zi_run_stats st;
    check_status(zi_inpaint_with_index(h, image.data.data(), mask.known.data(), &c, &ic, out.data(), recs.data(),
                                       recs.size(), &n, &st));
    return finish_run(image, std::move(out), recs, n, st);
}

ae_summary acceleration_error(const std::vector<iteration_record>& records) {
    ae_summary s;
    double sum = 0.0;
    for (const auto& r : records) {
        if (!r.bf_error) continue;
        if (*r.bf_error > 0.0) {
            sum += r.z_error / *r.bf_error - 1.0;
            ++s.contributing;
        } else if (r.z_error == 0.0) {
            ++s.contributing;
        } else {
            ++s.excluded;
        }
    }
    if (s.contributing > 0) s.mean = sum / static_cast<double>(s.contributing);
    return s;
}

// ------------------------------------------------------------------ io_index.hpp
void save_multi_index(const multi_index& mi, const std::string& path) {
    if (!mi.b200 || !mi.b200->mi) throw std::invalid_argument("save_multi_index: no device multi-index to save");
    check_status(zi_multi_index_save(mi.b200->mi, path.c_str()));
}

// Reads the ZIDX1 blocks into the host mirror (the layout indices are re-sorted on the device by
// from_descriptors, io_index.cpp:120); the device multi-index is created from the same file when
// the first query supplies the image.
multi_index load_multi_index(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("load_multi_index: cannot open " + path);
    auto rd = [&](void* dst, std::size_t bytes) {
        in.read(static_cast<char*>(dst), static_cast<std::streamsize>(bytes));
        if (!in) throw std::runtime_error("load_multi_index: truncated file");
    };
    auto st = std::make_shared<detail::mindex_state>();
    st->path = path;
    multi_index out;
    out.b200 = st;
    out.indices.resize(8);
    for (int l = 0; l < 8; ++l) {
        char magic[5];
        rd(magic, 5);
        if (std::memcmp(magic, "ZIDX1", 5) != 0) throw std::runtime_error("load_multi_index: bad magic");
        std::uint32_t K, D, lid, C;
        double cov;
        std::uint64_t n;
        rd(&K, 4);
        rd(&cov, 8);
        rd(&D, 4);
        rd(&lid, 4);
        rd(&n, 8);
        rd(&C, 4);
        if (lid != static_cast<std::uint32_t>(l)) throw std::runtime_error("load_multi_index: blocks out of order");
        if (l == 0) {
            out.cfg.patch_size = static_cast<int>(K);
            out.cfg.coverage = cov;
            out.cfg.dims = static_cast<int>(D);
            out.channels = static_cast<int>(C);
            st->channels = static_cast<int>(C);
        }
        const auto layouts = build_subset_layouts(static_cast<int>(K), cov);
        const int mc = static_cast<int>(layouts[0].pixels.size()) * static_cast<int>(C);
        std::vector<double> mean(mc), comp(static_cast<std::size_t>(D) * mc), eig(D), lo(D), hi(D);
        rd(mean.data(), mean.size() * 8);
        rd(comp.data(), comp.size() * 8);
        rd(eig.data(), eig.size() * 8);
        rd(lo.data(), lo.size() * 8);
        rd(hi.data(), hi.size() * 8);
        std::vector<std::uint8_t> coords(static_cast<std::size_t>(n) * D);
        std::vector<patch_key> keys(static_cast<std::size_t>(n));
        std::vector<std::uint8_t> entry(D + 8);
        for (std::uint64_t i = 0; i < n; ++i) {
            rd(entry.data(), entry.size());
            std::memcpy(coords.data() + i * D, entry.data(), D);
            std::uint32_t x, y;
            std::memcpy(&x, entry.data() + D, 4);
            std::memcpy(&y, entry.data() + D + 4, 4);
            if (x > 0xffffu || y > 0xffffu) throw std::runtime_error("load_multi_index: key out of range");
            keys[i] = patch_key{static_cast<std::uint16_t>(x), static_cast<std::uint16_t>(y)};
        }
        patch_index& p = out.indices[l];
        p.layout = layouts[l];
        fill_pca(p.pca, mc, static_cast<int>(D), mean, comp, eig);
        p.quant.lo = lo;
        p.quant.hi = hi;
        p.channels = static_cast<int>(C);
        if (l == 0) {
            out.dictionary = keys;
            std::sort(out.dictionary.begin(), out.dictionary.end());
        }
        p.index = zcurve_index::from_descriptors(std::move(coords), std::move(keys), D, static_cast<std::uint32_t>(l));
        auto ps = std::make_shared<detail::pindex_state>();
        ps->parent = st;
        ps->layout = l;
        p.b200 = ps;
    }
    return out;
}

}  // namespace zinpaint
