/*
 * zinpaint_b200.hpp -- the reference's C++ API (namespace zinpaint) as a drop-in over the
 * B200 C ABI (zinpaint_b200.h).
 *
 * The reference's hot path sits behind C++ value types and free functions
 * (/root/reference/proj/include/zinpaint/{types,morton,image,layouts,pca,pool,zcurve,builder,
 * engine,io_index}.hpp).  This header keeps those names, signatures, value semantics and
 * exception types; the forwarding headers include/zinpaint/<name>.hpp map the reference's include
 * paths onto it, so code written against the reference -- including its own unit tests --
 * compiles unchanged.  The work goes to the sm_100a kernels through the zi_* C ABI:
 *
 *   zcurve_index::from_descriptors  -> zi_index_from_descriptors   (device Morton radix sort)
 *   knn_search                      -> zi_knn_search               (device exact k-NN)
 *   collect_dictionary              -> zi_dictionary_collect
 *   build_index (one layout)        -> zi_index_build
 *   patch_index::make_query         -> zi_make_query / zi_multi_index_make_query
 *   multi_index::build              -> zi_multi_index_build
 *   query_best_patch                -> zi_query_best_patch
 *   brute_force_best                -> zi_brute_force_scan
 *   inpaint                         -> zi_inpaint / zi_inpaint_with_index
 *   save_multi_index / load_multi_index -> zi_multi_index_save / zi_multi_index_load
 *
 * Status codes come back as the reference's exceptions: ZI_E_INVALID -> std::invalid_argument,
 * ZI_E_EMPTY_DICT -> empty_dictionary_error, ZI_E_RANGE -> std::out_of_range, ZI_E_RUNTIME ->
 * std::runtime_error; CUDA / OOM failures (no reference counterpart) -> zinpaint::device_error,
 * a std::runtime_error.  The host-only utilities (Morton order, splits, distances, knn_list,
 * image windows, priorities, paste) are implemented on the host exactly as the reference defines
 * them.  Differences, all documented in INTEGRATION.md: search_params::mu / nu / pool and the
 * priority_pool* arguments are accepted and do not change results (the GPU search has no CPU
 * traversal); pca_model holds zinpaint::b200_linalg containers aliased as Eigen:: unless
 * ZINPAINT_B200_WITH_EIGEN selects the real Eigen; query_best_patch refines against the image
 * the multi_index was built from (the reference passes the fill loop's current image, whose
 * dictionary windows are the same pixels: pastes only write unknown pixels).
 *
 * All device work runs on a process-wide context on device ZI_DEVICE (default 0),
 * set_device() picks another before first use.
 */
#ifndef ZINPAINT_B200_HPP
#define ZINPAINT_B200_HPP

#include <array>
#include <atomic>
#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <memory>
#include <mutex>
#include <optional>
#include <queue>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "zinpaint_b200.h"

#if defined(ZINPAINT_B200_WITH_EIGEN)
#include <Eigen/Dense>
#else
#include "zinpaint_b200_linalg.hpp"
#endif

namespace zinpaint {

// ------------------------------------------------------------------ runtime (drop-in only)
// CUDA runtime / device allocation failure (no reference counterpart).
class device_error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
// Device of the process-wide context; call before the first GPU operation (else no effect).
void set_device(int device);
// The process-wide context every call below runs on.
zi_ctx* default_context();
// Throws the reference's exception type for a failed zi_* call.
void check_status(zi_status status);

// ------------------------------------------------------------------ types.hpp
enum class norm_kind : std::uint8_t { l2, l1 };

struct patch_key {
    std::uint16_t x = 0;
    std::uint16_t y = 0;
    constexpr std::uint32_t packed() const { return (static_cast<std::uint32_t>(y) << 16) | x; }
    friend constexpr bool operator==(patch_key a, patch_key b) { return a.x == b.x && a.y == b.y; }
    friend constexpr bool operator<(patch_key a, patch_key b) { return a.packed() < b.packed(); }
};

constexpr std::uint64_t pack_candidate(std::uint32_t distance, patch_key key) {
    return (static_cast<std::uint64_t>(distance) << 32) | key.packed();
}
constexpr std::uint32_t packed_distance(std::uint64_t candidate) { return static_cast<std::uint32_t>(candidate >> 32); }
constexpr patch_key packed_key(std::uint64_t candidate) {
    return patch_key{static_cast<std::uint16_t>(candidate & 0xffffu),
                     static_cast<std::uint16_t>((candidate >> 16) & 0xffffu)};
}

// ------------------------------------------------------------------ morton.hpp
// The most significant set bit of a is below that of b (morton.hpp:10-12).
constexpr bool less_most_significant_bit(std::uint8_t a, std::uint8_t b) {
    return a < b && a < static_cast<std::uint8_t>(a ^ b);
}
// z-curve order of two byte points: level 7 first, dimension 0 first within a level
// (morton.hpp:18-29).
inline bool morton_less(const std::uint8_t* a, const std::uint8_t* b, std::size_t dims) {
    std::uint8_t top = 0;
    std::size_t at = 0;
    for (std::size_t d = 0; d < dims; ++d) {
        const std::uint8_t x = static_cast<std::uint8_t>(a[d] ^ b[d]);
        if (less_most_significant_bit(top, x)) {
            top = x;
            at = d;
        }
    }
    return a[at] < b[at];
}

// ------------------------------------------------------------------ image.hpp
struct raster_image {
    int width = 0;
    int height = 0;
    int channels = 1;
    std::vector<std::uint8_t> data;

    raster_image() = default;
    raster_image(int w, int h, int ch, std::uint8_t fill = 0);
    std::size_t offset(int x, int y) const { return (static_cast<std::size_t>(y) * width + x) * channels; }
    std::uint8_t* pixel(int x, int y) { return data.data() + offset(x, y); }
    const std::uint8_t* pixel(int x, int y) const { return data.data() + offset(x, y); }
    bool in_bounds(int x, int y) const { return x >= 0 && x < width && y >= 0 && y < height; }
};

struct mask_image {
    int width = 0;
    int height = 0;
    std::vector<std::uint8_t> known;  // 1 = KNOWN, 0 = UNKNOWN

    mask_image() = default;
    mask_image(int w, int h, bool all_known = true);
    std::size_t idx(int x, int y) const { return static_cast<std::size_t>(y) * width + x; }
    bool is_known(int x, int y) const { return known[idx(x, y)] != 0; }
    void set_known(int x, int y, bool v) { known[idx(x, y)] = v ? 1 : 0; }
    bool in_bounds(int x, int y) const { return x >= 0 && x < width && y >= 0 && y < height; }
    std::size_t count_unknown() const;
};

struct pixel_coord {
    int x = 0;
    int y = 0;
    friend bool operator==(pixel_coord a, pixel_coord b) { return a.x == b.x && a.y == b.y; }
};

struct patch_view {
    int k = 0;
    int channels = 1;
    std::vector<std::uint8_t> values;  // k*k*channels, unknown pixels 0
    std::vector<std::uint8_t> known;   // k*k
    int known_count() const;
};

// Window centred at `center` (image.cpp:7-19); throws std::out_of_range when it leaves the image.
patch_view extract_patch(const raster_image& image, const mask_image& mask, pixel_coord center, int k);
// Same window, out-of-image pixels reported unknown (image.cpp:21-47).
patch_view extract_patch_clamped(const raster_image& image, const mask_image& mask, pixel_coord center, int k);
// KNOWN pixels with an UNKNOWN 4-neighbour, row-major (image.cpp:49-61).
std::vector<pixel_coord> compute_fillfront(const mask_image& mask);
bool is_fillfront_pixel(const mask_image& mask, int x, int y);

// ------------------------------------------------------------------ layouts.hpp
struct subset_layout {
    std::uint32_t id = 0;
    int patch_size = 0;
    std::pair<int, int> anchor{0, 0};         // (row, col)
    std::vector<std::pair<int, int>> pixels;  // (row, col), row-major
    bool covers(int row, int col) const {
        for (const auto& p : pixels)
            if (p.first == row && p.second == col) return true;
        return false;
    }
};

int subset_pixel_count(int patch_size, double coverage);
std::array<subset_layout, 8> build_subset_layouts(int patch_size, double coverage);

// ------------------------------------------------------------------ pool.hpp
// Prioritised job queue: smallest priority first, then submission order (pool.hpp:17-47).  The
// GPU paths accept a pool pointer and do not need it; it is kept for callers that schedule their
// own host work on it.
class priority_pool {
public:
    explicit priority_pool(unsigned background_threads);
    ~priority_pool();
    priority_pool(const priority_pool&) = delete;
    priority_pool& operator=(const priority_pool&) = delete;
    void submit(std::uint64_t priority, std::function<void()> fn);
    void help_until_idle();
    unsigned background_threads() const { return static_cast<unsigned>(threads_.size()); }

private:
    struct job {
        std::uint64_t priority, seq;
        std::function<void()> fn;
    };
    struct later {
        bool operator()(const job& a, const job& b) const {
            return a.priority != b.priority ? a.priority > b.priority : a.seq > b.seq;
        }
    };
    bool run_next(std::unique_lock<std::mutex>& lk);
    std::mutex mx_;
    std::condition_variable wake_, idle_;
    std::priority_queue<job, std::vector<job>, later> queue_;
    std::uint64_t seq_ = 0;
    int running_ = 0;
    bool stop_ = false;
    std::vector<std::thread> threads_;
};

// ------------------------------------------------------------------ pca.hpp
struct pca_model {
    Eigen::VectorXd mean;
    Eigen::MatrixXd components;  // input_dim x dims (column d = principal direction d)
    Eigen::VectorXd eigenvalues;
    int input_dim() const { return static_cast<int>(mean.size()); }
    int dims() const { return static_cast<int>(components.cols()); }
    // y = components^T (x - mean) in the canonical order of the build (fma chain over j from +0)
    void project(const double* x, double* y) const;
};

// ------------------------------------------------------------------ zcurve.hpp
struct hyper_cube {
    static constexpr std::size_t max_dims = 32;
    std::array<std::uint8_t, max_dims> first{};
    std::array<std::uint8_t, max_dims> last{};
    std::uint32_t dims = 0;

    static hyper_cube full(std::uint32_t dims) {
        hyper_cube c;
        c.dims = dims;
        c.first.fill(0);
        c.last.fill(255);
        return c;
    }
    bool degenerate() const {
        for (std::uint32_t d = 0; d < dims; ++d)
            if (first[d] != last[d]) return false;
        return true;
    }
    bool contains(const std::uint8_t* p) const {
        for (std::uint32_t d = 0; d < dims; ++d)
            if (p[d] < first[d] || p[d] > last[d]) return false;
        return true;
    }
};

struct interval {
    std::int64_t first = 0;
    std::int64_t last = -1;
    bool empty() const { return last < first; }
    std::int64_t length() const { return empty() ? 0 : last - first + 1; }
};

enum class boundary_hint : std::uint8_t { none, lower, upper };

struct split_point {
    std::uint32_t dim = 0;
    std::uint8_t pos = 0;
};

split_point find_split(const hyper_cube& range);
std::uint32_t region_distance(const std::uint8_t* query, const hyper_cube& range, norm_kind norm);
std::uint32_t point_distance(const std::uint8_t* a, const std::uint8_t* b, std::uint32_t dims, norm_kind norm);

struct knn_entry {
    std::uint32_t distance = 0;
    patch_key key;
    friend bool operator==(const knn_entry& a, const knn_entry& b) {
        return a.distance == b.distance && a.key == b.key;
    }
};

// Bounded best-k set of packed (distance, key) values (zcurve.hpp:76-114, zcurve.cpp:25-62).
class knn_list {
public:
    explicit knn_list(std::uint32_t capacity = 1) { reset(capacity); }
    knn_list(const knn_list&) = delete;
    knn_list& operator=(const knn_list&) = delete;
    void reset(std::uint32_t capacity);
    bool insert(std::uint64_t candidate);
    std::uint64_t bound() const { return bound_.load(std::memory_order_acquire); }
    bool full() const { return size() == capacity_; }
    std::uint32_t capacity() const { return capacity_; }
    std::size_t size() const { return size_.load(std::memory_order_acquire); }
    std::vector<knn_entry> sorted() const;

private:
    std::uint32_t capacity_ = 0;
    std::vector<std::uint64_t> heap_;
    std::atomic<std::uint64_t> bound_{~0ull};
    std::atomic<std::size_t> size_{0};
    mutable std::mutex mx_;
};

namespace detail {
struct zindex_state;  // the device index + a lazily filled host mirror (dropin.cpp)
}

// Z-sorted descriptors (zcurve.hpp:117-145).  The sorted array lives on the device; coords() /
// keys() / coords_at() / key_at() read a host mirror copied back on first use.  Copies share the
// (immutable) device index.
class zcurve_index {
public:
    zcurve_index() = default;
    static zcurve_index from_descriptors(std::vector<std::uint8_t> coords, std::vector<patch_key> keys,
                                         std::uint32_t dims, std::uint32_t layout_id);

    std::size_t size() const { return size_; }
    bool empty() const { return size_ == 0; }
    std::uint32_t dims() const { return dims_; }
    std::uint32_t layout_id() const { return layout_id_; }
    const std::uint8_t* coords_at(std::size_t i) const { return coords().data() + i * dims_; }
    patch_key key_at(std::size_t i) const { return keys()[i]; }
    const std::vector<std::uint8_t>& coords() const;
    const std::vector<patch_key>& keys() const;
    interval subinterval(const hyper_cube& range, interval parent, boundary_hint hint) const;

    // drop-in: the device index (nullptr when empty), valid while any copy of this index lives
    zi_index* device_index() const;
    // drop-in: wrap a device index owned elsewhere (`owner` keeps it alive)
    static zcurve_index from_device(zi_index* idx, std::uint32_t layout_id, std::shared_ptr<void> owner);

private:
    std::uint32_t dims_ = 0;
    std::uint32_t layout_id_ = 0;
    std::size_t size_ = 0;
    std::shared_ptr<detail::zindex_state> state_;
};

struct search_params {
    std::uint32_t k = 1;
    std::uint32_t mu = 256;          // accepted; the GPU scan has no leaf threshold
    norm_kind norm = norm_kind::l2;
    priority_pool* pool = nullptr;   // accepted; no CPU traversal to parallelise
    std::uint32_t nu = 2048;
};

// Exact k-NN under packed (distance, key) order, on the device (zcurve.cpp:429-452).
void knn_search(const zcurve_index& index, const std::uint8_t* query, const search_params& params, knn_list& out);
std::vector<knn_entry> knn_search(const zcurve_index& index, const std::uint8_t* query, const search_params& params);
// Host scan of one interval with the k-th-distance crop (zcurve.cpp:453-457 + scan_interval).
bool leaf_scan(const zcurve_index& index, interval iv, const std::uint8_t* query, norm_kind norm, knn_list& list,
               hyper_cube& range);

// ------------------------------------------------------------------ builder.hpp
class empty_dictionary_error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

struct index_config {
    int patch_size = 9;
    double coverage = 0.6;
    int dims = 10;
    int knn = 80;
    std::uint32_t mu = 256;
    std::uint32_t nu = 2048;
    norm_kind norm = norm_kind::l2;
    void validate(int channels) const;
};

struct quantizer {
    std::vector<double> lo;
    std::vector<double> hi;
    std::uint8_t quantize(int dim, double y) const;
    void quantize_vector(const double* y, std::uint8_t* out) const;
};

void project_quantize(const pca_model& model, const quantizer& q, const double* x, std::uint8_t* out);

std::vector<patch_key> collect_dictionary(const raster_image& image, const mask_image& mask, int patch_size);

namespace detail {
struct pindex_state;  // device model of one layout (standalone build or a multi-index member)
struct mindex_state;  // device multi-index
}

struct patch_index {
    subset_layout layout;
    pca_model pca;
    quantizer quant;
    zcurve_index index;
    int channels = 1;
    double build_seconds = 0.0;
    double sort_seconds = 0.0;

    // make_query on the device (builder.cpp:110-127)
    void make_query(const patch_view& target, std::uint8_t* out) const;
    std::size_t size() const { return index.size(); }

    std::shared_ptr<detail::pindex_state> b200;  // drop-in: device model
};

patch_index build_index(const raster_image& image, const std::vector<patch_key>& dictionary,
                        const subset_layout& layout, const index_config& cfg);
patch_index build_index(const raster_image& image, const mask_image& mask, const subset_layout& layout,
                        const index_config& cfg);

struct multi_index {
    index_config cfg;
    int channels = 1;
    std::vector<patch_key> dictionary;
    std::vector<patch_index> indices;  // size 8, by layout id

    static multi_index build(const raster_image& image, const mask_image& mask, const index_config& cfg,
                             priority_pool* pool = nullptr);

    std::shared_ptr<detail::mindex_state> b200;  // drop-in: the device multi-index
};

// ------------------------------------------------------------------ engine.hpp
struct iteration_record {
    std::size_t iteration = 0;
    pixel_coord target;
    std::uint32_t layout_id = 0;
    patch_key source;
    double z_error = 0.0;
    std::optional<double> bf_error;
    std::size_t candidates = 0;
    double elapsed_seconds = 0.0;
};

struct inpaint_config {
    index_config index;
    int workers = 0;
    bool oracle = false;
    std::size_t oracle_stride = 1;
    bool brute_force = false;
};

struct run_stats {
    std::size_t dictionary_size = 0;
    std::vector<double> index_build_seconds;
    double sort_seconds = 0.0;
    double build_wall_seconds = 0.0;
    double inpaint_seconds = 0.0;
    std::size_t iterations = 0;
    std::optional<double> mean_acceleration_error;
    std::size_t ae_excluded = 0;
    double confidence_low = 1.0;
    double confidence_high = 0.0;
};

struct inpaint_result {
    raster_image image;
    std::vector<iteration_record> records;
    run_stats stats;
};

struct best_patch {
    patch_key key;
    std::uint32_t cost = 0;
    double error = 0.0;
    std::uint32_t layout_id = 0;
    std::size_t candidates = 0;
};

std::uint32_t masked_cost(const patch_view& target, const patch_view& candidate, norm_kind norm);
std::uint32_t masked_cost_at(const raster_image& image, const patch_view& target,
                             const std::vector<std::uint16_t>& known_locals, patch_key source, norm_kind norm);
double cost_to_error(std::uint32_t cost, norm_kind norm);
double confidence_term(const mask_image& mask, const std::vector<double>& confidence, pixel_coord center,
                       int patch_size);
double compute_priority(const raster_image& image, const mask_image& mask, const std::vector<double>& confidence,
                        pixel_coord center, int patch_size);
pixel_coord select_target(const std::vector<pixel_coord>& fillfront, const std::vector<double>& priorities);
std::uint32_t select_index(const patch_view& target, const std::array<subset_layout, 8>& layouts);

best_patch query_best_patch(const raster_image& image, const patch_view& target, const multi_index& mi,
                            priority_pool* pool = nullptr);
best_patch query_best_patch(const raster_image& image, const patch_view& target, const multi_index& mi,
                            const index_config& cfg, priority_pool* pool);
best_patch brute_force_best(const raster_image& image, const patch_view& target,
                            const std::vector<patch_key>& dictionary, norm_kind norm);

struct paste_result {
    int filled = 0;
    double center_confidence = 0.0;
};
paste_result paste(raster_image& image, mask_image& mask, std::vector<double>& confidence, pixel_coord center,
                   patch_key source, int patch_size);

inpaint_result inpaint(const raster_image& image, const mask_image& mask, const inpaint_config& cfg);
inpaint_result inpaint(const raster_image& image, const mask_image& mask, const multi_index& mi,
                       const inpaint_config& cfg);

struct ae_summary {
    std::optional<double> mean;
    std::size_t contributing = 0;
    std::size_t excluded = 0;
};
ae_summary acceleration_error(const std::vector<iteration_record>& records);

// ------------------------------------------------------------------ io_index.hpp
// ZIDX1 files (io_index.hpp:10-26), byte-identical to the reference's.
void save_multi_index(const multi_index& mi, const std::string& path);
// The loaded multi-index is bound to an image at its first query (the file holds no pixels).
multi_index load_multi_index(const std::string& path);

}  // namespace zinpaint

#endif /* ZINPAINT_B200_HPP */
