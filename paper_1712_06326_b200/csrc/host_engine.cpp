// host_engine.cpp -- the sequential fill loop (host) around the device query.
//
// Restates proj/src/engine.cpp:83-146 (confidence / priority), :238-257 (paste),
// :283-369 (fill_driver), :371-438 (run_loop), :259-276 (acceleration_error).  The loop is
// inherently sequential (each paste changes the next target), so it stays on the host; each
// iteration's patch search runs on the GPU (zi::query_best_patch / zi::brute_force_best).
// Sources are dictionary windows, which are fully known and never overwritten, so the
// device copy of the input image stays valid for every cost evaluation.
//
// Built with -ffp-contract=off: priorities are compared exactly (std::set order, `!=`
// refresh), so no expression may be silently fused.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <limits>
#include <set>
#include <utility>
#include <thread>
#include <vector>

#include "zi_internal.h"

namespace zi {
namespace {

constexpr double kPriorityEpsilon = 1e-3;

// rows [0, h) split over the host's cores (the fill loop's one-time setup: pure per-pixel work,
// so the results do not depend on the split)
template <typename F>
void parallel_rows(int h, F&& f) {
    const int nt = static_cast<int>(std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
    if (nt == 1 || h < 256) {
        f(0, h);
        return;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t) {
        const int y0 = static_cast<int>(static_cast<int64_t>(h) * t / nt), y1 = static_cast<int>(static_cast<int64_t>(h) * (t + 1) / nt);
        th.emplace_back([&f, y0, y1] { f(y0, y1); });
    }
    for (auto& t : th) t.join();
}

struct raster {
    int w, h, C;
    std::vector<uint8_t> px;
    const uint8_t* at(int x, int y) const { return px.data() + (static_cast<size_t>(y) * w + x) * C; }
    uint8_t* at(int x, int y) { return px.data() + (static_cast<size_t>(y) * w + x) * C; }
};

struct mask {
    int w, h;
    std::vector<uint8_t> known;
    bool is_known(int x, int y) const { return known[static_cast<size_t>(y) * w + x] != 0; }
    bool in_bounds(int x, int y) const { return x >= 0 && x < w && y >= 0 && y < h; }
    size_t idx(int x, int y) const { return static_cast<size_t>(y) * w + x; }
};

// proj/src/image.cpp:49-55
bool is_fillfront_pixel(const mask& m, int x, int y) {
    if (!m.is_known(x, y)) return false;
    return (x > 0 && !m.is_known(x - 1, y)) || (x + 1 < m.w && !m.is_known(x + 1, y)) ||
           (y > 0 && !m.is_known(x, y - 1)) || (y + 1 < m.h && !m.is_known(x, y + 1));
}

double channel_mean(const uint8_t* p, int C) {
    int sum = 0;
    for (int c = 0; c < C; ++c) sum += p[c];
    return static_cast<double>(sum) / C;
}

// proj/src/engine.cpp:83-94.  conf is 0 at unknown pixels, so adding it there is exact (x + 0.0
// == x) and the known test is not needed inside the window.
double confidence_term(const mask& m, const std::vector<double>& conf, int cx, int cy, int K) {
    const int r = (K - 1) / 2;
    double sum = 0.0;
    const int y0 = std::max(cy - r, 0), y1 = std::min(cy + r, m.h - 1);
    const int x0 = std::max(cx - r, 0), x1 = std::min(cx + r, m.w - 1);
    for (int y = y0; y <= y1; ++y) {
        const double* row = conf.data() + static_cast<size_t>(y) * m.w;
        for (int x = x0; x <= x1; ++x) sum += row[x];
    }
    return sum / (static_cast<double>(K) * K);
}

// Per-pixel caches of the data term's inputs, kept current across pastes:
//   inten[i] = channel_mean (int channel sum / C as double, proj/src/engine.cpp:24-28)
//   sq[i]    = gx^2 + gy^2 of the central-difference gradient when the pixel is interior and it
//              and its 4 neighbours are known (engine.cpp:110-121), else -2 (below any candidate:
//              the window scan starts from -1 and keeps the first strict maximum)
// A paste changes inten inside its window and the known flags there, so sq changes only within
// one pixel of it (refresh); the argmax pixel's gx, gy are recomputed from inten, same formula.
struct grad_cache {
    std::vector<double> inten, sq;
    int w = 0;
    void init(const raster& img, const mask& m) {
        w = m.w;
        inten.assign(static_cast<size_t>(m.w) * m.h, 0.0);
        sq.assign(static_cast<size_t>(m.w) * m.h, -2.0);
        parallel_rows(m.h, [&](int y0, int y1) {
            for (int y = y0; y < y1; ++y)
                for (int x = 0; x < m.w; ++x) inten[m.idx(x, y)] = channel_mean(img.at(x, y), img.C);
        });
        parallel_rows(m.h, [&](int y0, int y1) { refresh(m, 0, y0, m.w - 1, y1 - 1); });
    }
    void set_pixel(const raster& img, const mask& m, int x, int y) { inten[m.idx(x, y)] = channel_mean(img.at(x, y), img.C); }
    double gx(size_t i) const { return (inten[i + 1] - inten[i - 1]) / 2.0; }
    double gy(size_t i) const { return (inten[i + w] - inten[i - w]) / 2.0; }
    void refresh(const mask& m, int xa, int ya, int xb, int yb) {
        xa = std::max(xa, 0);
        ya = std::max(ya, 0);
        xb = std::min(xb, m.w - 1);
        yb = std::min(yb, m.h - 1);
        for (int y = ya; y <= yb; ++y)
            for (int x = xa; x <= xb; ++x) {
                const size_t i = m.idx(x, y);
                const bool g = x >= 1 && y >= 1 && x + 1 < m.w && y + 1 < m.h && m.is_known(x, y) &&
                               m.is_known(x - 1, y) && m.is_known(x + 1, y) && m.is_known(x, y - 1) &&
                               m.is_known(x, y + 1);
                if (g) {
                    const double a = gx(i), b = gy(i);
                    sq[i] = a * a + b * b;
                } else {
                    sq[i] = -2.0;
                }
            }
    }
};

// proj/src/engine.cpp:96-146: priority = confidence term x data term
double data_term(const mask& m, const grad_cache& gc, int cx, int cy, int K);
double compute_priority(const raster& img, const mask& m, const std::vector<double>& conf, const grad_cache& gc,
                        int cx, int cy, int K) {
    (void)img;
    return confidence_term(m, conf, cx, cy, K) * data_term(m, gc, cx, cy, K);
}

double data_term(const mask& m, const grad_cache& gc, int cx, int cy, int K) {
    const int r = (K - 1) / 2;
    double best_sq = -1.0, bgx = 0.0, bgy = 0.0;
    size_t best_i = 0;
    const int y0 = std::max(cy - r, 0), y1 = std::min(cy + r, m.h - 1);
    const int x0 = std::max(cx - r, 0), x1 = std::min(cx + r, m.w - 1);
    for (int y = y0; y <= y1; ++y) {
        const size_t row = static_cast<size_t>(y) * m.w;
        const double* sq = gc.sq.data() + row;
        for (int x = x0; x <= x1; ++x)
            if (sq[x] > best_sq) {  // the first strict maximum in scan order, as the reference
                best_sq = sq[x];
                best_i = row + x;
            }
    }
    if (best_sq > -1.0) {
        bgx = gc.gx(best_i);
        bgy = gc.gy(best_i);
    }
    auto unknown_at = [&](int x, int y) {
        x = std::clamp(x, 0, m.w - 1);
        y = std::clamp(y, 0, m.h - 1);
        return m.is_known(x, y) ? 0.0 : 1.0;
    };
    const double nx = (unknown_at(cx + 1, cy) - unknown_at(cx - 1, cy)) / 2.0;
    const double ny = (unknown_at(cx, cy + 1) - unknown_at(cx, cy - 1)) / 2.0;
    const double nlen = std::hypot(nx, ny);
    double data = kPriorityEpsilon;
    if (best_sq > 0.0 && nlen > 0.0) {
        const double iso_x = -bgy, iso_y = bgx;
        data = std::abs(iso_x * nx / nlen + iso_y * ny / nlen) / 255.0 + kPriorityEpsilon;
    }
    return data;
}

struct by_priority {
    bool operator()(const std::pair<double, uint32_t>& a, const std::pair<double, uint32_t>& b) const {
        if (a.first != b.first) return a.first > b.first;
        return a.second < b.second;
    }
};

// proj/src/engine.cpp:283-369 -- fill front ordered by (priority desc, row-major asc),
// priorities cached and refreshed only where a paste could change them.
class fill_driver {
public:
    fill_driver(raster& img, mask& m, int K)
        : img_(img), m_(m), K_(K), conf_(static_cast<size_t>(m.w) * m.h, 0.0),
          cached_(static_cast<size_t>(m.w) * m.h, 0.0), in_front_(static_cast<size_t>(m.w) * m.h, 0) {
        for (size_t i = 0; i < conf_.size(); ++i) conf_[i] = m.known[i] ? 1.0 : 0.0;
        gc_.init(img_, m_);
        // the initial front's priorities in parallel, then the queue in pixel order
        parallel_rows(m.h, [&](int y0, int y1) {
            for (int y = y0; y < y1; ++y)
                for (int x = 0; x < m.w; ++x)
                    if (is_fillfront_pixel(m_, x, y)) {
                        const size_t i = m_.idx(x, y);
                        cached_[i] = compute_priority(img_, m_, conf_, gc_, x, y, K_);
                        in_front_[i] = 1;
                    }
        });
        for (size_t i = 0; i < in_front_.size(); ++i)
            if (in_front_[i]) {
                ++live_;
                push(cached_[i], static_cast<uint32_t>(i));
            }
    }
    bool empty() {
        prune();
        return heap_.empty();
    }
    void next_target(int& x, int& y) {
        prune();
        const uint32_t pos = heap_.front().second;
        x = static_cast<int>(pos % m_.w);
        y = static_cast<int>(pos / m_.w);
    }
    // paste (engine.cpp:238-257) + membership / priority refresh (engine.cpp:307-330), in two
    // halves so that the first can run while the device answers the query:
    //  prepare_paste: everything that does not depend on the source patch -- the center's
    //    pre-paste confidence, the filled pixels' known flags and confidences, the new fill-front
    //    membership of the zone, and the confidence terms of the zone's front pixels;
    //  finish_paste: the pasted values, the gradient cache, the data terms, the queue updates.
    // Priorities only read the post-paste state, and the queue's final content does not depend
    // on the order of its updates, so the result equals the one-step paste.
    void prepare_paste(int cx, int cy) {
        const int r = (K_ - 1) / 2;
        pcx_ = cx;
        pcy_ = cy;
        pcc_ = confidence_term(m_, conf_, cx, cy, K_);
        filled_.clear();
        for (int dy = 0; dy < K_; ++dy) {
            const int y = cy - r + dy;
            for (int dx = 0; dx < K_; ++dx) {
                const int x = cx - r + dx;
                if (!m_.in_bounds(x, y) || m_.is_known(x, y)) continue;
                filled_.push_back(static_cast<uint32_t>(dy * K_ + dx));
                m_.known[m_.idx(x, y)] = 1;
                conf_[m_.idx(x, y)] = pcc_;
            }
        }
        acts_.clear();
        if (filled_.empty()) return;
        const int refresh = K_ - 1;
        for (int y = cy - refresh; y <= cy + refresh; ++y) {
            if (y < 0 || y >= m_.h) continue;
            for (int x = cx - refresh; x <= cx + refresh; ++x) {
                if (x < 0 || x >= m_.w) continue;
                const size_t i = m_.idx(x, y);
                const bool zone = std::abs(x - cx) <= r + 1 && std::abs(y - cy) <= r + 1;
                const bool now = zone ? is_fillfront_pixel(m_, x, y) : in_front_[i] != 0;
                if (in_front_[i] && !now) acts_.push_back({static_cast<uint32_t>(i), 0, 0.0});
                else if (now) acts_.push_back({static_cast<uint32_t>(i), in_front_[i] ? 2 : 1, confidence_term(m_, conf_, x, y, K_)});
            }
        }
    }
    int finish_paste(uint32_t src, double* center_conf) {
        const int r = (K_ - 1) / 2, cx = pcx_, cy = pcy_;
        const int sx = static_cast<int>(src & 0xffffu), sy = static_cast<int>(src >> 16);
        for (const uint32_t l : filled_) {
            const int dy = static_cast<int>(l) / K_, dx = static_cast<int>(l) % K_;
            const int x = cx - r + dx, y = cy - r + dy;
            const uint8_t* sp = img_.at(sx + dx, sy + dy);
            uint8_t* d = img_.at(x, y);
            for (int c = 0; c < img_.C; ++c) d[c] = sp[c];
            gc_.set_pixel(img_, m_, x, y);
        }
        *center_conf = pcc_;
        if (filled_.empty()) return 0;
        gc_.refresh(m_, cx - r - 1, cy - r - 1, cx + r + 1, cy + r + 1);
        for (const act& a : acts_) {
            const int x = static_cast<int>(a.i % static_cast<uint32_t>(m_.w)), y = static_cast<int>(a.i / static_cast<uint32_t>(m_.w));
            if (a.kind == 0) {
                remove(x, y);
                continue;
            }
            const double fresh = a.cterm * data_term(m_, gc_, x, y, K_);
            if (a.kind == 1) {
                cached_[a.i] = fresh;
                in_front_[a.i] = 1;
                ++live_;
                push(fresh, a.i);
            } else if (fresh != cached_[a.i]) {
                cached_[a.i] = fresh;
                push(fresh, a.i);
            }
        }
        return static_cast<int>(filled_.size());
    }

private:
    void add(int x, int y) {
        const size_t i = m_.idx(x, y);
        cached_[i] = compute_priority(img_, m_, conf_, gc_, x, y, K_);
        in_front_[i] = 1;
        ++live_;
        push(cached_[i], static_cast<uint32_t>(i));
    }
    void remove(int x, int y) {
        const size_t i = m_.idx(x, y);
        in_front_[i] = 0;  // its heap entries go stale
        --live_;
    }
    void refresh_one(int x, int y) {
        const size_t i = m_.idx(x, y);
        const double fresh = compute_priority(img_, m_, conf_, gc_, x, y, K_);
        if (fresh != cached_[i]) {
            cached_[i] = fresh;
            push(fresh, static_cast<uint32_t>(i));
        }
    }
    raster& img_;
    mask& m_;
    int K_;
    std::vector<double> conf_, cached_;
    std::vector<uint8_t> in_front_;
    // The fill front ordered as the reference's std::set<(priority, pixel)> with by_priority
    // (priority desc, pixel index asc; engine.cpp:283-306): a binary heap under the same strict
    // order with lazy deletion -- an entry is live iff its pixel is on the front with exactly
    // that cached priority.  The set's begin() is then the heap's first live entry (keys are
    // unique: one pixel, one cached priority), without a node allocation per update.
    std::vector<std::pair<double, uint32_t>> heap_;
    size_t live_ = 0;
    static bool heap_less(const std::pair<double, uint32_t>& a, const std::pair<double, uint32_t>& b) {
        return by_priority{}(b, a);  // std heaps keep the largest under `less` first
    }
    bool live(const std::pair<double, uint32_t>& e) const { return in_front_[e.second] && cached_[e.second] == e.first; }
    void push(double p, uint32_t i) {
        heap_.emplace_back(p, i);
        std::push_heap(heap_.begin(), heap_.end(), heap_less);
        if (heap_.size() > 64 && heap_.size() > 8 * front_size()) compact();
    }
    size_t front_size() const { return live_; }
    void prune() {
        while (!heap_.empty() && !live(heap_.front())) {
            std::pop_heap(heap_.begin(), heap_.end(), heap_less);
            heap_.pop_back();
        }
    }
    void compact() {  // drop stale entries (and duplicates of a live key) and re-heapify
        std::vector<std::pair<double, uint32_t>> keep;
        keep.reserve(live_ + 16);
        for (const auto& e : heap_)
            if (live(e)) keep.push_back(e);
        std::sort(keep.begin(), keep.end());
        keep.erase(std::unique(keep.begin(), keep.end()), keep.end());
        heap_.swap(keep);
        std::make_heap(heap_.begin(), heap_.end(), heap_less);
    }
    grad_cache gc_;
    struct act {
        uint32_t i;
        int kind;      // 0 leaves the front, 1 joins it, 2 stays (priority refreshed)
        double cterm;  // post-paste confidence term (kinds 1, 2)
    };
    int pcx_ = 0, pcy_ = 0;
    double pcc_ = 0.0;
    std::vector<uint32_t> filled_;
    std::vector<act> acts_;
};

// extract_patch_clamped (proj/src/image.cpp:7-47)
void extract_clamped(const raster& img, const mask& m, int cx, int cy, int K, std::vector<uint8_t>& tv,
                     std::vector<uint8_t>& tk) {
    const int r = (K - 1) / 2;
    std::fill(tv.begin(), tv.end(), 0);
    std::fill(tk.begin(), tk.end(), 0);
    for (int dy = 0; dy < K; ++dy) {
        const int y = cy - r + dy;
        for (int dx = 0; dx < K; ++dx) {
            const int x = cx - r + dx;
            if (!m.in_bounds(x, y) || !m.is_known(x, y)) continue;
            const int local = dy * K + dx;
            tk[local] = 1;
            const uint8_t* s = img.at(x, y);
            for (int c = 0; c < img.C; ++c) tv[static_cast<size_t>(local) * img.C + c] = s[c];
        }
    }
}

double cost_to_error(uint32_t cost, int norm) {
    return norm == ZI_NORM_L2 ? std::sqrt(static_cast<double>(cost)) : static_cast<double>(cost);
}

}  // namespace

// run_loop (proj/src/engine.cpp:371-438)
void run_inpaint(zi_multi_index* mi, const uint8_t* image, const uint8_t* known, const zi_index_config& cfg,
                 const zi_inpaint_config& icfg, uint8_t* image_out, zi_iteration_record* records, uint64_t cap,
                 uint64_t* n_records, zi_run_stats* stats) {
    raster img{mi->w, mi->h, mi->C, std::vector<uint8_t>(image, image + static_cast<size_t>(mi->w) * mi->h * mi->C)};
    mask m{mi->w, mi->h, std::vector<uint8_t>(static_cast<size_t>(mi->w) * mi->h)};
    for (size_t i = 0; i < m.known.size(); ++i) m.known[i] = known[i] ? 1 : 0;
    uint64_t unknown_left = 0;
    for (auto v : m.known) unknown_left += v == 0;
    uint64_t it = 0;
    double ae_sum = 0.0;
    uint64_t ae_contrib = 0, ae_excl = 0;
    stats->iterations = 0;
    stats->mean_ae = std::numeric_limits<double>::quiet_NaN();
    stats->ae_excluded = 0;
    stats->confidence_low = 1.0;
    stats->confidence_high = 0.0;
    if (unknown_left == 0) {
        std::copy(img.px.begin(), img.px.end(), image_out);
        *n_records = 0;
        stats->inpaint_seconds = 0.0;
        return;
    }
    const auto t0 = std::chrono::steady_clock::now();
    const int K = mi->K;
    fill_driver drv(img, m, K);
    std::vector<uint8_t> tv(static_cast<size_t>(K) * K * mi->C), tk(static_cast<size_t>(K) * K);
    const uint32_t k = static_cast<uint32_t>(std::max(cfg.knn, 1));
    double t_query = 0.0, t_paste = 0.0, t_select = 0.0;
    while (unknown_left > 0) {
        const auto t_it = std::chrono::steady_clock::now();
        if (drv.empty()) throw error(ZI_E_RUNTIME, "inpaint: unknown pixels unreachable from the fillfront");
        int tx, ty;
        drv.next_target(tx, ty);
        extract_clamped(img, m, tx, ty, K, tv, tk);
        t_select += std::chrono::duration<double>(std::chrono::steady_clock::now() - t_it).count();
        bool prepared = false;
        const std::function<void()> prepare = [&] {
            drv.prepare_paste(tx, ty);
            prepared = true;
        };
        zi_iteration_record rec{};
        rec.iteration = it;
        rec.target_x = tx;
        rec.target_y = ty;
        uint64_t best;
        const auto tq0 = std::chrono::steady_clock::now();
        if (icfg.brute_force) {
            best = brute_force_best(mi, tv.data(), tk.data(), cfg.norm);
            rec.layout_id = 0;
            rec.candidates = mi->n;
        } else {
            const query_result q = query_best_patch(mi, tv.data(), tk.data(), k, cfg.norm, nullptr, &prepare);
            best = q.best;
            rec.layout_id = q.lid;
            rec.candidates = q.count;
        }
        rec.cost = static_cast<uint32_t>(best >> 32);
        rec.source_key = static_cast<uint32_t>(best & 0xffffffffu);
        rec.z_error = cost_to_error(rec.cost, cfg.norm);
        rec.bf_error = std::numeric_limits<double>::quiet_NaN();
        if (icfg.oracle && !icfg.brute_force && it % std::max<uint64_t>(1, icfg.oracle_stride) == 0) {
            const uint64_t o = brute_force_best(mi, tv.data(), tk.data(), cfg.norm);
            rec.bf_error = cost_to_error(static_cast<uint32_t>(o >> 32), cfg.norm);
        } else if (icfg.brute_force) {
            rec.bf_error = rec.z_error;
        }
        // acceleration_error (engine.cpp:259-276)
        if (!std::isnan(rec.bf_error)) {
            if (rec.bf_error > 0.0) {
                ae_sum += rec.z_error / rec.bf_error - 1.0;
                ++ae_contrib;
            } else if (rec.z_error == 0.0) {
                ++ae_contrib;
            } else {
                ++ae_excl;
            }
        }
        const auto tp0 = std::chrono::steady_clock::now();
        t_query += std::chrono::duration<double>(tp0 - tq0).count();
        double cc;
        if (!prepared) prepare();  // brute-force runs (and the oracle scan) take no callback
        unknown_left -= static_cast<uint64_t>(drv.finish_paste(rec.source_key, &cc));
        t_paste += std::chrono::duration<double>(std::chrono::steady_clock::now() - tp0).count();
        stats->confidence_low = std::min(stats->confidence_low, cc);
        stats->confidence_high = std::max(stats->confidence_high, cc);
        rec.elapsed_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_it).count();
        if (records && it < cap) records[it] = rec;
        ++it;
    }
    std::copy(img.px.begin(), img.px.end(), image_out);
    *n_records = it;
    stats->iterations = it;
    stats->inpaint_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (ae_contrib > 0) stats->mean_ae = ae_sum / static_cast<double>(ae_contrib);
    if (std::getenv("ZI_DEBUG_QUERY") || std::getenv("ZI_DEBUG_FILL"))
        std::fprintf(stderr, "fill loop: %llu iterations, select+extract %.1f us/it, query %.1f us/it, paste+priorities %.1f us/it, total %.1f us/it\n",
                     static_cast<unsigned long long>(it), 1e6 * t_select / it, 1e6 * t_query / it, 1e6 * t_paste / it,
                     1e6 * std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / it);
    stats->ae_excluded = ae_excl;
}

}  // namespace zi
