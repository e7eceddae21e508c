// zoracle.cpp -- CPU restatement of the reference hot path.  TEST INFRASTRUCTURE ONLY:
// see zoracle.h for the rules and the pinned canonical fp64 order.
//
// Build: g++ -O3 -std=c++17 -ffp-contract=off -fPIC -shared (oracle/Makefile).
// -ffp-contract=off matters: priorities and projections must not be silently fused.
#include "zoracle.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <numeric>
#include <set>
#include <string>
#include <thread>
#include <utility>
#include <vector>

namespace {

thread_local std::string g_err;

void set_err(const char* m) { g_err = m; }

// proj/include/zinpaint/types.hpp:15-17 (packed = y<<16 | x)
inline uint32_t pk(int x, int y) { return (static_cast<uint32_t>(y) << 16) | static_cast<uint32_t>(x); }
inline int key_x(uint32_t k) { return static_cast<int>(k & 0xffffu); }
inline int key_y(uint32_t k) { return static_cast<int>(k >> 16); }

}  // namespace

extern "C" {

const char* zo_error(void) { return g_err.c_str(); }

// ---------------------------------------------------------------- layouts
// proj/src/layouts.cpp:9-11 -- llround(c*K^2), half away from zero
int zo_subset_pixel_count(int K, double coverage) {
    return static_cast<int>(std::llround(coverage * K * K));
}

// proj/src/layouts.cpp:13-60 -- 8 anchors N,E,S,W,NW,NE,SW,SE; stable sort by squared
// distance to the anchor (row-major ties), keep `count`, re-sort row-major.
int zo_build_subset_layouts(int K, double coverage, int* rc_out) {
    if (K < 3 || K % 2 == 0) { set_err("subset layouts: K must be odd and >= 3"); return -1; }
    if (!(coverage > 0.0 && coverage <= 1.0)) { set_err("subset layouts: coverage must be in (0, 1]"); return -1; }
    const int count = zo_subset_pixel_count(K, coverage);
    if (count < 1) { set_err("subset layouts: coverage keeps no pixels"); return -1; }
    const int mid = (K - 1) / 2;
    const int anchors[8][2] = {{0, mid}, {mid, K - 1}, {K - 1, mid}, {mid, 0},
                               {0, 0},   {0, K - 1},   {K - 1, 0},   {K - 1, K - 1}};
    std::vector<std::pair<int, int>> offsets;
    for (int r = 0; r < K; ++r)
        for (int c = 0; c < K; ++c) offsets.emplace_back(r, c);
    for (int id = 0; id < 8; ++id) {
        const int ar = anchors[id][0], ac = anchors[id][1];
        auto v = offsets;
        std::stable_sort(v.begin(), v.end(), [&](const auto& a, const auto& b) {
            const int da = (a.first - ar) * (a.first - ar) + (a.second - ac) * (a.second - ac);
            const int db = (b.first - ar) * (b.first - ar) + (b.second - ac) * (b.second - ac);
            return da < db;
        });
        v.resize(static_cast<size_t>(count));
        std::sort(v.begin(), v.end());
        for (int i = 0; i < count; ++i) {
            rc_out[(id * count + i) * 2 + 0] = v[i].first;
            rc_out[(id * count + i) * 2 + 1] = v[i].second;
        }
    }
    return count;
}

// ---------------------------------------------------------------- Morton
// proj/include/zinpaint/morton.hpp:10-12
int zo_less_msb(int a, int b) {
    const uint8_t ua = static_cast<uint8_t>(a), ub = static_cast<uint8_t>(b);
    return (ua < ub) && (ua < (ua ^ ub));
}

// proj/include/zinpaint/morton.hpp:18-29
int zo_morton_less(const uint8_t* a, const uint8_t* b, int dims) {
    uint8_t best_diff = 0;
    int best_dim = 0;
    for (int d = 0; d < dims; ++d) {
        const uint8_t diff = static_cast<uint8_t>(a[d] ^ b[d]);
        if (zo_less_msb(best_diff, diff)) {
            best_diff = diff;
            best_dim = d;
        }
    }
    return a[best_dim] < b[best_dim];
}

// ---------------------------------------------------------------- dictionary
// proj/src/builder.cpp:74-108 -- summed-area table of unknown flags, windows with zero
// unknown pixels, row-major order.
int64_t zo_collect_dictionary(const uint8_t* known, int w, int h, int K, uint32_t* keys_out) {
    int64_t n = 0;
    if (w < K || h < K) return 0;
    std::vector<uint32_t> sat(static_cast<size_t>(w + 1) * (h + 1), 0);
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            const uint32_t unk = known[static_cast<size_t>(y) * w + x] ? 0 : 1;
            sat[static_cast<size_t>(y + 1) * (w + 1) + (x + 1)] =
                unk + sat[static_cast<size_t>(y) * (w + 1) + (x + 1)] +
                sat[static_cast<size_t>(y + 1) * (w + 1) + x] - sat[static_cast<size_t>(y) * (w + 1) + x];
        }
    for (int y = 0; y + K <= h; ++y)
        for (int x = 0; x + K <= w; ++x) {
            const uint32_t u = sat[static_cast<size_t>(y + K) * (w + 1) + (x + K)] -
                               sat[static_cast<size_t>(y) * (w + 1) + (x + K)] -
                               sat[static_cast<size_t>(y + K) * (w + 1) + x] +
                               sat[static_cast<size_t>(y) * (w + 1) + x];
            if (u == 0) keys_out[n++] = pk(x, y);
        }
    return n;
}

// ---------------------------------------------------------------- moments
// Exact integer restatement of the mean pass (proj/src/pca.cpp:20-30) and the raw second
// moments behind the covariance pass (proj/src/pca.cpp:32-37), for the full K*K*C vector.
void zo_patch_moments(const uint8_t* img, int w, int h, int C, int K, const uint32_t* keys,
                      int64_t n, int64_t* s_out, int64_t* S_out) {
    (void)h;
    const int F = K * K * C;
    std::fill(s_out, s_out + F, 0);
    std::fill(S_out, S_out + static_cast<size_t>(F) * F, 0);
    std::vector<int32_t> acc(static_cast<size_t>(F) * F, 0);
    std::vector<int32_t> x(F);
    const int64_t kBlock = 4096;  // 4096 * 255^2 < 2^31
    for (int64_t b = 0; b < n; b += kBlock) {
        const int64_t e = std::min(n, b + kBlock);
        std::fill(acc.begin(), acc.end(), 0);
        for (int64_t i = b; i < e; ++i) {
            const int kx = key_x(keys[i]), ky = key_y(keys[i]);
            int f = 0;
            for (int r = 0; r < K; ++r) {
                const uint8_t* row = img + (static_cast<size_t>(ky + r) * w + kx) * C;
                for (int c = 0; c < K * C; ++c) x[f++] = row[c];
            }
            for (int a = 0; a < F; ++a) {
                s_out[a] += x[a];
                const int32_t xa = x[a];
                int32_t* arow = acc.data() + static_cast<size_t>(a) * F;
                for (int c = a; c < F; ++c) arow[c] += xa * x[c];
            }
        }
        for (int a = 0; a < F; ++a)
            for (int c = a; c < F; ++c) S_out[static_cast<size_t>(a) * F + c] += acc[static_cast<size_t>(a) * F + c];
    }
    for (int a = 0; a < F; ++a)
        for (int c = 0; c < a; ++c) S_out[static_cast<size_t>(a) * F + c] = S_out[static_cast<size_t>(c) * F + a];
}

// proj/src/pca.cpp:22-28 (mean) and :45-46 (cov / (n-1) iff n > 1), restated on exact moments.
void zo_layout_covariance(const int64_t* s, const int64_t* S, int F, int64_t n, const int* cols,
                          int mc, double* mean_out, double* cov_out) {
    for (int i = 0; i < mc; ++i) mean_out[i] = static_cast<double>(s[cols[i]]) / static_cast<double>(n);
    const double den = n > 1 ? static_cast<double>(n) * static_cast<double>(n - 1) : 1.0;
    for (int i = 0; i < mc; ++i)
        for (int j = 0; j < mc; ++j) {
            const __int128 num = static_cast<__int128>(n) * S[static_cast<size_t>(cols[i]) * F + cols[j]] -
                                 static_cast<__int128>(s[cols[i]]) * s[cols[j]];
            cov_out[static_cast<size_t>(i) * mc + j] = static_cast<double>(num) / den;
        }
}

// proj/src/pca.cpp:39-67 -- eigenpairs, top-D descending (Eigen's ascending order
// reversed), sign flipped so the first max-|v| entry is positive, eigenvalues clamped >= 0.
// The eigensolver is a cyclic Jacobi (Eigen is not available; parity vs the reference binary
// is unpinned at the last-ulp level).
int zo_pca_from_cov(const double* cov, int mc, int D, double* comp_out, double* eig_out) {
    if (D < 1 || D > mc) { set_err("pca: dims must be in [1, input_dim]"); return -1; }
    const int n = mc;
    std::vector<double> A(cov, cov + static_cast<size_t>(n) * n);
    std::vector<double> V(static_cast<size_t>(n) * n, 0.0);
    for (int i = 0; i < n; ++i) V[static_cast<size_t>(i) * n + i] = 1.0;
    auto a = [&](int i, int j) -> double& { return A[static_cast<size_t>(i) * n + j]; };
    auto v = [&](int i, int j) -> double& { return V[static_cast<size_t>(i) * n + j]; };
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0, diag = 0.0;
        for (int i = 0; i < n; ++i) {
            diag += a(i, i) * a(i, i);
            for (int j = i + 1; j < n; ++j) off += a(i, j) * a(i, j);
        }
        if (off == 0.0 || off <= 1e-34 * (diag + off)) break;
        for (int p = 0; p < n - 1; ++p)
            for (int q = p + 1; q < n; ++q) {
                const double apq = a(p, q);
                if (apq == 0.0) continue;
                const double app = a(p, p), aqq = a(q, q);
                const double theta = (aqq - app) / (2.0 * apq);
                double t;
                if (std::fabs(theta) > 1e150) t = 0.5 / theta;
                else t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
                const double c = 1.0 / std::sqrt(t * t + 1.0);
                const double sn = t * c;
                for (int k = 0; k < n; ++k) {
                    if (k == p || k == q) continue;
                    const double akp = a(k, p), akq = a(k, q);
                    a(k, p) = a(p, k) = c * akp - sn * akq;
                    a(k, q) = a(q, k) = sn * akp + c * akq;
                }
                a(p, p) = app - t * apq;
                a(q, q) = aqq + t * apq;
                a(p, q) = a(q, p) = 0.0;
                for (int k = 0; k < n; ++k) {
                    const double vkp = v(k, p), vkq = v(k, q);
                    v(k, p) = c * vkp - sn * vkq;
                    v(k, q) = sn * vkp + c * vkq;
                }
            }
    }
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return a(x, x) < a(y, y); });
    for (int j = 0; j < D; ++j) {
        const int src = order[n - 1 - j];
        int arg = 0;
        for (int i = 1; i < n; ++i)
            if (std::fabs(v(i, src)) > std::fabs(v(arg, src))) arg = i;
        const double sgn = v(arg, src) < 0 ? -1.0 : 1.0;
        for (int i = 0; i < n; ++i) comp_out[static_cast<size_t>(j) * n + i] = sgn * v(i, src);
        eig_out[j] = std::max(0.0, a(src, src));
    }
    return 0;
}

// ---------------------------------------------------------------- quantiser
// proj/src/builder.cpp:55-61
uint8_t zo_quantize(double l, double h, double y) {
    if (!(h > l)) return 0;
    const double clamped = y < l ? l : (h < y ? h : y);  // std::clamp(y, l, h)
    return static_cast<uint8_t>(std::llround(255.0 * (clamped - l) / (h - l)));
}

// ---------------------------------------------------------------- projection
// canonical order: xc_j = x_j - mean_j ; y_d = fma(comp[d][j], xc_j, y_d), j ascending.
static void project_one(const double* x, const double* mean, const double* comp, int mc, int D,
                        double* y) {
    for (int d = 0; d < D; ++d) y[d] = 0.0;
    for (int j = 0; j < mc; ++j) {
        const double xc = x[j] - mean[j];
        for (int d = 0; d < D; ++d) y[d] = std::fma(comp[static_cast<size_t>(d) * mc + j], xc, y[d]);
    }
}

// proj/src/builder.cpp:20-34 (fill_chunk gather, pixel-major channel-minor) +
// :159-187 (pass 3 lo/hi over all projections, pass 4 quantise).
void zo_project_build(const uint8_t* img, int w, int h, int C, const uint32_t* keys, int64_t n,
                      const int* rc, int m, const double* mean, const double* comp, int D,
                      double* lo, double* hi, uint8_t* coords_out, double* y_out) {
    (void)h;
    const int mc = m * C;
    std::vector<double> x(mc), y(D);
    std::vector<double> ys(static_cast<size_t>(n) * D);
    for (int d = 0; d < D; ++d) {
        lo[d] = std::numeric_limits<double>::infinity();
        hi[d] = -std::numeric_limits<double>::infinity();
    }
    for (int64_t i = 0; i < n; ++i) {
        const int kx = key_x(keys[i]), ky = key_y(keys[i]);
        int col = 0;
        for (int p = 0; p < m; ++p) {
            const uint8_t* px = img + (static_cast<size_t>(ky + rc[2 * p]) * w + kx + rc[2 * p + 1]) * C;
            for (int ch = 0; ch < C; ++ch) x[col++] = static_cast<double>(px[ch]);
        }
        project_one(x.data(), mean, comp, mc, D, ys.data() + static_cast<size_t>(i) * D);
        for (int d = 0; d < D; ++d) {
            const double vv = ys[static_cast<size_t>(i) * D + d];
            lo[d] = std::min(lo[d], vv);
            hi[d] = std::max(hi[d], vv);
        }
    }
    for (int64_t i = 0; i < n; ++i)
        for (int d = 0; d < D; ++d)
            coords_out[static_cast<size_t>(i) * D + d] = zo_quantize(lo[d], hi[d], ys[static_cast<size_t>(i) * D + d]);
    if (y_out) std::memcpy(y_out, ys.data(), ys.size() * sizeof(double));
}

// ---------------------------------------------------------------- sort
// proj/src/zcurve.cpp:108-138 -- sort row ids by (morton_less, then packed key), copy out.
int zo_from_descriptors(const uint8_t* coords, const uint32_t* keys, int64_t n, int D,
                        uint8_t* coords_out, uint32_t* keys_out) {
    if (D < 1 || D > 32) { set_err("zcurve_index: dims must be in [1, 32]"); return -1; }
    std::vector<uint32_t> order(static_cast<size_t>(n));
    std::iota(order.begin(), order.end(), 0u);
    std::sort(order.begin(), order.end(), [&](uint32_t ia, uint32_t ib) {
        const uint8_t* a = coords + static_cast<size_t>(ia) * D;
        const uint8_t* b = coords + static_cast<size_t>(ib) * D;
        if (zo_morton_less(a, b, D)) return true;
        if (zo_morton_less(b, a, D)) return false;
        return keys[ia] < keys[ib];
    });
    for (int64_t i = 0; i < n; ++i) {
        std::memcpy(coords_out + static_cast<size_t>(i) * D, coords + static_cast<size_t>(order[i]) * D, D);
        keys_out[i] = keys[order[i]];
    }
    return 0;
}

// ---------------------------------------------------------------- knn
// proj/src/zcurve.cpp:81-106 (point_distance) + proj/tests/support/oracles.hpp:55-74.
static inline uint32_t point_distance(const uint8_t* a, const uint8_t* b, int D, int norm) {
    uint32_t acc = 0;
    for (int d = 0; d < D; ++d) {
        const int32_t diff = static_cast<int32_t>(a[d]) - b[d];
        acc += norm == 0 ? static_cast<uint32_t>(diff * diff) : static_cast<uint32_t>(diff < 0 ? -diff : diff);
    }
    return acc;
}

// Exact top-k by a plain scan: every entry's packed (distance, key) against a bounded max-heap
// (insert iff < the k-th value of a full heap, the knn_list rule of zcurve.cpp:33-49).  Large
// inputs are split over host threads, each with its own heap, and merged: the packed values are
// unique, so the result does not depend on the split.
static void knn_scan_range(const uint8_t* coords, const uint32_t* keys, int64_t b, int64_t e, int D,
                           const uint8_t* query, size_t keep, int norm, std::vector<uint64_t>& heap) {
    heap.clear();
    heap.reserve(keep + 1);
    for (int64_t i = b; i < e; ++i) {
        const uint64_t c =
            (static_cast<uint64_t>(point_distance(query, coords + static_cast<size_t>(i) * D, D, norm)) << 32) | keys[i];
        if (heap.size() < keep) {
            heap.push_back(c);
            std::push_heap(heap.begin(), heap.end());
        } else if (c < heap.front()) {
            std::pop_heap(heap.begin(), heap.end());
            heap.back() = c;
            std::push_heap(heap.begin(), heap.end());
        }
    }
}

int64_t zo_knn_linear(const uint8_t* coords, const uint32_t* keys, int64_t n, int D,
                      const uint8_t* query, int64_t k, int norm, uint64_t* out) {
    const int64_t keep = std::min<int64_t>(std::max<int64_t>(k, 1), n);
    if (keep <= 0) return 0;
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const int T = n >= (1 << 20) ? static_cast<int>(std::min<unsigned>(hw, 32)) : 1;
    std::vector<std::vector<uint64_t>> heaps(T);
    if (T == 1) {
        knn_scan_range(coords, keys, 0, n, D, query, static_cast<size_t>(keep), norm, heaps[0]);
    } else {
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t)
            th.emplace_back([&, t] {
                knn_scan_range(coords, keys, n * t / T, n * (t + 1) / T, D, query, static_cast<size_t>(keep), norm,
                               heaps[t]);
            });
        for (auto& x : th) x.join();
    }
    std::vector<uint64_t> all;
    for (auto& hp : heaps) all.insert(all.end(), hp.begin(), hp.end());
    std::partial_sort(all.begin(), all.begin() + keep, all.end());
    std::memcpy(out, all.data(), static_cast<size_t>(keep) * sizeof(uint64_t));
    return keep;
}

// ---------------------------------------------------------------- query side
// proj/src/engine.cpp:162-176 -- strict '>' over overlap counts starting at 0.
int zo_select_index(const uint8_t* tk, int K, const int* layouts_rc, int m) {
    int best_id = 0;
    int best = 0;
    for (int l = 0; l < 8; ++l) {
        int overlap = 0;
        for (int p = 0; p < m; ++p)
            overlap += tk[layouts_rc[(l * m + p) * 2] * K + layouts_rc[(l * m + p) * 2 + 1]] != 0;
        if (overlap > best) {
            best = overlap;
            best_id = l;
        }
    }
    return best_id;
}

// proj/src/builder.cpp:110-127 -- unknown layout pixels take pca.mean[col]; then
// project_quantize (proj/src/builder.cpp:63-72; proj/src/pca.cpp:7-11).
void zo_make_query(const uint8_t* tv, const uint8_t* tk, int K, int C, const int* rc, int m,
                   const double* mean, const double* comp, const double* lo, const double* hi,
                   int D, uint8_t* out) {
    const int mc = m * C;
    std::vector<double> x(mc), y(D);
    int col = 0;
    for (int p = 0; p < m; ++p) {
        const int local = rc[2 * p] * K + rc[2 * p + 1];
        for (int ch = 0; ch < C; ++ch, ++col)
            x[col] = tk[local] ? static_cast<double>(tv[local * C + ch]) : mean[col];
    }
    project_one(x.data(), mean, comp, mc, D, y.data());
    for (int d = 0; d < D; ++d) out[d] = zo_quantize(lo[d], hi[d], y[d]);
}

// ---------------------------------------------------------------- costs
// proj/src/engine.cpp:48-76
uint32_t zo_masked_cost_at(const uint8_t* img, int w, int h, int C, const uint8_t* tv,
                           const uint8_t* tk, int K, uint32_t key, int norm) {
    (void)h;
    const int sx = key_x(key), sy = key_y(key);
    uint32_t acc = 0;
    for (int local = 0; local < K * K; ++local) {
        if (!tk[local]) continue;
        const int ly = local / K, lx = local % K;
        const uint8_t* s = img + (static_cast<size_t>(sy + ly) * w + sx + lx) * C;
        const uint8_t* t = tv + static_cast<size_t>(local) * C;
        for (int c = 0; c < C; ++c) {
            const int32_t d = static_cast<int32_t>(t[c]) - s[c];
            acc += norm == 0 ? static_cast<uint32_t>(d * d) : static_cast<uint32_t>(d < 0 ? -d : d);
        }
    }
    return acc;
}

// proj/src/engine.cpp:220-236 -- min over (cost, packed key).
uint64_t zo_brute_force_best(const uint8_t* img, int w, int h, int C, const uint8_t* tv,
                             const uint8_t* tk, int K, const uint32_t* keys, int64_t n, int norm) {
    uint64_t best = ~0ull;
    for (int64_t i = 0; i < n; ++i) {
        const uint64_t c = (static_cast<uint64_t>(zo_masked_cost_at(img, w, h, C, tv, tk, K, keys[i], norm)) << 32) | keys[i];
        best = std::min(best, c);
    }
    return best;
}

// proj/src/image.cpp:7-47 (clamped variant)
void zo_extract_patch_clamped(const uint8_t* img, const uint8_t* known, int w, int h, int C,
                              int cx, int cy, int K, uint8_t* tv, uint8_t* tk) {
    const int r = (K - 1) / 2;
    std::memset(tv, 0, static_cast<size_t>(K) * K * C);
    std::memset(tk, 0, static_cast<size_t>(K) * K);
    for (int dy = 0; dy < K; ++dy) {
        const int y = cy - r + dy;
        for (int dx = 0; dx < K; ++dx) {
            const int x = cx - r + dx;
            if (x < 0 || x >= w || y < 0 || y >= h) continue;
            if (!known[static_cast<size_t>(y) * w + x]) continue;
            const int local = dy * K + dx;
            tk[local] = 1;
            for (int c = 0; c < C; ++c) tv[local * C + c] = img[(static_cast<size_t>(y) * w + x) * C + c];
        }
    }
}

// ---------------------------------------------------------------- priorities
// proj/src/engine.cpp:83-94
double zo_confidence_term(const uint8_t* known, int w, int h, const double* conf, int cx, int cy,
                          int K) {
    const int r = (K - 1) / 2;
    double sum = 0.0;
    for (int y = cy - r; y <= cy + r; ++y)
        for (int x = cx - r; x <= cx + r; ++x) {
            if (x < 0 || x >= w || y < 0 || y >= h || !known[static_cast<size_t>(y) * w + x]) continue;
            sum += conf[static_cast<size_t>(y) * w + x];
        }
    return sum / (static_cast<double>(K) * K);
}

static inline double channel_mean(const uint8_t* px, int C) {
    int sum = 0;
    for (int c = 0; c < C; ++c) sum += px[c];
    return static_cast<double>(sum) / C;
}

// proj/src/engine.cpp:96-146
double zo_compute_priority(const uint8_t* img, const uint8_t* known, int w, int h, int C,
                           const double* conf, int cx, int cy, int K) {
    const int r = (K - 1) / 2;
    const double cterm = zo_confidence_term(known, w, h, conf, cx, cy, K);
    auto kn = [&](int x, int y) { return known[static_cast<size_t>(y) * w + x] != 0; };
    auto px = [&](int x, int y) { return img + (static_cast<size_t>(y) * w + x) * C; };
    double best_sq = -1.0, best_gx = 0.0, best_gy = 0.0;
    for (int y = cy - r; y <= cy + r; ++y)
        for (int x = cx - r; x <= cx + r; ++x) {
            if (x < 1 || y < 1 || x + 1 >= w || y + 1 >= h) continue;
            if (!kn(x, y) || !kn(x - 1, y) || !kn(x + 1, y) || !kn(x, y - 1) || !kn(x, y + 1)) continue;
            const double gx = (channel_mean(px(x + 1, y), C) - channel_mean(px(x - 1, y), C)) / 2.0;
            const double gy = (channel_mean(px(x, y + 1), C) - channel_mean(px(x, y - 1), C)) / 2.0;
            const double sq = gx * gx + gy * gy;
            if (sq > best_sq) {
                best_sq = sq;
                best_gx = gx;
                best_gy = gy;
            }
        }
    auto unknown_at = [&](int x, int y) {
        x = std::clamp(x, 0, w - 1);
        y = std::clamp(y, 0, h - 1);
        return kn(x, y) ? 0.0 : 1.0;
    };
    const double nx = (unknown_at(cx + 1, cy) - unknown_at(cx - 1, cy)) / 2.0;
    const double ny = (unknown_at(cx, cy + 1) - unknown_at(cx, cy - 1)) / 2.0;
    const double nlen = std::hypot(nx, ny);
    double data = 1e-3;
    if (best_sq > 0.0 && nlen > 0.0) {
        const double iso_x = -best_gy, iso_y = best_gx;
        data = std::abs(iso_x * nx / nlen + iso_y * ny / nlen) / 255.0 + 1e-3;
    }
    return cterm * data;
}

}  // extern "C"

// ---------------------------------------------------------------- multi-index
struct zo_mi {
    int w = 0, h = 0, C = 1, K = 9, m = 0, mc = 0, dims = 0;
    double coverage = 0.6;
    std::vector<uint32_t> dictionary;
    std::vector<int> rc;  // 8*m*2
    struct layout_index {
        std::vector<double> mean, comp, eig, lo, hi;
        std::vector<uint8_t> coords;
        std::vector<uint32_t> keys;
    } idx[8];
    zo_knn_fn knn_fn = nullptr;  // optional k-NN of a layout (the compiled reference's knn_search)
    void* knn_user = nullptr;
};

extern "C" {

// proj/src/builder.cpp:129-224 (build_index x 8 over one dictionary)
zo_mi* zo_mi_build(const uint8_t* img, const uint8_t* known, int w, int h, int C, int K,
                   double coverage, int dims, const double* pca_mean, const double* pca_comp,
                   int layout_mask, int threads) {
    auto mi = new zo_mi();
    mi->w = w; mi->h = h; mi->C = C; mi->K = K; mi->coverage = coverage;
    mi->m = zo_subset_pixel_count(K, coverage);
    if (mi->m < 1 || K < 3 || K % 2 == 0) { set_err("config: bad K/coverage"); delete mi; return nullptr; }
    mi->mc = mi->m * C;
    mi->rc.resize(static_cast<size_t>(8) * mi->m * 2);
    if (zo_build_subset_layouts(K, coverage, mi->rc.data()) < 0) { delete mi; return nullptr; }
    mi->dictionary.resize(static_cast<size_t>(w) * h);
    const int64_t n = zo_collect_dictionary(known, w, h, K, mi->dictionary.data());
    mi->dictionary.resize(static_cast<size_t>(n));
    if (n == 0) { set_err("no fully known patch window; inpainting impossible"); delete mi; return nullptr; }
    mi->dims = std::min<int64_t>(dims, std::min<int64_t>(mi->mc, n));
    const int F = K * K * C;
    std::vector<int64_t> s, S;
    if (!pca_mean) {
        s.resize(F);
        S.resize(static_cast<size_t>(F) * F);
        zo_patch_moments(img, w, h, C, K, mi->dictionary.data(), n, s.data(), S.data());
    }
    std::vector<int> todo;
    for (int l = 0; l < 8; ++l)
        if (layout_mask & (1 << l)) todo.push_back(l);
    std::vector<int> failed(8, 0);
    auto build_layout = [&](int l) {
        auto& L = mi->idx[l];
        const int* rc = mi->rc.data() + static_cast<size_t>(l) * mi->m * 2;
        L.mean.resize(mi->mc);
        L.comp.resize(static_cast<size_t>(mi->dims) * mi->mc);
        L.eig.assign(mi->dims, 0.0);
        if (pca_mean) {
            std::memcpy(L.mean.data(), pca_mean + static_cast<size_t>(l) * mi->mc, mi->mc * sizeof(double));
            std::memcpy(L.comp.data(), pca_comp + static_cast<size_t>(l) * mi->dims * mi->mc,
                        L.comp.size() * sizeof(double));
        } else {
            std::vector<int> cols;
            for (int p = 0; p < mi->m; ++p)
                for (int ch = 0; ch < C; ++ch) cols.push_back((rc[2 * p] * K + rc[2 * p + 1]) * C + ch);
            std::vector<double> cov(static_cast<size_t>(mi->mc) * mi->mc);
            zo_layout_covariance(s.data(), S.data(), F, n, cols.data(), mi->mc, L.mean.data(), cov.data());
            if (zo_pca_from_cov(cov.data(), mi->mc, mi->dims, L.comp.data(), L.eig.data()) != 0) {
                failed[l] = 1;
                return;
            }
        }
        L.lo.resize(mi->dims);
        L.hi.resize(mi->dims);
        std::vector<uint8_t> coords(static_cast<size_t>(n) * mi->dims);
        zo_project_build(img, w, h, C, mi->dictionary.data(), n, rc, mi->m, L.mean.data(), L.comp.data(),
                         mi->dims, L.lo.data(), L.hi.data(), coords.data(), nullptr);
        L.coords.resize(coords.size());
        L.keys.resize(static_cast<size_t>(n));
        zo_from_descriptors(coords.data(), mi->dictionary.data(), n, mi->dims, L.coords.data(), L.keys.data());
    };
    const int T = std::max(1, std::min<int>(threads, static_cast<int>(todo.size())));
    if (T == 1) {
        for (int l : todo) build_layout(l);
    } else {
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t)
            th.emplace_back([&, t] {
                for (size_t i = t; i < todo.size(); i += T) build_layout(todo[i]);
            });
        for (auto& x : th) x.join();
    }
    for (int l = 0; l < 8; ++l)
        if (failed[l]) {
            set_err("pca: eigen-solve failed");
            delete mi;
            return nullptr;
        }
    return mi;
}

void zo_mi_free(zo_mi* mi) { delete mi; }

void zo_mi_set_knn(zo_mi* mi, zo_knn_fn fn, void* user) {
    mi->knn_fn = fn;
    mi->knn_user = user;
}

void zo_mi_set_layout(zo_mi* mi, int l, const double* mean, const double* comp, const double* lo, const double* hi,
                      const uint8_t* coords, const uint32_t* keys) {
    auto& L = mi->idx[l];
    const size_t n = mi->dictionary.size(), D = static_cast<size_t>(mi->dims), mc = static_cast<size_t>(mi->mc);
    L.mean.assign(mean, mean + mc);
    L.comp.assign(comp, comp + D * mc);
    L.eig.assign(D, 0.0);
    L.lo.assign(lo, lo + D);
    L.hi.assign(hi, hi + D);
    L.coords.assign(coords, coords + n * D);
    L.keys.assign(keys, keys + n);
}
int64_t zo_mi_size(const zo_mi* mi) { return static_cast<int64_t>(mi->dictionary.size()); }
int zo_mi_dims(const zo_mi* mi) { return mi->dims; }
int zo_mi_mc(const zo_mi* mi) { return mi->mc; }
int zo_mi_m(const zo_mi* mi) { return mi->m; }
void zo_mi_dictionary(const zo_mi* mi, uint32_t* keys_out) {
    std::memcpy(keys_out, mi->dictionary.data(), mi->dictionary.size() * sizeof(uint32_t));
}
void zo_mi_layout(const zo_mi* mi, int l, int* rc_out) {
    std::memcpy(rc_out, mi->rc.data() + static_cast<size_t>(l) * mi->m * 2, static_cast<size_t>(mi->m) * 2 * sizeof(int));
}
void zo_mi_pca(const zo_mi* mi, int l, double* mean, double* comp, double* eig, double* lo, double* hi) {
    const auto& L = mi->idx[l];
    if (mean) std::memcpy(mean, L.mean.data(), L.mean.size() * sizeof(double));
    if (comp) std::memcpy(comp, L.comp.data(), L.comp.size() * sizeof(double));
    if (eig) std::memcpy(eig, L.eig.data(), L.eig.size() * sizeof(double));
    if (lo) std::memcpy(lo, L.lo.data(), L.lo.size() * sizeof(double));
    if (hi) std::memcpy(hi, L.hi.data(), L.hi.size() * sizeof(double));
}
void zo_mi_index(const zo_mi* mi, int l, uint8_t* coords_out, uint32_t* keys_out) {
    const auto& L = mi->idx[l];
    std::memcpy(coords_out, L.coords.data(), L.coords.size());
    std::memcpy(keys_out, L.keys.data(), L.keys.size() * sizeof(uint32_t));
}

// proj/src/engine.cpp:178-213 -- select_index, make_query, knn (linear scan == knn_search),
// refine by masked_cost_at keeping min (cost, packed key).
uint64_t zo_mi_query_best_patch(const zo_mi* mi, const uint8_t* img, const uint8_t* tv,
                                const uint8_t* tk, int64_t k, int norm, int* lid_out,
                                int64_t* ncand_out, uint64_t* knn_out) {
    const int lid = zo_select_index(tk, mi->K, mi->rc.data(), mi->m);
    const auto& L = mi->idx[lid];
    std::vector<uint8_t> q(mi->dims);
    zo_make_query(tv, tk, mi->K, mi->C, mi->rc.data() + static_cast<size_t>(lid) * mi->m * 2, mi->m, L.mean.data(),
                  L.comp.data(), L.lo.data(), L.hi.data(), mi->dims, q.data());
    const int64_t n = static_cast<int64_t>(L.keys.size());
    std::vector<uint64_t> cand(static_cast<size_t>(std::min<int64_t>(std::max<int64_t>(k, 1), n)));
    const int64_t cnt = mi->knn_fn ? mi->knn_fn(mi->knn_user, lid, q.data(), k, norm, cand.data())
                                   : zo_knn_linear(L.coords.data(), L.keys.data(), n, mi->dims, q.data(), k, norm,
                                                   cand.data());
    uint64_t best = ~0ull;
    for (int64_t i = 0; i < cnt; ++i) {
        const uint32_t key = static_cast<uint32_t>(cand[i] & 0xffffffffu);
        const uint64_t c = (static_cast<uint64_t>(zo_masked_cost_at(img, mi->w, mi->h, mi->C, tv, tk, mi->K, key, norm)) << 32) | key;
        best = std::min(best, c);
    }
    if (lid_out) *lid_out = lid;
    if (ncand_out) *ncand_out = cnt;
    if (knn_out) std::memcpy(knn_out, cand.data(), static_cast<size_t>(cnt) * sizeof(uint64_t));
    return best;
}

}  // extern "C"

// ---------------------------------------------------------------- fill loop
namespace {

// proj/src/image.cpp:49-61 (4-neighbour fillfront)
bool is_front(const std::vector<uint8_t>& known, int w, int h, int x, int y) {
    auto k = [&](int xx, int yy) { return known[static_cast<size_t>(yy) * w + xx] != 0; };
    if (!k(x, y)) return false;
    return (x > 0 && !k(x - 1, y)) || (x + 1 < w && !k(x + 1, y)) || (y > 0 && !k(x, y - 1)) ||
           (y + 1 < h && !k(x, y + 1));
}

struct by_priority {
    bool operator()(const std::pair<double, uint32_t>& a, const std::pair<double, uint32_t>& b) const {
        if (a.first != b.first) return a.first > b.first;
        return a.second < b.second;
    }
};

// proj/src/engine.cpp:283-369
struct fill_driver {
    std::vector<uint8_t>& img;
    std::vector<uint8_t>& known;
    int w, h, C, K;
    std::vector<double> conf, cached;
    std::vector<uint8_t> in_front;
    std::set<std::pair<double, uint32_t>, by_priority> queue;

    fill_driver(std::vector<uint8_t>& im, std::vector<uint8_t>& kn, int w_, int h_, int C_, int K_)
        : img(im), known(kn), w(w_), h(h_), C(C_), K(K_),
          conf(static_cast<size_t>(w_) * h_, 0.0), cached(static_cast<size_t>(w_) * h_, 0.0),
          in_front(static_cast<size_t>(w_) * h_, 0) {
        for (size_t i = 0; i < conf.size(); ++i) conf[i] = known[i] ? 1.0 : 0.0;
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x)
                if (is_front(known, w, h, x, y)) add(x, y);
    }
    double prio(int x, int y) {
        return zo_compute_priority(img.data(), known.data(), w, h, C, conf.data(), x, y, K);
    }
    void add(int x, int y) {
        const size_t i = static_cast<size_t>(y) * w + x;
        cached[i] = prio(x, y);
        in_front[i] = 1;
        queue.emplace(cached[i], static_cast<uint32_t>(i));
    }
    void remove(int x, int y) {
        const size_t i = static_cast<size_t>(y) * w + x;
        queue.erase({cached[i], static_cast<uint32_t>(i)});
        in_front[i] = 0;
    }
    void refresh(int x, int y) {
        const size_t i = static_cast<size_t>(y) * w + x;
        const double fresh = prio(x, y);
        if (fresh != cached[i]) {
            queue.erase({cached[i], static_cast<uint32_t>(i)});
            cached[i] = fresh;
            queue.emplace(fresh, static_cast<uint32_t>(i));
        }
    }
    // proj/src/engine.cpp:238-257 (paste) + :307-330 (apply_paste refresh)
    int apply_paste(int cx, int cy, uint32_t src, double* center_conf) {
        const int r = (K - 1) / 2;
        const double cc = zo_confidence_term(known.data(), w, h, conf.data(), cx, cy, K);
        int filled = 0;
        const int sx = static_cast<int>(src & 0xffff), sy = static_cast<int>(src >> 16);
        for (int dy = 0; dy < K; ++dy) {
            const int y = cy - r + dy;
            for (int dx = 0; dx < K; ++dx) {
                const int x = cx - r + dx;
                if (x < 0 || x >= w || y < 0 || y >= h || known[static_cast<size_t>(y) * w + x]) continue;
                for (int c = 0; c < C; ++c)
                    img[(static_cast<size_t>(y) * w + x) * C + c] = img[(static_cast<size_t>(sy + dy) * w + sx + dx) * C + c];
                known[static_cast<size_t>(y) * w + x] = 1;
                conf[static_cast<size_t>(y) * w + x] = cc;
                ++filled;
            }
        }
        const int refresh_r = K - 1;
        for (int y = cy - refresh_r; y <= cy + refresh_r; ++y) {
            if (y < 0 || y >= h) continue;
            for (int x = cx - refresh_r; x <= cx + refresh_r; ++x) {
                if (x < 0 || x >= w) continue;
                const size_t i = static_cast<size_t>(y) * w + x;
                const bool zone = std::abs(x - cx) <= r + 1 && std::abs(y - cy) <= r + 1;
                const bool now = zone ? is_front(known, w, h, x, y) : in_front[i] != 0;
                if (in_front[i] && !now) remove(x, y);
                else if (!in_front[i] && now) add(x, y);
                else if (in_front[i] && now) refresh(x, y);
            }
        }
        *center_conf = cc;
        return filled;
    }
};

}  // namespace

extern "C" {

// proj/src/engine.cpp:371-506 (run_loop + inpaint)
int64_t zo_inpaint(const zo_mi* mi, const uint8_t* img0, const uint8_t* known0, int w, int h,
                   int C, int K, int64_t knn, int norm, int brute_force, int oracle,
                   int64_t oracle_stride, uint8_t* img_out, zo_record* records, int64_t cap,
                   int64_t max_iter) {
    std::vector<uint8_t> img(img0, img0 + static_cast<size_t>(w) * h * C);
    std::vector<uint8_t> known(known0, known0 + static_cast<size_t>(w) * h);
    size_t unknown_left = 0;
    for (auto v : known) unknown_left += v == 0;
    if (unknown_left == 0) {
        std::memcpy(img_out, img.data(), img.size());
        return 0;
    }
    std::vector<uint32_t> dictionary;
    if (mi) dictionary = mi->dictionary;
    else {
        dictionary.resize(static_cast<size_t>(w) * h);
        dictionary.resize(static_cast<size_t>(zo_collect_dictionary(known0, w, h, K, dictionary.data())));
        if (dictionary.empty()) { set_err("no fully known patch window; inpainting impossible"); return -1; }
    }
    fill_driver drv(img, known, w, h, C, K);
    std::vector<uint8_t> tv(static_cast<size_t>(K) * K * C), tk(static_cast<size_t>(K) * K);
    int64_t it = 0;
    while (unknown_left > 0 && (max_iter <= 0 || it < max_iter)) {
        if (drv.queue.empty()) { set_err("inpaint: unknown pixels unreachable from the fillfront"); return -1; }
        const uint32_t pos = drv.queue.begin()->second;
        const int tx = static_cast<int>(pos % w), ty = static_cast<int>(pos / w);
        zo_extract_patch_clamped(img.data(), known.data(), w, h, C, tx, ty, K, tv.data(), tk.data());
        uint64_t best;
        int lid = 0;
        int64_t ncand;
        if (brute_force) {
            best = zo_brute_force_best(img.data(), w, h, C, tv.data(), tk.data(), K, dictionary.data(),
                                       static_cast<int64_t>(dictionary.size()), norm);
            ncand = static_cast<int64_t>(dictionary.size());
        } else {
            best = zo_mi_query_best_patch(mi, img.data(), tv.data(), tk.data(), knn, norm, &lid, &ncand, nullptr);
        }
        const uint32_t cost = static_cast<uint32_t>(best >> 32);
        const uint32_t src = static_cast<uint32_t>(best & 0xffffffffu);
        zo_record rec{};
        rec.tx = tx; rec.ty = ty; rec.layout_id = lid;
        rec.sx = static_cast<int>(src & 0xffff); rec.sy = static_cast<int>(src >> 16);
        rec.cost = cost;
        rec.z_error = norm == 0 ? std::sqrt(static_cast<double>(cost)) : static_cast<double>(cost);
        rec.bf_error = std::numeric_limits<double>::quiet_NaN();
        rec.candidates = ncand;
        if (oracle && !brute_force && it % std::max<int64_t>(1, oracle_stride) == 0) {
            const uint64_t o = zo_brute_force_best(img.data(), w, h, C, tv.data(), tk.data(), K, dictionary.data(),
                                                   static_cast<int64_t>(dictionary.size()), norm);
            const uint32_t oc = static_cast<uint32_t>(o >> 32);
            rec.bf_error = norm == 0 ? std::sqrt(static_cast<double>(oc)) : static_cast<double>(oc);
        } else if (brute_force) {
            rec.bf_error = rec.z_error;
        }
        double cc;
        unknown_left -= static_cast<size_t>(drv.apply_paste(tx, ty, src, &cc));
        if (records && it < cap) records[it] = rec;
        ++it;
    }
    std::memcpy(img_out, img.data(), img.size());
    return it;
}

}  // extern "C"

// ---------------------------------------------------------------- cfg5 vector index
// Test infrastructure: the canonical order the device build (k_vector.cu) is pinned to.
// proj/src/pca.cpp:20-37 (mean, covariance) restated with a fixed summation order.
extern "C" void zo_vec_mean_cov(const float* X, int64_t n, int dim, int64_t stripe, double* mean, double* cov) {
    std::vector<double> tot(dim, 0.0);
    const int64_t sub = 4096;  // stripe sums add their 4096-row sub-chunk sums in order
    for (int64_t s0 = 0; s0 < n; s0 += stripe) {
        const int64_t s1 = std::min<int64_t>(n, s0 + stripe);
        for (int j = 0; j < dim; ++j) {
            double st = 0.0;
            for (int64_t u0 = s0; u0 < s1; u0 += sub) {
                const int64_t u1 = std::min<int64_t>(s1, u0 + sub);
                double s = 0.0;
                for (int64_t r = u0; r < u1; ++r) s += static_cast<double>(X[r * dim + j]);
                st += s;
            }
            tot[j] += st;
        }
    }
    for (int j = 0; j < dim; ++j) mean[j] = tot[j] / static_cast<double>(n);
    std::vector<double> G(static_cast<size_t>(dim) * dim, 0.0), Gs(static_cast<size_t>(dim) * dim);
    std::vector<double> xc(dim);
    for (int64_t s0 = 0; s0 < n; s0 += stripe) {
        const int64_t s1 = std::min<int64_t>(n, s0 + stripe);
        std::fill(Gs.begin(), Gs.end(), 0.0);
        for (int64_t r = s0; r < s1; ++r) {
            for (int j = 0; j < dim; ++j) xc[j] = static_cast<double>(X[r * dim + j]) - mean[j];
            for (int i = 0; i < dim; ++i)
                for (int j = i; j < dim; ++j) Gs[static_cast<size_t>(i) * dim + j] = std::fma(xc[i], xc[j], Gs[static_cast<size_t>(i) * dim + j]);
        }
        for (size_t q = 0; q < G.size(); ++q) G[q] += Gs[q];
    }
    for (int i = 0; i < dim; ++i)
        for (int j = i; j < dim; ++j) {
            const double g = G[static_cast<size_t>(i) * dim + j];
            const double v = n > 1 ? g / static_cast<double>(n - 1) : g;
            cov[static_cast<size_t>(i) * dim + j] = v;
            cov[static_cast<size_t>(j) * dim + i] = v;
        }
}

// proj/src/pca.cpp:7-11 + builder.cpp:55-61,159-187 for vectors
extern "C" void zo_vec_project(const float* X, int64_t n, int dim, const double* mean, const double* comp, int D,
                               double* lo, double* hi, uint8_t* coords) {
    std::vector<double> y(static_cast<size_t>(n) * D);
    for (int d = 0; d < D; ++d) {
        lo[d] = std::numeric_limits<double>::infinity();
        hi[d] = -std::numeric_limits<double>::infinity();
    }
    for (int64_t r = 0; r < n; ++r)
        for (int d = 0; d < D; ++d) {
            double acc = 0.0;
            for (int j = 0; j < dim; ++j)
                acc = std::fma(comp[static_cast<size_t>(d) * dim + j], static_cast<double>(X[r * dim + j]) - mean[j], acc);
            y[static_cast<size_t>(r) * D + d] = acc;
            lo[d] = std::min(lo[d], acc);
            hi[d] = std::max(hi[d], acc);
        }
    for (int64_t r = 0; r < n; ++r)
        for (int d = 0; d < D; ++d) coords[r * D + d] = zo_quantize(lo[d], hi[d], y[static_cast<size_t>(r) * D + d]);
}

// proj/src/builder.cpp:110-127 for vectors: unknown coordinate -> mean
extern "C" void zo_vec_make_query(const float* x, const uint8_t* known, int dim, const double* mean, const double* comp,
                                  const double* lo, const double* hi, int D, uint8_t* out) {
    for (int d = 0; d < D; ++d) {
        double acc = 0.0;
        for (int j = 0; j < dim; ++j) {
            const double v = known[j] ? static_cast<double>(x[j]) : mean[j];
            acc = std::fma(comp[static_cast<size_t>(d) * dim + j], v - mean[j], acc);
        }
        out[d] = zo_quantize(lo[d], hi[d], acc);
    }
}
