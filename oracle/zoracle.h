/*
 * zoracle.h -- CPU restatement of the reference (`zinpaint`, arXiv 1712.06326) hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_1712_06326_b200/) may
 * include, link or call this; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg use it, and only as the checker or the timed
 * CPU baseline.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj).  The Eigen-dependent parts of the reference (pca.cpp,
 * builder.cpp, engine.cpp) cannot be compiled here (Eigen is absent), so they are
 * restated with a pinned canonical fp64 order:
 *   mean_j  = (double)s_j / (double)n                      (exact int64 column sums)
 *   cov_ij  = (double)(n*S_ij - s_i*s_j) / ((double)n*(double)(n-1))   (int128 numerator)
 *   xc_j    = (double)x_j - mean_j
 *   y_d     = fma(comp[d][j], xc_j, y_d)   for j = 0 .. m*C-1 in order, y_d starting at +0.0
 * The parts that do compile (zcurve.cpp, layouts.cpp, image.cpp, pool.cpp) are built
 * unmodified into oracle/_ref/libzref.so (see ref_shim.cpp) and pin this restatement.
 */
#ifndef ZORACLE_H
#define ZORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- layouts (proj/src/layouts.cpp:9-60) ---- */
int zo_subset_pixel_count(int K, double coverage);
/* rc_out: 8 * m * 2 ints (row, col) per layout in row-major order; returns m or -1 */
int zo_build_subset_layouts(int K, double coverage, int* rc_out);

/* ---- Morton order (proj/include/zinpaint/morton.hpp:10-29) ---- */
int zo_less_msb(int a, int b);
int zo_morton_less(const uint8_t* a, const uint8_t* b, int dims);

/* ---- dictionary (proj/src/builder.cpp:74-108); keys packed y<<16|x; returns n ---- */
int64_t zo_collect_dictionary(const uint8_t* known, int w, int h, int K, uint32_t* keys_out);

/* ---- exact moments of the full K*K*C patch vector over the dictionary ----
 * column f = (r*K + c)*C + ch; s_out[F], S_out[F*F] with F = K*K*C */
void zo_patch_moments(const uint8_t* img, int w, int h, int C, int K, const uint32_t* keys,
                      int64_t n, int64_t* s_out, int64_t* S_out);

/* mean and covariance of one layout's columns (proj/src/pca.cpp:20-37,45-46) */
void zo_layout_covariance(const int64_t* s, const int64_t* S, int F, int64_t n, const int* cols,
                          int mc, double* mean_out, double* cov_out);

/* eigen-decomposition + top-D + sign rule + eigenvalue clamp (proj/src/pca.cpp:39-67).
 * comp_out is D rows of mc (row d = component d).  Jacobi; returns 0 or -1 */
int zo_pca_from_cov(const double* cov, int mc, int D, double* comp_out, double* eig_out);

/* ---- quantiser (proj/src/builder.cpp:55-61) ---- */
uint8_t zo_quantize(double lo, double hi, double y);

/* ---- projection (passes 3-4, proj/src/builder.cpp:159-187) ----
 * rc: m (row,col) pairs of the layout; mean[mc]; comp[D*mc]. Writes lo/hi[D],
 * coords_out[n*D] (dictionary order) and, if y_out != NULL, the fp64 projections [n*D]. */
void zo_project_build(const uint8_t* img, int w, int h, int C, const uint32_t* keys, int64_t n,
                      const int* rc, int m, const double* mean, const double* comp, int D,
                      double* lo, double* hi, uint8_t* coords_out, double* y_out);

/* ---- z-curve sort (proj/src/zcurve.cpp:108-138): returns 0, or -1 on bad dims ---- */
int zo_from_descriptors(const uint8_t* coords, const uint32_t* keys, int64_t n, int D,
                        uint8_t* coords_out, uint32_t* keys_out);

/* ---- exact knn by linear scan (proj/tests/support/oracles.hpp:55-74), which the
 * reference proves equal to knn_search (proj/tests/unit/test_zcurve.cpp:347-373).
 * out: packed (dist<<32 | key) ascending; returns count = min(k, n) ---- */
int64_t zo_knn_linear(const uint8_t* coords, const uint32_t* keys, int64_t n, int D,
                      const uint8_t* query, int64_t k, int norm, uint64_t* out);

/* ---- query side (proj/src/engine.cpp:162-176; proj/src/builder.cpp:110-127) ---- */
int zo_select_index(const uint8_t* target_known, int K, const int* layouts_rc, int m);
void zo_make_query(const uint8_t* tv, const uint8_t* tk, int K, int C, const int* rc, int m,
                   const double* mean, const double* comp, const double* lo, const double* hi,
                   int D, uint8_t* out);

/* ---- costs (proj/src/engine.cpp:48-76, 220-236); norm 0 = L2, 1 = L1 ---- */
uint32_t zo_masked_cost_at(const uint8_t* img, int w, int h, int C, const uint8_t* tv,
                           const uint8_t* tk, int K, uint32_t key, int norm);
/* returns packed (cost<<32 | key) of the best dictionary patch */
uint64_t zo_brute_force_best(const uint8_t* img, int w, int h, int C, const uint8_t* tv,
                             const uint8_t* tk, int K, const uint32_t* keys, int64_t n, int norm);

/* ---- target extraction (proj/src/image.cpp:7-47) ---- */
void zo_extract_patch_clamped(const uint8_t* img, const uint8_t* known, int w, int h, int C,
                              int cx, int cy, int K, uint8_t* tv, uint8_t* tk);

/* ---- priority pieces (proj/src/engine.cpp:83-146) ---- */
double zo_confidence_term(const uint8_t* known, int w, int h, const double* conf, int cx, int cy,
                          int K);
double zo_compute_priority(const uint8_t* img, const uint8_t* known, int w, int h, int C,
                           const double* conf, int cx, int cy, int K);

/* ---- multi-index + fill loop ---- */
typedef struct zo_mi zo_mi;
/* pca_mean: 8*mc doubles, pca_comp: 8*D*mc doubles (row-major per layout) or NULL for the
 * oracle's own Jacobi fit.  layout_mask: bit l set -> build layout l (0xff: all eight; the
 * others stay empty); threads: layouts built concurrently (the reference builds the eight
 * indices on its priority_pool, proj/src/builder.cpp:212-218; results do not depend on it).
 * Returns NULL on error (zo_error() tells why). */
zo_mi* zo_mi_build(const uint8_t* img, const uint8_t* known, int w, int h, int C, int K,
                   double coverage, int dims, const double* pca_mean, const double* pca_comp,
                   int layout_mask, int threads);
void zo_mi_free(zo_mi* mi);
/* k-NN of layout `layout` for the fill loop: packed (dist<<32|key) ascending into out, returns the
 * count.  Default (fn NULL): the linear scan.  bench.py plugs in the compiled reference's
 * knn_search (oracle/_ref, zr_hook_knn) to time the reference's own fill loop query. */
typedef int64_t (*zo_knn_fn)(void* user, int layout, const uint8_t* query, int64_t k, int norm, uint64_t* out);
void zo_mi_set_knn(zo_mi* mi, zo_knn_fn fn, void* user);
/* replace layout l's model, quantiser and sorted index (n = dictionary size entries) */
void zo_mi_set_layout(zo_mi* mi, int l, const double* mean, const double* comp, const double* lo,
                      const double* hi, const uint8_t* coords, const uint32_t* keys);
int64_t zo_mi_size(const zo_mi* mi);
int zo_mi_dims(const zo_mi* mi);
int zo_mi_mc(const zo_mi* mi);
int zo_mi_m(const zo_mi* mi);
void zo_mi_dictionary(const zo_mi* mi, uint32_t* keys_out);
void zo_mi_layout(const zo_mi* mi, int l, int* rc_out);
void zo_mi_pca(const zo_mi* mi, int l, double* mean, double* comp, double* eig, double* lo,
               double* hi);
void zo_mi_index(const zo_mi* mi, int l, uint8_t* coords_out, uint32_t* keys_out);
/* query_best_patch (proj/src/engine.cpp:178-213): returns packed (cost<<32|key);
 * lid/ncand out; knn_out (optional, k entries) receives the sorted candidate list */
uint64_t zo_mi_query_best_patch(const zo_mi* mi, const uint8_t* img, const uint8_t* tv,
                                const uint8_t* tk, int64_t k, int norm, int* lid_out,
                                int64_t* ncand_out, uint64_t* knn_out);

typedef struct {
    int32_t tx, ty;
    int32_t layout_id;
    int32_t sx, sy;
    uint32_t cost;
    double z_error;
    double bf_error; /* NaN when not instrumented */
    int64_t candidates;
} zo_record;

/* inpaint / run_loop (proj/src/engine.cpp:371-506).  mi may be NULL when brute_force.
 * max_iter > 0 stops after that many iterations (a prefix of the full run; img_out then holds
 * the partially filled picture) -- test-only, the reference always runs to completion.
 * Returns number of records (iterations) or -1 (error; zo_error()). */
int64_t zo_inpaint(const zo_mi* mi, const uint8_t* img, const uint8_t* known, int w, int h,
                   int C, int K, int64_t knn, int norm, int brute_force, int oracle,
                   int64_t oracle_stride, uint8_t* img_out, zo_record* records, int64_t cap,
                   int64_t max_iter);

/* cfg5 vector index, in the canonical fp64 order of paper_1712_06326_b200/csrc/k_vector.cu:
 * column sums and the Gram as row-ordered chains inside stripes of `stripe` rows, stripe
 * partials added in order; cov = G / (n - 1).  comp: D rows of dim (the reference's columns). */
void zo_vec_mean_cov(const float* X, int64_t n, int dim, int64_t stripe, double* mean, double* cov);
void zo_vec_project(const float* X, int64_t n, int dim, const double* mean, const double* comp, int D,
                    double* lo, double* hi, uint8_t* coords);
void zo_vec_make_query(const float* x, const uint8_t* known, int dim, const double* mean, const double* comp,
                       const double* lo, const double* hi, int D, uint8_t* out);

const char* zo_error(void);

#ifdef __cplusplus
}
#endif
#endif
