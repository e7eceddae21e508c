// host_pca.cpp -- host side of the index build: subset layouts, config validation and the
// PCA eigen-solve over the device-computed exact moments.
//
//   subset_pixel_count / build_subset_layouts    proj/src/layouts.cpp:9-60
//   index_config::validate                       proj/src/builder.cpp:38-53
//   pca_accumulator::finish_mean / finalize      proj/src/pca.cpp:26-67
//
// The covariance of each layout is a sub-block of ONE exact int64 Gram of the full K*K*C
// patch vector (computed on the GPU, k_build.cu), so it is order-free and reproducible:
//   mean_j = s_j / n,   cov_ij = (n*S_ij - s_i*s_j) / (n*(n-1))   (int128 numerator).
// Eigen's SelfAdjointEigenSolver is replaced by Householder tridiagonalisation, Sturm
// bisection for the top-D eigenvalues and inverse iteration with in-cluster
// re-orthogonalisation, then the reference's ordering / sign / clamp rules.
#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <vector>

#include "zi_internal.h"

namespace zi {

int subset_pixel_count(int K, double c) { return static_cast<int>(std::llround(c * K * K)); }

void layout_anchors(int K, int32_t* rc) {
    const int mid = (K - 1) / 2;
    // edge midpoints N, E, S, W then corners NW, NE, SW, SE
    const int a[8][2] = {{0, mid}, {mid, K - 1}, {K - 1, mid}, {mid, 0}, {0, 0}, {0, K - 1}, {K - 1, 0}, {K - 1, K - 1}};
    for (int l = 0; l < 8; ++l) {
        rc[2 * l] = a[l][0];
        rc[2 * l + 1] = a[l][1];
    }
}

int subset_layouts(int K, double c, std::vector<int32_t>& rc) {
    if (K < 3 || K % 2 == 0) throw error(ZI_E_INVALID, "subset layouts: K must be odd and >= 3");
    if (!(c > 0.0 && c <= 1.0)) throw error(ZI_E_INVALID, "subset layouts: coverage must be in (0, 1]");
    const int count = subset_pixel_count(K, c);
    if (count < 1) throw error(ZI_E_INVALID, "subset layouts: coverage keeps no pixels");
    int32_t anch[16];
    layout_anchors(K, anch);
    const int(*anchors)[2] = reinterpret_cast<const int(*)[2]>(anch);
    rc.assign(static_cast<size_t>(8) * count * 2, 0);
    std::vector<int> order(static_cast<size_t>(K) * K);
    for (int id = 0; id < 8; ++id) {
        const int ar = anchors[id][0], ac = anchors[id][1];
        std::iota(order.begin(), order.end(), 0);  // row-major offsets
        auto dist = [&](int o) {
            const int r = o / K, cc = o % K;
            return (r - ar) * (r - ar) + (cc - ac) * (cc - ac);
        };
        // nearest `count` offsets, distance ties in row-major order, then row-major again
        std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return dist(a) < dist(b); });
        std::vector<int> keep(order.begin(), order.begin() + count);
        std::sort(keep.begin(), keep.end());
        for (int i = 0; i < count; ++i) {
            rc[(static_cast<size_t>(id) * count + i) * 2] = keep[i] / K;
            rc[(static_cast<size_t>(id) * count + i) * 2 + 1] = keep[i] % K;
        }
    }
    return count;
}

void validate_config(const zi_index_config& cfg, int channels) {
    if (cfg.patch_size < 3 || cfg.patch_size % 2 == 0)
        throw error(ZI_E_INVALID, "config: patch size K must be odd and >= 3");
    if (!(cfg.coverage > 0.0 && cfg.coverage <= 1.0)) throw error(ZI_E_INVALID, "config: coverage c must be in (0, 1]");
    const int subset = subset_pixel_count(cfg.patch_size, cfg.coverage);
    if (subset < 1) throw error(ZI_E_INVALID, "config: coverage keeps no pixels");
    const int input_dim = subset * channels;
    if (cfg.dims < 1 || cfg.dims > input_dim)
        throw error(ZI_E_INVALID, "config: dims D must be in [1, subset pixels * channels]");
    if (cfg.dims > 32) throw error(ZI_E_INVALID, "config: dims D above the supported maximum of 32");
    if (cfg.knn < 1) throw error(ZI_E_INVALID, "config: k must be >= 1");
    if (cfg.mu < 1) throw error(ZI_E_INVALID, "config: mu must be >= 1");
    if (cfg.nu < cfg.mu) throw error(ZI_E_INVALID, "config: nu must be >= mu");
}

namespace {

// Dot product with 8 independent partial sums (a fixed, deterministic association that lets
// the compiler use AVX lanes despite -ffp-contract=off and strict IEEE semantics).
inline double dot8(const double* a, const double* b, int m) {
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int j = 0;
    for (; j + 8 <= m; j += 8)
        for (int t = 0; t < 8; ++t) acc[t] += a[j + t] * b[j + t];
    for (; j < m; ++j) acc[j & 7] += a[j] * b[j];
    return ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
}

// Householder reduction A = Q T Q^T (row-major n x n, lower triangle used, destroyed).
// Reflector k acts on rows/cols k+1..n-1: H_k = I - tau_k v_k v_k^T.
struct tridiag {
    int n;
    std::vector<double> d, e;              // diagonal, sub-diagonal (n-1)
    std::vector<std::vector<double>> v;    // reflectors
    std::vector<double> tau;
};

tridiag householder(std::vector<double>& A, int n) {
    tridiag t;
    t.n = n;
    t.d.assign(n, 0.0);
    t.e.assign(n > 1 ? n - 1 : 1, 0.0);
    t.v.resize(n > 2 ? n - 2 : 0);
    t.tau.assign(n > 2 ? n - 2 : 0, 0.0);
    std::vector<double> p(n), w(n);
    for (int k = 0; k + 2 < n; ++k) {
        const int m = n - k - 1;  // length of the column below the diagonal
        double norm2 = 0.0;
        for (int i = 0; i < m; ++i) norm2 += A[static_cast<size_t>(k + 1 + i) * n + k] * A[static_cast<size_t>(k + 1 + i) * n + k];
        const double x0 = A[static_cast<size_t>(k + 1) * n + k];
        auto& v = t.v[k];
        v.assign(m, 0.0);
        if (norm2 == 0.0) {
            t.e[k] = 0.0;
            t.tau[k] = 0.0;
            continue;
        }
        const double alpha = x0 >= 0 ? -std::sqrt(norm2) : std::sqrt(norm2);
        for (int i = 0; i < m; ++i) v[i] = A[static_cast<size_t>(k + 1 + i) * n + k];
        v[0] -= alpha;
        const double vtv = dot8(v.data(), v.data(), m);
        if (vtv == 0.0) {
            t.e[k] = x0;
            t.tau[k] = 0.0;
            continue;
        }
        const double tau = 2.0 / vtv;
        t.tau[k] = tau;
        t.e[k] = alpha;
        // p = tau * A22 v from the lower triangle only: row i contributes its prefix dot
        // product to p[i] and, transposed, an axpy into p[0..i-1]
        for (int i = 0; i < m; ++i) {
            const double* row = &A[static_cast<size_t>(k + 1 + i) * n + k + 1];
            p[i] = dot8(row, v.data(), i + 1);
            const double vi = v[i];
            for (int j = 0; j < i; ++j) p[j] += row[j] * vi;
        }
        for (int i = 0; i < m; ++i) p[i] *= tau;
        const double vp = dot8(v.data(), p.data(), m);
        const double K2 = 0.5 * tau * vp;
        for (int i = 0; i < m; ++i) w[i] = p[i] - K2 * v[i];
        // A22 -= v w^T + w v^T  (lower triangle)
        for (int i = 0; i < m; ++i) {
            double* row = &A[static_cast<size_t>(k + 1 + i) * n + k + 1];
            const double vi = v[i], wi = w[i];
            for (int j = 0; j <= i; ++j) row[j] -= vi * w[j] + wi * v[j];
        }
    }
    for (int i = 0; i < n; ++i) t.d[i] = A[static_cast<size_t>(i) * n + i];
    if (n >= 2) t.e[n - 2] = A[static_cast<size_t>(n - 1) * n + n - 2];
    return t;
}

// solve (T - sigma I) x = b in place (tridiagonal LU with partial pivoting)
void tri_solve(const tridiag& t, double sigma, double tiny, std::vector<double>& b) {
    const int n = t.n;
    std::vector<double> u1(n), u2(n, 0.0), u3(n, 0.0), mult(n, 0.0);
    std::vector<char> piv(n, 0);
    double dcur = t.d[0] - sigma;
    double scur = n > 1 ? t.e[0] : 0.0;
    for (int i = 0; i + 1 < n; ++i) {
        const double a = t.e[i];  // sub-diagonal entry of row i+1
        const double bn = t.d[i + 1] - sigma;
        const double cn = i + 2 < n ? t.e[i + 1] : 0.0;
        if (std::fabs(dcur) >= std::fabs(a)) {
            if (dcur == 0.0) dcur = tiny;
            const double m = a / dcur;
            u1[i] = dcur;
            u2[i] = scur;
            u3[i] = 0.0;
            mult[i] = m;
            piv[i] = 0;
            dcur = bn - m * scur;
            scur = cn;
        } else {
            const double m = dcur / a;
            u1[i] = a;
            u2[i] = bn;
            u3[i] = cn;
            mult[i] = m;
            piv[i] = 1;
            dcur = scur - m * bn;
            scur = -m * cn;
        }
    }
    if (dcur == 0.0) dcur = tiny;
    u1[n - 1] = dcur;
    for (int i = 0; i + 1 < n; ++i) {
        if (piv[i]) std::swap(b[i], b[i + 1]);
        b[i + 1] -= mult[i] * b[i];
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = b[i];
        if (i + 1 < n) s -= u2[i] * b[i + 1];
        if (i + 2 < n) s -= u3[i] * b[i + 2];
        double piv_ = u1[i];
        if (std::fabs(piv_) < tiny) piv_ = piv_ < 0 ? -tiny : tiny;
        b[i] = s / piv_;
    }
}

}  // namespace

void pca_fit_layout(const std::vector<int64_t>& s, const std::vector<int64_t>& S, int F, uint64_t n,
                    const std::vector<int32_t>& cols, int dims, std::vector<double>& mean, std::vector<double>& comp,
                    std::vector<double>& eig) {
    const int mc = static_cast<int>(cols.size());
    mean.assign(mc, 0.0);
    for (int i = 0; i < mc; ++i) mean[i] = static_cast<double>(s[cols[i]]) / static_cast<double>(n);
    std::vector<double> A(static_cast<size_t>(mc) * mc);
    const double den = n > 1 ? static_cast<double>(n) * static_cast<double>(n - 1) : 1.0;
    for (int i = 0; i < mc; ++i)
        for (int j = 0; j < mc; ++j) {
            const __int128 num = static_cast<__int128>(n) * S[static_cast<size_t>(cols[i]) * F + cols[j]] -
                                 static_cast<__int128>(s[cols[i]]) * s[cols[j]];
            A[static_cast<size_t>(i) * mc + j] = static_cast<double>(num) / den;
        }
    comp.assign(static_cast<size_t>(dims) * mc, 0.0);
    eig.assign(dims, 0.0);
    if (mc == 1) {
        comp[0] = 1.0;
        eig[0] = std::max(0.0, A[0]);
        return;
    }
    const tridiag t = householder(A, mc);
    double tnorm = 0.0;
    for (int i = 0; i < mc; ++i) {
        const double r = std::fabs(t.d[i]) + (i > 0 ? std::fabs(t.e[i - 1]) : 0.0) + (i + 1 < mc ? std::fabs(t.e[i]) : 0.0);
        tnorm = std::max(tnorm, r);
    }
    const double eps = std::numeric_limits<double>::epsilon();
    const double safe = tnorm > 0 ? tnorm : 1.0;
    const double pivmin = std::numeric_limits<double>::min() * 1e4 * std::max(1.0, safe * safe);
    double gl = -safe, gu = safe;
    for (int i = 0; i < mc; ++i) {
        const double r = (i > 0 ? std::fabs(t.e[i - 1]) : 0.0) + (i + 1 < mc ? std::fabs(t.e[i]) : 0.0);
        gl = std::min(gl, t.d[i] - r);
        gu = std::max(gu, t.d[i] + r);
    }
    gl -= 2 * eps * safe + pivmin;
    gu += 2 * eps * safe + pivmin;
    // top-D eigenvalues, descending (index mc-1-j among ascending): D independent Sturm
    // bisections advanced together so the divide chains overlap (identical arithmetic per chain)
    std::vector<double> lam(dims), blo(dims, gl), bhi(dims, gu), mid(dims), q(dims);
    std::vector<int> cnt(dims);
    std::vector<char> active(dims, 1);
    std::vector<double> e2(mc > 1 ? mc - 1 : 1);
    for (int i = 0; i + 1 < mc; ++i) e2[i] = t.e[i] * t.e[i];
    for (int it = 0; it < 256; ++it) {
        int nact = 0;
        for (int j = 0; j < dims; ++j) {
            if (!active[j]) continue;
            const double lo = blo[j], hi = bhi[j];
            const double md = 0.5 * (lo + hi);
            if (md <= lo || md >= hi || hi - lo <= 2 * eps * std::max(std::fabs(lo), std::fabs(hi)) + pivmin) {
                active[j] = 0;
                continue;
            }
            mid[j] = md;
            ++nact;
        }
        if (nact == 0) break;
        for (int j = 0; j < dims; ++j) {
            q[j] = t.d[0] - mid[j];
            if (std::fabs(q[j]) < pivmin) q[j] = -pivmin;
            cnt[j] = q[j] < 0;
        }
        for (int i = 1; i < mc; ++i) {
            const double di = t.d[i], ei = e2[i - 1];
            for (int j = 0; j < dims; ++j) {
                double v = di - mid[j] - ei / q[j];
                if (std::fabs(v) < pivmin) v = -pivmin;
                q[j] = v;
                cnt[j] += v < 0;
            }
        }
        for (int j = 0; j < dims; ++j) {
            if (!active[j]) continue;
            if (cnt[j] > mc - 1 - j) bhi[j] = mid[j];
            else blo[j] = mid[j];
        }
    }
    for (int j = 0; j < dims; ++j) lam[j] = 0.5 * (blo[j] + bhi[j]);
    // inverse iteration, re-orthogonalised inside clusters of close eigenvalues
    const double tiny = eps * safe;
    const double cluster = 1e-3 * safe;
    std::vector<std::vector<double>> z(dims, std::vector<double>(mc));
    double sigma_prev = 0.0;
    for (int j = 0; j < dims; ++j) {
        double sigma = lam[j];
        if (j > 0 && std::fabs(sigma - sigma_prev) < 10 * tiny) sigma = sigma_prev - 10 * tiny;
        sigma_prev = sigma;
        std::vector<double>& x = z[j];
        for (int i = 0; i < mc; ++i) x[i] = 1.0 + 0.5 * std::sin(0.7 * i + 1.3 * j + 0.1);
        for (int it = 0; it < 5; ++it) {
            double nrm = 0.0;
            for (double vv : x) nrm += vv * vv;
            nrm = std::sqrt(nrm);
            for (double& vv : x) vv /= nrm;
            tri_solve(t, sigma, tiny, x);
            for (int p = 0; p < j; ++p) {
                if (std::fabs(lam[p] - lam[j]) > cluster) continue;
                double dot = 0.0;
                for (int i = 0; i < mc; ++i) dot += z[p][i] * x[i];
                for (int i = 0; i < mc; ++i) x[i] -= dot * z[p][i];
            }
        }
        double nrm = 0.0;
        for (double vv : x) nrm += vv * vv;
        nrm = std::sqrt(nrm);
        for (double& vv : x) vv /= nrm;
    }
    // back-transform x = H_0 H_1 ... H_{n-3} z, sign rule, clamp (proj/src/pca.cpp:55-65)
    for (int j = 0; j < dims; ++j) {
        std::vector<double>& x = z[j];
        for (int k = mc - 3; k >= 0; --k) {
            if (t.tau[k] == 0.0) continue;
            const auto& v = t.v[k];
            const int m = mc - k - 1;
            const double f = t.tau[k] * dot8(v.data(), &x[k + 1], m);
            for (int i = 0; i < m; ++i) x[k + 1 + i] -= f * v[i];
        }
        int arg = 0;
        for (int i = 1; i < mc; ++i)
            if (std::fabs(x[i]) > std::fabs(x[arg])) arg = i;
        const double sgn = x[arg] < 0 ? -1.0 : 1.0;
        for (int i = 0; i < mc; ++i) comp[static_cast<size_t>(j) * mc + i] = sgn * x[i];
        eig[j] = std::max(0.0, lam[j]);
    }
}

}  // namespace zi
