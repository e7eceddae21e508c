// k_pca.cu -- the PCA fit of the 8 layout indices on the device (proj/src/pca.cpp:26-67).
//
// Input: the exact int64 moments (s, S) of the full K*K*C patch vector (k_build.cu).  Each
// layout's covariance cov_ij = (n*S_ij - s_i*s_j) / (n*(n-1)) comes from the int128 numerator with
// a correctly rounded int128 -> double conversion.  Three kernels, no host round trip:
//
//   k_pca_tri  one 8-CTA thread-block cluster per layout.  Householder tridiagonalisation with the
//              full symmetric matrix distributed by rows over the cluster (row i on CTA i % 8, 28
//              rows x 219 columns = 48 KB per CTA).  Per column: the pivot row's owner forms the
//              reflector and broadcasts it through distributed shared memory; every CTA forms its
//              rows of p = tau*A*v and broadcasts them; after a second cluster barrier every CTA
//              applies the rank-2 update to its own rows.  v / p are double-buffered by column
//              parity so two cluster barriers per column suffice.  Writes d, e, tau, reflectors.
//   k_pca_vec  one CTA per (layout, component): the reflectors stream into shared memory by one
//              TMA bulk copy while 128 lanes run multisection on Sturm counts for lambda_j; one
//              thread then runs inverse iteration (LU factored once, 3 solves); one warp applies
//              the reflectors with the vector held in registers.
//   k_pca_fin  one CTA per layout: Gram-Schmidt inside clusters of close eigenvalues, the
//              reference's sign rule (first max-|v| entry positive), eigenvalue clamp at 0, and
//              the components written straight into the projection kernels' [j][d] layout.
//   k_pca_lz   (first, when ZI_PCA_LZ is not 0) the Lanczos fast path: K = max(32, 2D+8) steps
//              with full reorthogonalisation on the same distributed rows, then k_pca_vec in
//              Lanczos mode solves T_K and forms the Ritz vectors; a layout whose Ritz residuals
//              are not below 1e-10 |T| (or whose Krylov space broke down early) runs the
//              Householder kernels above, which skip every layout the fast path delivered.
// The host eigen-solver (host_pca.cpp) remains for m*C > 224.
#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace zi {

namespace cg = cooperative_groups;

constexpr int kCl = 8;             // CTAs per layout (one cluster; 4: 0.67 ms, 16: 1.26 ms, 8: 0.58 ms on cfg2)
constexpr int kTriThreads = 512;
constexpr int kVecThreads = 128;
constexpr int kPcaMaxN = 224;
constexpr int kSlots = (kPcaMaxN + 31) / 32;  // vector entries per lane in the back-transform

// reflector k (entries k+1 .. n-1 of column k) starts at refl_off(k)
__host__ __device__ inline size_t refl_off(int k, int n) {
    return static_cast<size_t>(k) * static_cast<size_t>(2 * n - k - 1) / 2;
}
__host__ __device__ inline size_t refl_stride(int n) { return (refl_off(n - 2, n) + 1) & ~static_cast<size_t>(1); }

// correctly rounded (RN) conversion of a signed 128-bit integer
__device__ inline double i128_to_double(__int128 x) {
    if (x == 0) return 0.0;
    const bool neg = x < 0;
    unsigned __int128 u = neg ? static_cast<unsigned __int128>(-x) : static_cast<unsigned __int128>(x);
    const unsigned long long hi = static_cast<unsigned long long>(u >> 64);
    double r;
    if (hi == 0) {
        r = __ull2double_rn(static_cast<unsigned long long>(u));
    } else {
        const int lz = __clzll(hi);           // normalise so bit 127 is set
        u <<= lz;
        unsigned long long top = static_cast<unsigned long long>(u >> 64);
        const unsigned long long rest = static_cast<unsigned long long>(u);
        top |= rest != 0 ? 1ull : 0ull;       // sticky: 64 >= 53 + 2 bits, one RN is exact
        r = scalbn(__ull2double_rn(top), 64 - lz);
    }
    return neg ? -r : r;
}

// 1/x to full double precision: MUFU seed + two Newton steps (no IEEE division on the chains)
__device__ inline double fast_rcp(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

// 1/x to ~2^-40 relative (one Newton step): ample for a Sturm count's sign decisions
__device__ inline double rcp_1nr(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    const double e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

// Sturm counts at 4 points at once (4 independent dependency chains per thread)
__device__ inline void sturm_count4(const double* d, const double* e2, int n, const double (&x)[4], double pivmin,
                                    int (&cnt)[4]) {
    double q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        q[u] = d[0] - x[u];
        if (fabs(q[u]) < pivmin) q[u] = -pivmin;
        cnt[u] = q[u] < 0;
    }
    for (int i = 1; i < n; ++i) {
        const double di = d[i], ei = e2[i - 1];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            q[u] = (di - x[u]) - ei * rcp_1nr(q[u]);
            if (fabs(q[u]) < pivmin) q[u] = -pivmin;
            cnt[u] += q[u] < 0;
        }
    }
}

// number of eigenvalues of T below x (Sturm sequence in ratio form, pivmin guard as dstebz)
__device__ int sturm_count_dev(const double* d, const double* e2, int n, double x, double pivmin) {
    int cnt = 0;
    double q = d[0] - x;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0;
    for (int i = 1; i < n; ++i) {
        q = (d[i] - x) - e2[i - 1] * fast_rcp(q);
        if (fabs(q) < pivmin) q = -pivmin;
        cnt += q < 0;
    }
    return cnt;
}

// LU of (T - sigma I) with partial pivoting, factored once per eigenvector:
//   u1i = 1 / pivot, u2/u3 the two super-diagonals of U, mult the multipliers, piv the row swaps
__device__ void tri_factor(const double* d, const double* e, int n, double sigma, double tiny, double* u1i,
                           double* u2, double* u3, double* mult, unsigned char* piv) {
    double dcur = d[0] - sigma;
    double scur = n > 1 ? e[0] : 0.0;
    for (int i = 0; i + 1 < n; ++i) {
        const double a = e[i];
        const double bn = d[i + 1] - sigma;
        const double cn = i + 2 < n ? e[i + 1] : 0.0;
        if (fabs(dcur) >= fabs(a)) {
            if (dcur == 0.0) dcur = tiny;
            const double r = fast_rcp(dcur);
            const double m = a * r;
            u1i[i] = fabs(dcur) < tiny ? fast_rcp(dcur < 0 ? -tiny : tiny) : r;
            u2[i] = scur;
            u3[i] = 0.0;
            mult[i] = m;
            piv[i] = 0;
            dcur = bn - m * scur;
            scur = cn;
        } else {
            const double r = fast_rcp(a);
            const double m = dcur * r;
            u1i[i] = fabs(a) < tiny ? fast_rcp(a < 0 ? -tiny : tiny) : r;
            u2[i] = bn;
            u3[i] = cn;
            mult[i] = m;
            piv[i] = 1;
            dcur = scur - m * bn;
            scur = -m * cn;
        }
    }
    if (dcur == 0.0) dcur = tiny;
    u1i[n - 1] = fast_rcp(fabs(dcur) < tiny ? (dcur < 0 ? -tiny : tiny) : dcur);
    u2[n - 1] = 0.0;  // read (times zero) by the first back-substitution step: never stale
    u3[n - 1] = 0.0;
}

// b := (T - sigma I)^-1 b with the factors above; the recurrences carry their state in registers.
// Returns max |b_i| of the result.
__device__ double tri_apply(const double* u1i, const double* u2, const double* u3, const double* mult,
                            const unsigned char* piv, int n, double* b) {
    double cur = b[0];
    for (int i = 0; i + 1 < n; ++i) {
        double nxt = b[i + 1];
        if (piv[i]) {
            const double t = cur;
            cur = nxt;
            nxt = t;
        }
        b[i] = cur;
        cur = nxt - mult[i] * cur;
    }
    b[n - 1] = cur;
    double x1 = 0.0, x2 = 0.0, mx = 0.0;
    for (int i = n - 1; i >= 0; --i) {
        const double xi = (b[i] - u2[i] * x1 - u3[i] * x2) * u1i[i];
        b[i] = xi;
        mx = fmax(mx, fabs(xi));
        x2 = x1;
        x1 = xi;
    }
    return mx;
}

__device__ inline void cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__device__ inline unsigned smem_addr(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
// address of the same shared-memory location in CTA `rank` of the cluster
__device__ inline unsigned peer_addr(unsigned local, int rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
    return r;
}
// 8-byte store into a peer CTA that completes 8 transaction bytes on the peer's mbarrier
__device__ inline void st_async_f64(unsigned raddr, double v, unsigned rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(raddr), "d"(v),
                 "r"(rbar)
                 : "memory");
}
__device__ inline void mbar_init(unsigned bar) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory"); }
__device__ inline void mbar_expect(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ inline void mbar_wait_cluster(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred P1;\n WAITC_%=:\n"
        " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
        " @!P1 bra WAITC_%=;\n}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}

// CTA-wide sum (fixed order -> deterministic), result in every thread
template <int T>
__device__ inline double cta_sum(double v, double* s_red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
#pragma unroll
    for (int i = 0; i < T / 32; ++i) t += s_red[i];
    return t;
}

__device__ inline double warp_allsum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// work buffer layout (doubles), see pca_work_doubles
constexpr int kLzMax = 64;  // Lanczos steps at most
struct pca_work_view {
    double *d, *e, *tau, *tn, *lam, *X, *refl;
    size_t rstride;
    double *lzab, *lzk, *lzQ, *stat;  // Lanczos: alpha/beta [8][2][kLzMax], steps [8], Q [8][kLzMax][n], status [8]
};
__host__ __device__ inline pca_work_view pca_work_split(double* w, int n, int D) {
    pca_work_view v;
    v.d = w;
    v.e = v.d + 8 * n;
    v.tau = v.e + 8 * n;
    v.tn = v.tau + 8 * n;
    v.lam = v.tn + 8;
    v.X = v.lam + 8 * 32;
    v.refl = v.X + static_cast<size_t>(8) * D * n;
    v.refl += (reinterpret_cast<uintptr_t>(v.refl) & 15) ? 1 : 0;  // 16-byte aligned for TMA
    v.rstride = refl_stride(n);
    v.lzab = v.refl + 8 * v.rstride;
    v.lzk = v.lzab + 8 * 2 * kLzMax;
    v.stat = v.lzk + 8;
    v.lzQ = v.stat + 8;
    return v;
}
size_t pca_work_doubles(int mc, int D) {
    return static_cast<size_t>(8) * (3 * mc + 1 + 32 + static_cast<size_t>(D) * mc) + 8 * refl_stride(mc) + 4 +
           8 * (2 * kLzMax + 2 + static_cast<size_t>(kLzMax) * mc);
}

struct tri_args {
    const unsigned long long* moments;  // F (s) + F*F (S), int64 values, tile pairs ti <= tj
    int F;
    unsigned long long n;
    const int32_t* cols;  // 8 * mc feature indices (layout-major)
    int mc;
    double* mean;  // 8 * mc
    pca_work_view w;
    long long* dbg;  // optional per-phase clock totals (ZI_DEBUG_PCA)
    const double* cov;  // optional: precomputed covariance per model (mc x mc, row-major); the
                        // moments, cols and mean are then unused
    int lzk;            // Lanczos steps (0: Householder path only)
};

// this CTA's rows i = rank + kCl*li of layout l's covariance (int128 numerators, correctly rounded)
// or of a precomputed covariance; rank 0 also writes the layout's mean
__device__ void pca_load_rows(const tri_args& a, int l, int rank, int n, int nloc, double* A) {
    const int tid = threadIdx.x;
    const long long* s = reinterpret_cast<const long long*>(a.moments);
    const long long* S = s + a.F;
    const long long nn = static_cast<long long>(a.n);
    const int32_t* cols = a.cols + l * n;
    const double den = a.n > 1 ? static_cast<double>(a.n) * static_cast<double>(a.n - 1) : 1.0;
    for (int idx = tid; idx < nloc * n; idx += blockDim.x) {
        const int li = idx / n, j = idx - li * n, i = rank + kCl * li;
        if (a.cov) {
            A[idx] = a.cov[(static_cast<size_t>(l) * n + i) * n + j];
            continue;
        }
        int ca = cols[i], cb = cols[j];
        if (ca / 128 > cb / 128) {  // k_moments fills the 128x128 tile pairs ti <= tj only
            const int t = ca;
            ca = cb;
            cb = t;
        }
        const __int128 num = static_cast<__int128>(nn) * S[static_cast<long long>(ca) * a.F + cb] -
                             static_cast<__int128>(s[cols[i]]) * s[cols[j]];
        A[idx] = i128_to_double(num) / den;
    }
    if (rank == 0 && !a.cov)
        for (int i = tid; i < n; i += blockDim.x)
            a.mean[l * n + i] = static_cast<double>(s[cols[i]]) / static_cast<double>(a.n);
}

__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kTriThreads) k_pca_tri(tri_args a) {
    extern __shared__ double sm[];
    if (a.lzk > 0 && a.w.stat[blockIdx.x / kCl] == 0.0) return;  // the Lanczos path delivered this layout
    cg::cluster_group cl = cg::this_cluster();
    const int n = a.mc, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int kWarps = kTriThreads / 32;
    const int rank = static_cast<int>(cl.block_rank());
    const int l = blockIdx.x / kCl;
    const int rows_max = (n + kCl - 1) / kCl;
    const int nloc = rank < n ? (n - rank + kCl - 1) / kCl : 0;  // my rows: i = rank + kCl * li
    double* A = sm;                                          // rows_max x n, full rows
    double* v = A + static_cast<size_t>(rows_max) * n;       // [2][n] reflector, by column parity
    double* p = v + 2 * n;                                   // [2][n] tau * A v
    double* npart = p + 2 * n;                               // [2][kCl][warps] partial |column|^2
    pca_load_rows(a, l, rank, n, nloc, A);
    double* d_out = a.w.d + l * n;
    double* e_out = a.w.e + l * n;
    double* tau_out = a.w.tau + l * n;
    double* refl = a.w.refl + l * a.w.rstride;
    __syncthreads();
    cluster_barrier();  // every CTA of the cluster runs before the first DSMEM store
    long long tacc[6] = {0, 0, 0, 0, 0, 0};
    long long tc = clock64();
#define TRI_T(i)                          \
    {                                     \
        const long long t2_ = clock64();  \
        tacc[i] += t2_ - tc;              \
        tc = t2_;                         \
    }
    // Column c's sub-diagonal entries A(i, c), i > c, live in the rows' owners (full rows): each
    // warp pushes the entries of its rows and its partial |.|^2 to every CTA, so the next
    // reflector is assembled everywhere without a single-owner broadcast.  The exchanges are
    // st.async stores that complete transaction bytes on the receiver's mbarrier (one per buffer
    // parity for v and for p): a CTA proceeds as soon as its own bytes have landed, with no
    // cluster-wide rendezvous per column.
    constexpr int kParts = kCl * kWarps;
    __shared__ __align__(8) unsigned long long s_bar[4];  // v[0], v[1], p[0], p[1]
    if (tid == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(smem_addr(&s_bar[i]));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const unsigned v_local = smem_addr(v), p_local = smem_addr(p), np_local = smem_addr(npart);
    const unsigned bar_local = smem_addr(&s_bar[0]);
    auto push_entry = [&](int c, int bb, int i, double y) {  // warp-uniform call
        if (lane < kCl)
            st_async_f64(peer_addr(v_local + 8u * (bb * n + (i - c - 1)), lane), y, peer_addr(bar_local + 8u * bb, lane));
    };
    auto push_partial = [&](int bb, double part) {
        if (lane < kCl)
            st_async_f64(peer_addr(np_local + 8u * (bb * kParts + rank * kWarps + warp), lane), part,
                         peer_addr(bar_local + 8u * bb, lane));
    };
    unsigned ph_v[2] = {0u, 0u}, ph_p[2] = {0u, 0u};
    __syncthreads();
    cluster_barrier();  // every mbarrier of the cluster is initialised before the first push
    {
        double part = 0.0;
        const int first = 1 > rank ? 1 : 0;
        for (int li = first + warp; li < nloc; li += kWarps) {
            const double y = A[static_cast<size_t>(li) * n];
            push_entry(0, 0, rank + kCl * li, y);
            part = fma(y, y, part);
        }
        push_partial(0, part);
    }
    for (int k = 0; k + 2 < n; ++k) {
        const int m = n - k - 1, b = k & 1;
        const double* vb = v + b * n;
        __syncthreads();  // this CTA's row updates of the previous column are visible to all warps
        // column k: m entries + the partials, from every CTA
        if (tid == 0) mbar_expect(bar_local + 8u * b, 8u * static_cast<unsigned>(m + kParts));
        mbar_wait_cluster(bar_local + 8u * b, ph_v[b]);
        ph_v[b] ^= 1u;
        // |column k|^2 from the per-warp partials, summed in the same order by every warp
        double np = 0.0;
#pragma unroll
        for (int q = 0; q < kParts / 32; ++q) np += npart[b * kParts + lane + 32 * q];
        const double norm2 = warp_allsum(np);
        const double x0 = vb[0];
        double alpha = x0, tk = 0.0;
        if (norm2 != 0.0) {
            alpha = x0 >= 0 ? -sqrt(norm2) : sqrt(norm2);
            tk = 1.0 / (norm2 - alpha * x0);  // 2 / |x - alpha e1|^2
        }
        const double v0 = tk != 0.0 ? x0 - alpha : x0;
        double vr[kSlots];
#pragma unroll
        for (int q = 0; q < kSlots; ++q) {
            const int j = lane + 32 * q;
            vr[q] = j < m ? vb[j] : 0.0;
        }
        if (lane == 0) vr[0] = v0;
        if (rank == 0 && warp == 0) {
#pragma unroll
            for (int q = 0; q < kSlots; ++q)
                if (lane + 32 * q < m) refl[refl_off(k, n) + lane + 32 * q] = vr[q];
            if (lane == 0) {
                e_out[k] = alpha;
                tau_out[k] = tk;
            }
        }
        const int li0 = k + 1 > rank ? (k + 1 - rank + kCl - 1) / kCl : 0;  // first trailing row
        const bool next = k + 3 < n;  // column k+1 is a Householder column
        double part = 0.0;
        TRI_T(0);
        if (tk != 0.0) {
            // p_i = tau * (A v)_i for my trailing rows, pushed to every CTA
            for (int li = li0 + warp; li < nloc; li += kWarps) {
                const int t = rank + kCl * li - k - 1;
                const double* row = A + static_cast<size_t>(li) * n + k + 1;
                double acc = 0.0;
#pragma unroll
                for (int q = 0; q < kSlots; ++q) {
                    const int j = lane + 32 * q;
                    if (j < m) acc = fma(row[j], vr[q], acc);
                }
                const double pt = tk * warp_allsum(acc);
                if (lane < kCl)
                    st_async_f64(peer_addr(p_local + 8u * (b * n + t), lane), pt, peer_addr(bar_local + 8u * (2 + b), lane));
            }
            TRI_T(1);
            if (tid == 0) mbar_expect(bar_local + 8u * (2 + b), 8u * static_cast<unsigned>(m));
            mbar_wait_cluster(bar_local + 8u * (2 + b), ph_p[b]);
            ph_p[b] ^= 1u;
            TRI_T(2);
            const double* pb = p + b * n;
            double wr[kSlots];
            double vp = 0.0;
#pragma unroll
            for (int q = 0; q < kSlots; ++q) {
                const int j = lane + 32 * q;
                wr[q] = j < m ? pb[j] : 0.0;
                vp = fma(vr[q], wr[q], vp);
            }
            const double K2 = 0.5 * tk * warp_allsum(vp);
#pragma unroll
            for (int q = 0; q < kSlots; ++q) wr[q] = fma(-K2, vr[q], wr[q]);  // w = p - K2 v
            // A22 -= v w^T + w v^T on my full rows; the new column k+1 entries go out at once
            for (int li = li0 + warp; li < nloc; li += kWarps) {
                const int t = rank + kCl * li - k - 1;
                double* row = A + static_cast<size_t>(li) * n + k + 1;
                const double vt = t == 0 ? v0 : vb[t];
                const double wt = fma(-K2, vt, pb[t]);
                double rv[kSlots];  // loads, math, stores in three batches (no smem aliasing chain)
#pragma unroll
                for (int q = 0; q < kSlots; ++q) {
                    const int j = lane + 32 * q;
                    rv[q] = j < m ? row[j] : 0.0;
                }
#pragma unroll
                for (int q = 0; q < kSlots; ++q) rv[q] = fma(-vt, wr[q], fma(-wt, vr[q], rv[q]));
#pragma unroll
                for (int q = 0; q < kSlots; ++q) {
                    const int j = lane + 32 * q;
                    if (j < m) row[j] = rv[q];
                }
                double y0 = rv[0];
                if (next && t >= 1) {
                    y0 = __shfl_sync(0xffffffffu, y0, 0);
                    push_entry(k + 1, b ^ 1, t + k + 1, y0);
                    part = fma(y0, y0, part);
                }
            }
            if (next) push_partial(b ^ 1, part);
            TRI_T(3);
        } else if (next) {
            for (int li = li0 + warp; li < nloc; li += kWarps) {
                const int i = rank + kCl * li;
                if (i < k + 2) continue;
                const double y = A[static_cast<size_t>(li) * n + k + 1];
                push_entry(k + 1, b ^ 1, i, y);
                part = fma(y, y, part);
            }
            push_partial(b ^ 1, part);
        }
        TRI_T(4);
        TRI_T(5);
    }
    __syncthreads();  // own rows final before the d / e read-out
    if (a.dbg && tid == 0)
        for (int i = 0; i < 6; ++i) a.dbg[blockIdx.x * 8 + i] = tacc[i];
#undef TRI_T
    for (int li = tid; li < nloc; li += kTriThreads) {
        const int i = rank + kCl * li;
        d_out[i] = A[static_cast<size_t>(li) * n + i];
        if (i == n - 1) {
            e_out[n - 2] = A[static_cast<size_t>(li) * n + n - 2];
            tau_out[n - 2] = 0.0;
        }
    }
    cluster_barrier();  // no CTA leaves while a peer may still store into its shared memory
}

// ------------------------------------------------------------------ Lanczos fast path
// k_pca_lz: one 8-CTA cluster per layout runs K steps of Lanczos with full reorthogonalisation
// (classical Gram-Schmidt twice, DGKS) on the covariance, rows distributed as in k_pca_tri.  The
// top eigenpairs of image-patch covariances converge in ~30 steps (they need only the leading
// part of the spectrum, against the 219 columns of a full tridiagonalisation).  Per step, three
// cluster exchanges, each st.async stores completing bytes on the receivers' mbarriers:
//   A  partial Q^T w      -> c1 (w -= Q c1)
//   B  partial Q^T w, |w|^2 -> c2 (w -= Q c2), beta^2 = |w|^2 - |c2|^2
//   C  the rows of q_{j+1} = w / beta into every CTA's full vector
// Every sum runs in a fixed order, so all CTAs hold identical alpha / beta.  k_pca_vec (Lanczos
// mode) then solves T_K, checks every Ritz residual |beta_K s_K| and falls the layout back to
// the Householder path (k_pca_tri + k_pca_vec) when one is not negligible.
__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kTriThreads) k_pca_lz(tri_args a) {
    extern __shared__ double sm[];
    __shared__ double s_red[kTriThreads / 32];
    __shared__ double s_ab[2 * kLzMax];
    __shared__ __align__(8) unsigned long long s_bar[3];
    __shared__ int s_k;
    cg::cluster_group cl = cg::this_cluster();
    const int n = a.mc, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int kWarps = kTriThreads / 32;
    constexpr int RS = kLzMax + 2;  // stride of a CTA's partials
    const int rank = static_cast<int>(cl.block_rank());
    const int l = blockIdx.x / kCl;
    const int rows_max = (n + kCl - 1) / kCl;
    const int nloc = rank < n ? (n - rank + kCl - 1) / kCl : 0;  // my rows: i = rank + kCl * li
    const int K = min(n, a.lzk);
    double* A = sm;                                      // rows_max x n
    double* Q = A + static_cast<size_t>(rows_max) * n;   // [kLzMax][rows_max]
    double* qf = Q + static_cast<size_t>(kLzMax) * rows_max;  // [2][n] full Lanczos vector
    double* wl = qf + 2 * n;                             // rows_max
    double* red0 = wl + rows_max;                        // [kCl][RS]
    double* red1 = red0 + kCl * RS;                      // [kCl][RS]
    double* part = red1 + kCl * RS;                      // RS
    double* c1 = part + RS;                              // RS
    double* c2 = c1 + RS;                                // RS
    pca_load_rows(a, l, rank, n, nloc, A);
    if (tid == 0) {
        for (int i = 0; i < 3; ++i) mbar_init(smem_addr(&s_bar[i]));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        s_k = K;
    }
    // deterministic start vector (identical on every CTA)
    double p0 = 0.0;
    for (int i = tid; i < n; i += kTriThreads) {
        const double f = 1.0 + 0.25 * sin(1.6180339887498949 * i);
        qf[i] = f;
        p0 = fma(f, f, p0);
    }
    const double inv0 = 1.0 / sqrt(cta_sum<kTriThreads>(p0, s_red));
    for (int i = tid; i < n; i += kTriThreads) qf[i] *= inv0;
    __syncthreads();
    for (int li = tid; li < nloc; li += kTriThreads) Q[li] = qf[rank + kCl * li];
    const unsigned red0_l = smem_addr(red0), red1_l = smem_addr(red1), qf_l = smem_addr(qf);
    const unsigned barA = smem_addr(&s_bar[0]), barB = smem_addr(&s_bar[1]), barC = smem_addr(&s_bar[2]);
    unsigned ph = 0;  // the three barriers complete once per step each: one shared phase bit
    __syncthreads();
    cluster_barrier();  // every mbarrier of the cluster is initialised before the first push
    for (int j = 0; j < K; ++j) {
        const int b = j & 1, nt = j + 1;
        const double* q = qf + b * n;
        // (1) my rows of w = A q
        for (int li = warp; li < nloc; li += kWarps) {
            double acc = 0.0;
            for (int c = lane; c < n; c += 32) acc = fma(A[static_cast<size_t>(li) * n + c], q[c], acc);
            acc = warp_allsum(acc);
            if (lane == 0) wl[li] = acc;
        }
        __syncthreads();
        // (2) round A: partial Q^T w over my rows -> every CTA
        if (tid < nt) {
            double acc = 0.0;
            for (int li = 0; li < nloc; ++li) acc = fma(Q[tid * rows_max + li], wl[li], acc);
            part[tid] = acc;
        }
        __syncthreads();
        if (tid == 0) mbar_expect(barA, static_cast<unsigned>(kCl * nt * 8));
        for (int idx = tid; idx < kCl * nt; idx += kTriThreads) {
            const int pr = idx / nt, t = idx - pr * nt;
            st_async_f64(peer_addr(red0_l + 8u * (rank * RS + t), pr), part[t], peer_addr(barA, pr));
        }
        mbar_wait_cluster(barA, ph);
        if (tid < nt) {
            double acc = 0.0;
#pragma unroll
            for (int r = 0; r < kCl; ++r) acc += red0[r * RS + tid];
            c1[tid] = acc;
        }
        __syncthreads();
        if (tid < nloc) {
            double w = wl[tid];
            for (int t = 0; t < nt; ++t) w = fma(-c1[t], Q[t * rows_max + tid], w);
            wl[tid] = w;
        }
        __syncthreads();
        // (3) round B: partial Q^T w and |w|^2
        if (tid <= nt) {
            double acc = 0.0;
            if (tid < nt)
                for (int li = 0; li < nloc; ++li) acc = fma(Q[tid * rows_max + li], wl[li], acc);
            else
                for (int li = 0; li < nloc; ++li) acc = fma(wl[li], wl[li], acc);
            part[tid] = acc;
        }
        __syncthreads();
        if (tid == 0) mbar_expect(barB, static_cast<unsigned>(kCl * (nt + 1) * 8));
        for (int idx = tid; idx < kCl * (nt + 1); idx += kTriThreads) {
            const int pr = idx / (nt + 1), t = idx - pr * (nt + 1);
            st_async_f64(peer_addr(red1_l + 8u * (rank * RS + t), pr), part[t], peer_addr(barB, pr));
        }
        mbar_wait_cluster(barB, ph);
        if (tid <= nt) {
            double acc = 0.0;
#pragma unroll
            for (int r = 0; r < kCl; ++r) acc += red1[r * RS + tid];
            c2[tid] = acc;
        }
        __syncthreads();
        if (tid < nloc) {
            double w = wl[tid];
            for (int t = 0; t < nt; ++t) w = fma(-c2[t], Q[t * rows_max + tid], w);
            wl[tid] = w;
        }
        double b2 = c2[nt];
        for (int t = 0; t < nt; ++t) b2 = fma(-c2[t], c2[t], b2);
        const double beta = sqrt(fmax(b2, 0.0));
        if (tid == 0) {
            s_ab[j] = c1[j] + c2[j];
            s_ab[kLzMax + j] = beta;
        }
        double anorm = 0.0;
        for (int t = 0; t <= j; ++t) anorm = fmax(anorm, fabs(c1[t] + c2[t]));
        __syncthreads();
        if (j + 1 == K || !(beta > 1e-13 * anorm)) {  // done, or an invariant subspace
            if (tid == 0) s_k = j + 1;
            break;
        }
        // (4) round C: my rows of q_{j+1} into every CTA's full vector
        const double ib = 1.0 / beta;
        if (tid == 0) mbar_expect(barC, static_cast<unsigned>(n * 8));
        const unsigned qn = qf_l + 8u * static_cast<unsigned>((b ^ 1) * n);
        for (int idx = tid; idx < kCl * nloc; idx += kTriThreads) {
            const int pr = idx / nloc, li = idx - pr * nloc;
            const double v = wl[li] * ib;
            if (pr == 0) Q[(j + 1) * rows_max + li] = v;
            st_async_f64(peer_addr(qn + 8u * static_cast<unsigned>(rank + kCl * li), pr), v, peer_addr(barC, pr));
        }
        mbar_wait_cluster(barC, ph);
        ph ^= 1;
        __syncthreads();
    }
    __syncthreads();
    const int k = s_k;
    if (rank == 0) {
        for (int t = tid; t < k; t += kTriThreads) {
            a.w.lzab[l * 2 * kLzMax + t] = s_ab[t];
            a.w.lzab[l * 2 * kLzMax + kLzMax + t] = s_ab[kLzMax + t];
        }
        if (tid == 0) {
            a.w.lzk[l] = static_cast<double>(k);
            a.w.stat[l] = 0.0;
        }
    }
    double* Qg = a.w.lzQ + static_cast<size_t>(l) * kLzMax * n;
    for (int idx = tid; idx < k * nloc; idx += kTriThreads) {
        const int t = idx / nloc, li = idx - t * nloc;
        Qg[static_cast<size_t>(t) * n + rank + kCl * li] = Q[t * rows_max + li];
    }
    cluster_barrier();  // no CTA leaves while a peer may still store into its shared memory
}

struct vec_args {
    int mc, D;
    pca_work_view w;
    long long* dbg;  // optional phase clocks (ZI_DEBUG_PCA): per CTA 4 values
    int lzmode;      // 1: eigenpairs of the Lanczos T_K and Ritz vectors Q s; 0: Householder path
    int lztried;     // Householder mode: skip the layouts the Lanczos path delivered
};

__device__ inline unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(kVecThreads) k_pca_vec(vec_args a) {
    extern __shared__ __align__(16) double sm[];
    __shared__ __align__(8) unsigned long long s_bar;
    __shared__ int s_first[kVecThreads / 32];
    __shared__ double s_scal[4];
    const int D = a.D, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int l = blockIdx.x / D, j = blockIdx.x % D;
    if (!a.lzmode && a.lztried && a.w.stat[l] == 0.0) return;  // the Lanczos path delivered this layout
    // the tridiagonal: Householder's T (size mc) or Lanczos' T_K (size K)
    const int n = a.lzmode ? static_cast<int>(a.w.lzk[l]) : a.mc;
    if (a.lzmode && j >= n) {  // fewer Lanczos vectors than components: Householder path
        if (tid == 0) a.w.stat[l] = 1.0;
        return;
    }
    const long long t_start = clock64();
    const size_t nref = a.w.rstride;
    double* R = sm;         // reflectors (TMA)
    double* dd = R + nref;  // n
    double* ee = dd + n;    // n
    double* e2 = ee + n;    // n
    double* tau = e2 + n;   // n
    double* x = tau + n;    // n
    double* f = x + n;      // 4n LU factors
    unsigned char* piv = reinterpret_cast<unsigned char*>(f + 4 * n);
    const double* src = a.w.refl + l * a.w.rstride;
    const unsigned bytes = static_cast<unsigned>(nref * sizeof(double));
    if (tid == 0 && !a.lzmode) {
        const unsigned bar = smem_u32(&s_bar);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(R)),
                     "l"(src), "r"(bytes), "r"(bar)
                     : "memory");
    }
    for (int i = tid; i < n; i += kVecThreads) {
        if (a.lzmode) {
            const double* ab = a.w.lzab + l * 2 * kLzMax;
            dd[i] = ab[i];
            const double ei = i + 1 < n ? ab[kLzMax + i] : 0.0;
            ee[i] = ei;
            e2[i] = ei * ei;
            tau[i] = 0.0;
        } else {
            dd[i] = a.w.d[l * n + i];
            const double ei = i + 1 < n ? a.w.e[l * n + i] : 0.0;
            ee[i] = ei;
            e2[i] = ei * ei;
            tau[i] = a.w.tau[l * n + i];
        }
    }
    __syncthreads();
    if (tid == 0) {
        double tn = 0.0, glo = DBL_MAX, ghi = -DBL_MAX;
        for (int i = 0; i < n; ++i) {
            const double r = (i > 0 ? fabs(ee[i - 1]) : 0.0) + (i + 1 < n ? fabs(ee[i]) : 0.0);
            tn = fmax(tn, fabs(dd[i]) + r);
            glo = fmin(glo, dd[i] - r);
            ghi = fmax(ghi, dd[i] + r);
        }
        const double safe = tn > 0 ? tn : 1.0;
        const double pivmin = DBL_MIN * 1e4 * fmax(1.0, safe * safe);
        s_scal[0] = safe;
        s_scal[1] = pivmin;
        s_scal[2] = glo - 2 * DBL_EPSILON * safe - pivmin;
        s_scal[3] = ghi + 2 * DBL_EPSILON * safe + pivmin;
        if (j == 0) a.w.tn[l] = safe;
    }
    __syncthreads();
    const double safe = s_scal[0], pivmin = s_scal[1];
    // lambda_j (j-th largest) by multisection: 4 points per lane, 512 per round
    constexpr int kPts = 4 * kVecThreads;
    const int target = n - 1 - j;
    double lo = s_scal[2], hi = s_scal[3];
    // stop at ~1e-10 relative: the Rayleigh quotient of the inverse-iteration vector below gives
    // the eigenvalue to working precision
    for (int it = 0; it < 64; ++it) {
        if (hi - lo <= 1e-10 * fmax(fabs(lo), fabs(hi)) + pivmin) break;
        double xq[4];
        int cq[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) xq[u] = lo + (hi - lo) * (4 * tid + u + 1) / static_cast<double>(kPts + 1);
        sturm_count4(dd, e2, n, xq, pivmin, cq);
        // first point past lambda_j: counts are monotone in the point index
        int first = kPts;
#pragma unroll
        for (int u = 3; u >= 0; --u)
            if (cq[u] > target) first = 4 * tid + u;
        first = min(first, kPts);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
        if (lane == 0) s_first[warp] = first;
        __syncthreads();
        int c = kPts;
#pragma unroll
        for (int w = 0; w < kVecThreads / 32; ++w) c = min(c, s_first[w]);
        __syncthreads();
        const double nlo = c > 0 ? lo + (hi - lo) * c / static_cast<double>(kPts + 1) : lo;
        const double nhi = c < kPts ? lo + (hi - lo) * (c + 1) / static_cast<double>(kPts + 1) : hi;
        if (!(nlo < nhi) || (nlo == lo && nhi == hi)) break;
        lo = nlo;
        hi = nhi;
    }
    const double lam = 0.5 * (lo + hi);
    const long long t_bis = clock64();
    // inverse iteration: LU of (T - lambda I) once, three solves from a pseudo-random start
    if (tid == 0) {
        const double tiny = DBL_EPSILON * safe;
        tri_factor(dd, ee, n, lam, tiny, f, f + n, f + 2 * n, f + 3 * n, piv);
        for (int i = 0; i < n; ++i) {  // splitmix64: starts differ per component
            unsigned long long z = (static_cast<unsigned long long>(j) << 32 | static_cast<unsigned>(i)) +
                                   0x9E3779B97F4A7C15ull;
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
            z ^= z >> 31;
            x[i] = static_cast<double>(z >> 11) * 0x1.0p-53 - 0.5;
        }
        for (int it = 0; it < 2; ++it) {  // the shift is exact to working precision: two solves
            const double mx = tri_apply(f, f + n, f + 2 * n, f + 3 * n, piv, n, x);
            const double sc = mx > 0.0 ? fast_rcp(mx) : 1.0;
            for (int i = 0; i < n; ++i) x[i] *= sc;
        }
        double nrm = 0.0;
        for (int i = 0; i < n; ++i) nrm = fma(x[i], x[i], nrm);
        const double inv = 1.0 / sqrt(nrm);
        for (int i = 0; i < n; ++i) x[i] *= inv;
        // Rayleigh quotient x^T T x (|x| = 1): eigenvalue error ~ residual^2 / gap
        double rq = dd[0] * x[0] * x[0];
        for (int i = 1; i < n; ++i) rq = fma(dd[i] * x[i], x[i], fma(2.0 * ee[i - 1] * x[i - 1], x[i], rq));
        a.w.lam[l * 32 + j] = rq;
        if (a.lzmode) {  // Ritz residual |A y - theta y| = |beta_K s_K| (full reorthogonalisation)
            const double res = fabs(a.w.lzab[l * 2 * kLzMax + kLzMax + n - 1] * x[n - 1]);
            if (!(res <= 1e-10 * safe)) a.w.stat[l] = 1.0;  // vector error ~ res / gap: far inside the 1e-7 budget
        }
    }
    __syncthreads();
    const long long t_inv = clock64();
    if (a.lzmode) {  // Ritz vector y = Q_K s
        const int nn = a.mc;
        const double* Qg = a.w.lzQ + static_cast<size_t>(l) * kLzMax * nn;
        double* out = a.w.X + (static_cast<size_t>(l) * D + j) * nn;
        for (int i = tid; i < nn; i += kVecThreads) {
            double acc = 0.0;
            for (int t = 0; t < n; ++t) acc = fma(Qg[static_cast<size_t>(t) * nn + i], x[t], acc);
            out[i] = acc;
        }
        return;
    }
    // back-transformation x = H_0 ... H_{n-3} x, one warp, the vector in registers
    if (warp == 0) {
        const unsigned bar = smem_u32(&s_bar);
        asm volatile(
            "{\n .reg .pred P1;\n WAIT_%=:\n"
            " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
            " @!P1 bra WAIT_%=;\n}\n" ::"r"(bar)
            : "memory");
        double xr[kSlots];
#pragma unroll
        for (int q = 0; q < kSlots; ++q) xr[q] = lane + 32 * q < n ? x[lane + 32 * q] : 0.0;
        for (int k = n - 3; k >= 0; --k) {
            const double tk = tau[k];
            if (tk == 0.0) continue;
            const double* r = R + refl_off(k, n) - (k + 1);  // r[i], i > k
            double part = 0.0;
#pragma unroll
            for (int q = 0; q < kSlots; ++q) {
                const int i = lane + 32 * q;
                if (i > k && i < n) part = fma(r[i], xr[q], part);
            }
            const double fct = tk * warp_allsum(part);
#pragma unroll
            for (int q = 0; q < kSlots; ++q) {
                const int i = lane + 32 * q;
                if (i > k && i < n) xr[q] = fma(-fct, r[i], xr[q]);
            }
        }
        if (a.dbg && lane == 0) {
            a.dbg[blockIdx.x * 4 + 0] = t_bis - t_start;
            a.dbg[blockIdx.x * 4 + 1] = t_inv - t_bis;
            a.dbg[blockIdx.x * 4 + 2] = clock64() - t_inv;
        }
        double* out = a.w.X + (static_cast<size_t>(l) * D + j) * n;
#pragma unroll
        for (int q = 0; q < kSlots; ++q)
            if (lane + 32 * q < n) out[lane + 32 * q] = xr[q];
    }
}

struct fin_args {
    int mc, D;
    pca_work_view w;
    double* comp;  // 8 * mc * D, [l][i][d]
    double* eig;   // 8 * D
};

__global__ void __launch_bounds__(256) k_pca_fin(fin_args a) {
    extern __shared__ double sm[];
    __shared__ double s_red[8];
    const int n = a.mc, D = a.D, l = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double* X = sm;  // D x n
    const double* lam = a.w.lam + l * 32;
    for (int i = tid; i < D * n; i += 256) X[i] = a.w.X[static_cast<size_t>(l) * D * n + i];
    __syncthreads();
    const double cluster = 1e-3 * a.w.tn[l];
    // Gram-Schmidt inside clusters of close eigenvalues (component j against the earlier ones)
    for (int j = 1; j < D; ++j) {
        for (int q = 0; q < j; ++q) {
            if (fabs(lam[q] - lam[j]) > cluster) continue;
            double* xj = X + static_cast<size_t>(j) * n;
            const double* xq = X + static_cast<size_t>(q) * n;
            double part = 0.0;
            for (int i = tid; i < n; i += 256) part = fma(xq[i], xj[i], part);
            const double dot = cta_sum<256>(part, s_red);
            for (int i = tid; i < n; i += 256) xj[i] = fma(-dot, xq[i], xj[i]);
            __syncthreads();
            part = 0.0;
            for (int i = tid; i < n; i += 256) part = fma(xj[i], xj[i], part);
            const double inv = 1.0 / sqrt(cta_sum<256>(part, s_red));
            for (int i = tid; i < n; i += 256) xj[i] *= inv;
            __syncthreads();
        }
    }
    // sign rule: the first entry of largest magnitude is positive (strict '>' keeps the earliest)
    for (int j = warp; j < D; j += 8) {
        const double* x = X + static_cast<size_t>(j) * n;
        double best = -1.0;
        int arg = 0;
        for (int i = lane; i < n; i += 32) {
            const double ax = fabs(x[i]);
            if (ax > best) {
                best = ax;
                arg = i;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
            if (ob > best || (ob == best && oa < arg)) {
                best = ob;
                arg = oa;
            }
        }
        const double sgn = x[arg] < 0 ? -1.0 : 1.0;
        for (int i = lane; i < n; i += 32) a.comp[(static_cast<size_t>(l) * n + i) * D + j] = sgn * x[i];
        if (lane == 0) a.eig[l * D + j] = fmax(0.0, lam[j]);
    }
}

static bool pca_launch(zi_ctx* ctx, int nl, const double* d_cov, const unsigned long long* d_moments, int F, uint64_t n,
                       const int32_t* d_cols, int mc, int D, double* d_mean, double* d_comp, double* d_eig,
                       double* d_work);

bool pca_on_device(zi_ctx* ctx, const unsigned long long* d_moments, int F, uint64_t n, const int32_t* d_cols, int mc,
                   int D, double* d_mean, double* d_comp, double* d_eig, double* d_work, int* /*d_status*/) {
    return pca_launch(ctx, 8, nullptr, d_moments, F, n, d_cols, mc, D, d_mean, d_comp, d_eig, d_work);
}

bool pca_on_device_n(zi_ctx* ctx, int layouts, const unsigned long long* d_moments, int F, uint64_t n,
                     const int32_t* d_cols, int mc, int D, double* d_mean, double* d_comp, double* d_eig,
                     double* d_work) {
    return pca_launch(ctx, layouts, nullptr, d_moments, F, n, d_cols, mc, D, d_mean, d_comp, d_eig, d_work);
}

bool pca_from_cov_on_device(zi_ctx* ctx, const double* d_cov, int mc, int D, double* d_comp, double* d_eig,
                            double* d_work) {
    return pca_launch(ctx, 1, d_cov, nullptr, 0, 0, nullptr, mc, D, nullptr, d_comp, d_eig, d_work);
}

static bool pca_launch(zi_ctx* ctx, int nl, const double* d_cov, const unsigned long long* d_moments, int F, uint64_t n,
                       const int32_t* d_cols, int mc, int D, double* d_mean, double* d_comp, double* d_eig,
                       double* d_work) {
    if (mc > kPcaMaxN || D > 32 || mc < 3) return false;
    int optin = 0;
    ZI_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
    const size_t limit = static_cast<size_t>(optin) - 1024;
    const int rows_max = (mc + kCl - 1) / kCl;
    const size_t smem_tri = (static_cast<size_t>(rows_max) * mc + 4 * mc + 2 * kCl * (kTriThreads / 32)) * sizeof(double);
    const size_t smem_vec = (refl_stride(mc) + 9 * static_cast<size_t>(mc)) * sizeof(double) + mc + 16;
    const size_t smem_fin = static_cast<size_t>(D) * mc * sizeof(double);
    if (smem_tri > limit || smem_vec > limit || smem_fin > limit) return false;
    smem_attr(ctx->device, k_pca_tri, smem_tri);
    if (kCl > 8) ZI_CUDA(cudaFuncSetAttribute(k_pca_tri, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    smem_attr(ctx->device, k_pca_vec, smem_vec);
    smem_attr(ctx->device, k_pca_fin, smem_fin);
    const pca_work_view w = pca_work_split(d_work, mc, D);
    static const char* lz_env = std::getenv("ZI_PCA_LZ");
    const bool lz_on = !(lz_env && lz_env[0] == '0');
    const int lzk = lz_on ? std::min(std::min(mc, kLzMax), std::max(32, 2 * D + 8)) : 0;
    tri_args ta{d_moments, F, n, d_cols, mc, d_mean, w, nullptr, d_cov, lzk};
    if (lzk > 0) {
        const size_t smem_lz = (static_cast<size_t>(rows_max) * mc + static_cast<size_t>(kLzMax) * rows_max + 2 * mc +
                                rows_max + (2 * kCl + 3) * (kLzMax + 2)) * sizeof(double);
        smem_attr(ctx->device, k_pca_lz, smem_lz);
        ZI_LAUNCH(ctx, "pca_lanczos", k_pca_lz, nl * kCl, kTriThreads, smem_lz, ta);
        vec_args la{mc, D, w, nullptr, 1, 0};
        ZI_LAUNCH(ctx, "pca_ritz", k_pca_vec, nl * D, kVecThreads, smem_vec, la);
    }
    static const bool debug = std::getenv("ZI_DEBUG_PCA") != nullptr;
    static dbuf<long long> dbg;
    if (debug) {
        ta.dbg = dbg.ensure(8 * kCl * 8);
        ZI_CUDA(cudaMemsetAsync(ta.dbg, 0, 8 * kCl * 8 * sizeof(long long), ctx->stream));
    }
    ZI_LAUNCH(ctx, "pca_tridiag", k_pca_tri, nl * kCl, kTriThreads, smem_tri, ta);
    if (debug) {
        long long h[8 * kCl * 8];
        ZI_CUDA(cudaMemcpyAsync(h, ta.dbg, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
        ZI_CUDA(cudaStreamSynchronize(ctx->stream));
        for (int c = 0; c < 2 * kCl; ++c)
            std::fprintf(stderr, "tri cta %2d: start %lld B %lld bar1 %lld C %lld push %lld bar2 %lld\n", c, h[c * 8],
                         h[c * 8 + 1], h[c * 8 + 2], h[c * 8 + 3], h[c * 8 + 4], h[c * 8 + 5]);
    }
    vec_args va{mc, D, w, nullptr, 0, lzk > 0 ? 1 : 0};
    static dbuf<long long> vdbg;
    if (debug) va.dbg = vdbg.ensure(8 * 32 * 4);
    ZI_LAUNCH(ctx, "pca_vectors", k_pca_vec, nl * D, kVecThreads, smem_vec, va);
    if (debug) {
        std::vector<long long> h(static_cast<size_t>(8) * D * 4);
        ZI_CUDA(cudaMemcpyAsync(h.data(), va.dbg, h.size() * sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
        ZI_CUDA(cudaStreamSynchronize(ctx->stream));
        for (int c = 0; c < 3; ++c)
            std::fprintf(stderr, "vec cta %d: bisect %lld inverse %lld backtransform %lld\n", c, h[c * 4], h[c * 4 + 1],
                         h[c * 4 + 2]);
    }
    fin_args fa{mc, D, w, d_comp, d_eig};
    ZI_LAUNCH(ctx, "pca_finish", k_pca_fin, nl, 256, smem_fin, fa);
    return true;
}

}  // namespace zi
