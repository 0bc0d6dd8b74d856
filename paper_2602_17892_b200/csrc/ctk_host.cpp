// ctk_host.cpp -- native host fp64 projected problem of hybrid GMRES.
//
// Per iteration the reference solves, on the (k+1) x k Hessenberg H_k:
//   SVD (ctkrylov/arnoldi.py:133-141), the 200-point lambda grid
//   (regparam.py:28-36), filter-factor norms (regparam.py:46-60), the L-curve
//   corner (regparam.py:82-107) or GCV minimum (regparam.py:110-134), and the
//   projected Tikhonov / least-squares solve (arnoldi.py:95-130).
// All of it stays on the host in fp64 (north star); here it runs in C++ so
// that host worker threads can solve several iterations' projected problems
// concurrently without the Python GIL.  The SVD is LAPACK dgesdd (the routine
// numpy.linalg.svd uses), reached through scipy's exported cython_lapack
// function pointer registered by the Python layer (ctk_set_lapack).
//
// Semantics match the reference's: grid endpoints exact, ties broken toward
// the larger lambda, DegenerateCurveError conditions reported as a flag.
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <limits>
#include <vector>

#include "../../include/ctk.h"

extern int ctk_fail(int code, const char* fmt, ...);

namespace {

typedef void (*dgesdd_t)(char* jobz, int* m, int* n, double* a, int* lda, double* s, double* u,
                         int* ldu, double* vt, int* ldvt, double* work, int* lwork, int* iwork,
                         int* info);
dgesdd_t g_dgesdd = nullptr;
typedef double (*ddot_t)(int* n, double* x, int* incx, double* y, int* incy);
ddot_t g_ddot = nullptr;

// numpy's pairwise summation (add.reduce over a contiguous float64 array):
// 8 partial sums for blocks <= 128, recursive halving above.  Matching it
// keeps the filter-factor norms bitwise equal to the reference's np.sum.
double pairwise_sum(const double* a, long n) {
    if (n < 8) {
        double r = 0.0;
        for (long i = 0; i < n; ++i) r += a[i];
        return r;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        long i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    }
    long n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise_sum(a, n2) + pairwise_sum(a + n2, n - n2);
}

// c . c as numpy's `c @ c` computes it (BLAS ddot) when BLAS is registered.
double dot_self(std::vector<double>& c) {
    if (g_ddot) {
        int n = (int)c.size(), inc = 1;
        return g_ddot(&n, c.data(), &inc, c.data(), &inc);
    }
    double r = 0.0;
    for (double v : c) r += v * v;
    return r;
}

struct Svd {
    int kp1 = 0, k = 0;
    std::vector<double> s, U, VT;   // U: kp1 x k col-major, VT: k x k col-major
};

int svd_hessenberg(const double* H, int kp1, int k, Svd& out) {
    out.kp1 = kp1;
    out.k = k;
    std::vector<double> A((size_t)kp1 * k);
    for (int i = 0; i < kp1; ++i)
        for (int j = 0; j < k; ++j) A[(size_t)i + (size_t)j * kp1] = H[(size_t)i * k + j];
    out.s.assign(k, 0.0);
    out.U.assign((size_t)kp1 * k, 0.0);
    out.VT.assign((size_t)k * k, 0.0);
    std::vector<int> iwork(8 * (size_t)k);
    char jobz = 'S';
    int m = kp1, n = k, lda = kp1, ldu = kp1, ldvt = k, lwork = -1, info = 0;
    double wq = 0.0;
    g_dgesdd(&jobz, &m, &n, A.data(), &lda, out.s.data(), out.U.data(), &ldu, out.VT.data(), &ldvt,
             &wq, &lwork, iwork.data(), &info);
    if (info != 0) return info;
    lwork = (int)wq + 1;
    std::vector<double> work(lwork);
    g_dgesdd(&jobz, &m, &n, A.data(), &lda, out.s.data(), out.U.data(), &ldu, out.VT.data(), &ldvt,
             work.data(), &lwork, iwork.data(), &info);
    return info;
}

// numpy.geomspace(lo, hi, count): 10 ** linspace(log10 lo, log10 hi), endpoints exact.
void geomspace(double lo, double hi, int count, std::vector<double>& g) {
    g.resize(count);
    const double a = log10(lo), b = log10(hi);
    const double step = count > 1 ? (b - a) / (double)(count - 1) : 0.0;
    for (int i = 0; i < count; ++i) g[i] = pow(10.0, (double)i * step + a);
    g[0] = lo;
    if (count > 1) g[count - 1] = hi;
}

// np.gradient with unit spacing (second-order interior, first-order edges).
void gradient(const std::vector<double>& f, std::vector<double>& d) {
    const int n = (int)f.size();
    d.resize(n);
    if (n < 2) {
        if (n == 1) d[0] = 0.0;
        return;
    }
    d[0] = f[1] - f[0];
    d[n - 1] = f[n - 1] - f[n - 2];
    for (int i = 1; i < n - 1; ++i) d[i] = (f[i + 1] - f[i - 1]) / 2.0;
}

enum { S_NONE = 0, S_FIXED = 1, S_LCURVE = 2, S_GCV = 3 };

// Returns 0 and sets lam, or 1 for a degenerate curve (DegenerateCurveError).
// s: singular values of H (k), c: beta * U[0, :] (the rotated right-hand side).
int select_sc(const double* sv, std::vector<double>& c, int k, int kp1, double beta,
              int strategy, int grid_count, double* lam) {
    double smax = 0.0, smin = std::numeric_limits<double>::infinity();
    for (int i = 0; i < k; ++i) {
        smax = std::max(smax, sv[i]);
        if (sv[i] > 0) smin = std::min(smin, sv[i]);
    }
    if (!(smax > 0.0)) return 1;                       // all singular values are zero
    std::vector<double> grid;
    geomspace(std::max(smin * 1e-4, 1e-12), smax, grid_count, grid);
    const double outside = std::max(beta * beta - dot_self(c), 0.0);
    std::vector<double> sol(grid_count), res(grid_count), tr(grid_count);
    std::vector<double> ta(k), tb(k), tf(k);
    for (int g = 0; g < grid_count; ++g) {
        const double l = grid[g], l2 = l * l;
        for (int i = 0; i < k; ++i) {
            const double s2 = sv[i] * sv[i];
            const double den = s2 + l2;
            const double a = sv[i] * c[i] / den;
            const double r = (l2 / den) * c[i];
            ta[i] = a * a;
            tb[i] = r * r;
            tf[i] = s2 / den;
        }
        sol[g] = pairwise_sum(ta.data(), k);
        res[g] = pairwise_sum(tb.data(), k) + outside;
        tr[g] = (double)kp1 - pairwise_sum(tf.data(), k);
    }
    if (strategy == S_GCV) {
        int best = -1;
        double bv = 0.0;
        for (int g = grid_count - 1; g >= 0; --g) {    // ties toward larger lambda
            if (tr[g] <= 0.0) return 1;                 // GCV trace underflow
            const double val = res[g] / (tr[g] * tr[g]);
            if (!isfinite(val)) return 1;
            if (best < 0 || val < bv) {
                best = g;
                bv = val;
            }
        }
        *lam = grid[best];
        return 0;
    }
    // L-curve corner
    if (grid_count < 5) return 1;
    std::vector<double> xr(grid_count), ys(grid_count), dx, dy, ddx, ddy;
    for (int g = 0; g < grid_count; ++g) {
        xr[g] = 0.5 * log(std::max(res[g], 1e-300));
        ys[g] = 0.5 * log(std::max(sol[g], 1e-300));
    }
    gradient(xr, dx);
    gradient(ys, dy);
    gradient(dx, ddx);
    gradient(dy, ddy);
    int best = -1;
    double bk = -std::numeric_limits<double>::infinity();
    bool any_finite = false;
    for (int g = grid_count - 1; g >= 0; --g) {
        const double den = pow(dx[g] * dx[g] + dy[g] * dy[g], 1.5);
        const double kap = (dx[g] * ddy[g] - dy[g] * ddx[g]) / den;
        if (!isfinite(kap)) continue;
        any_finite = true;
        if (best < 0 || kap > bk) {
            best = g;
            bk = kap;
        }
    }
    if (!any_finite) return 1;
    if (bk <= 1e-9) return 1;                            // CURVATURE_FLOOR
    *lam = grid[best];
    return 0;
}

int select(const Svd& v, double beta, int strategy, int grid_count, double* lam) {
    std::vector<double> c(v.k);
    for (int i = 0; i < v.k; ++i) c[i] = beta * v.U[(size_t)i * v.kp1];   // beta * U[0, i]
    return select_sc(v.s.data(), c, v.k, v.kp1, beta, strategy, grid_count, lam);
}

void tikhonov(const double* H, const Svd& v, double beta, double lam, double* y, double* res,
              int* rank_def) {
    const int k = v.k, kp1 = v.kp1;
    std::vector<double> coef(k, 0.0);
    int rank = 0;
    if (lam == 0.0) {
        const double cutoff = std::numeric_limits<double>::epsilon() * std::max(kp1, k) *
                              (k > 0 ? v.s[0] : 0.0);
        for (int i = 0; i < k; ++i)
            if (v.s[i] > cutoff) {
                coef[i] = beta * v.U[(size_t)i * kp1] / v.s[i];
                ++rank;
            }
    } else {
        for (int i = 0; i < k; ++i) {
            const double c = beta * v.U[(size_t)i * kp1];
            coef[i] = v.s[i] * c / (v.s[i] * v.s[i] + lam * lam);
        }
        rank = k;
    }
    for (int j = 0; j < k; ++j) {
        double a = 0.0;
        for (int i = 0; i < k; ++i) a += v.VT[(size_t)i + (size_t)j * k] * coef[i];
        y[j] = a;
    }
    double r2 = 0.0;
    for (int i = 0; i < kp1; ++i) {
        double a = (i == 0) ? -beta : 0.0;
        for (int j = 0; j < k; ++j) a += H[(size_t)i * k + j] * y[j];
        r2 += a * a;
    }
    *res = sqrt(r2);
    *rank_def = rank < k;
}

// ---------------------------------------------------------------------------
// Lock-free fast path.  OpenBLAS serialises concurrent LAPACK calls behind a
// global lock, so dgesdd from several worker threads runs one at a time; this
// path needs no level-2/3 BLAS: a hand-written Householder bidiagonalisation
// H = Q [B; 0] P^T (the left reflectors applied only to beta e1), LAPACK
// dbdsqr for the singular values of B with the rotations applied to that one
// vector (ncc = 1, level-1 BLAS only), and a Givens elimination of the damped
// bidiagonal problem for the Tikhonov solution y = P z.
// ---------------------------------------------------------------------------
typedef void (*dbdsqr_t)(char* uplo, int* n, int* ncvt, int* nru, int* ncc, double* d, double* e,
                         double* vt, int* ldvt, double* u, int* ldu, double* c, int* ldc,
                         double* work, int* info);
dbdsqr_t g_dbdsqr = nullptr;
bool g_lapack_bdsqr = [] {
    const char* e = getenv("CTK_LAPACK_BDSQR");    // 1: LAPACK dbdsqr instead of bdsvd()
    return e && e[0] == '1';
}();
bool g_fast = [] {
    const char* e = getenv("CTK_LAPACK_SVD");      // 1: always the dgesdd path
    return !(e && e[0] == '1');
}();

// ||x[1:n]||: plain sum of squares (vectorisable), rescaled only when it
// under/overflows (hypot per element costs ~30 ns).
double tail_norm(const double* x, int n, int stride) {
    double s = 0.0;
    for (int i = 1; i < n; ++i) {
        const double v = x[(size_t)i * stride];
        s += v * v;
    }
    if (s > 1e-290 && s < 1e290) return sqrt(s);
    double xn = 0.0;
    for (int i = 1; i < n; ++i) xn = hypot(xn, x[(size_t)i * stride]);
    return xn;
}

// dlarfg: reflector I - tau v v^T with v[0] = 1 mapping x to (beta, 0, ...).
void householder(double* x, int n, int stride, double* tau, double* beta) {
    const double alpha = x[0];
    const double xn = tail_norm(x, n, stride);
    if (xn == 0.0) {
        *tau = 0.0;
        *beta = alpha;
        return;
    }
    const double b = -copysign(hypot(alpha, xn), alpha);
    *tau = (b - alpha) / b;
    const double sc = 1.0 / (alpha - b);
    for (int i = 1; i < n; ++i) x[(size_t)i * stride] *= sc;
    x[0] = 1.0;
    *beta = b;
}

// Dense kernels of the bidiagonalisation (column-major, contiguous columns).
// The dot product is written with 8 independent partial sums so it
// vectorises without -ffast-math; AVX2/FMA clones are picked at load time.
#if defined(__x86_64__) && defined(__GNUC__) && !defined(__clang__)
#define CTK_HOT __attribute__((target_clones("arch=x86-64-v3", "default")))
#else
#define CTK_HOT
#endif

CTK_HOT double col_dot(const double* a, const double* b, int n) {
    double p[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int r = 0;
    for (; r + 8 <= n; r += 8)
        for (int q = 0; q < 8; ++q) p[q] += a[r + q] * b[r + q];
    double s = ((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]));
    for (; r < n; ++r) s += a[r] * b[r];
    return s;
}

CTK_HOT void col_axpy(double alpha, const double* x, double* y, int n) {
    for (int r = 0; r < n; ++r) y[r] += alpha * x[r];
}

// Four columns at a time (column-major, leading dimension ld): the per-column
// loop overhead, not the flops, bounded the unblocked kernels at k ~ 80.
// A[:, j] -= tau (v . A[:, j]) v for j < nc.  The four dot products of a
// column group share each load of v: AVX2/FMA when the CPU has it (checked
// once), else a portable loop.
#if defined(__x86_64__) && defined(__GNUC__) && !defined(__clang__)
#include <immintrin.h>
__attribute__((target("avx2,fma"))) void dots4_avx2(const double* v, const double* c0, int ld,
                                                   int len, double* out) {
    const double *c1 = c0 + ld, *c2 = c1 + ld, *c3 = c2 + ld;
    __m256d a0 = _mm256_setzero_pd(), a1 = a0, a2 = a0, a3 = a0;
    int r = 0;
    for (; r + 4 <= len; r += 4) {
        const __m256d vv = _mm256_loadu_pd(v + r);
        a0 = _mm256_fmadd_pd(vv, _mm256_loadu_pd(c0 + r), a0);
        a1 = _mm256_fmadd_pd(vv, _mm256_loadu_pd(c1 + r), a1);
        a2 = _mm256_fmadd_pd(vv, _mm256_loadu_pd(c2 + r), a2);
        a3 = _mm256_fmadd_pd(vv, _mm256_loadu_pd(c3 + r), a3);
    }
    // horizontal sums of the four accumulators at once
    const __m256d s01 = _mm256_hadd_pd(a0, a1), s23 = _mm256_hadd_pd(a2, a3);
    const __m256d t = _mm256_add_pd(_mm256_permute2f128_pd(s01, s23, 0x20),
                                    _mm256_permute2f128_pd(s01, s23, 0x31));
    _mm256_storeu_pd(out, t);
    for (; r < len; ++r) {
        out[0] += v[r] * c0[r];
        out[1] += v[r] * c1[r];
        out[2] += v[r] * c2[r];
        out[3] += v[r] * c3[r];
    }
}
const bool g_avx2 = [] {
    __builtin_cpu_init();       // runs in a static initializer: set up the CPU model first
    return __builtin_cpu_supports("avx2") && __builtin_cpu_supports("fma");
}();
#else
const bool g_avx2 = false;
void dots4_avx2(const double*, const double*, int, int, double*) {}
#endif

void dots4(const double* v, const double* c0, int ld, int len, double* out) {
    if (g_avx2) return dots4_avx2(v, c0, ld, len, out);
    for (int q = 0; q < 4; ++q) out[q] = col_dot(v, c0 + (size_t)q * ld, len);
}

CTK_HOT void left_update(const double* v, double* A, int ld, int nc, int len, double tau) {
    int j = 0;
    for (; j + 4 <= nc; j += 4) {
        double* c0 = A + (size_t)j * ld;
        double *c1 = c0 + ld, *c2 = c1 + ld, *c3 = c2 + ld;
        double sd[4];
        dots4(v, c0, ld, len, sd);
        const double s0 = -tau * sd[0], s1 = -tau * sd[1], s2 = -tau * sd[2], s3 = -tau * sd[3];
        for (int r = 0; r < len; ++r) {
            const double vv = v[r];
            c0[r] += s0 * vv;
            c1[r] += s1 * vv;
            c2[r] += s2 * vv;
            c3[r] += s3 * vv;
        }
    }
    for (; j < nc; ++j) {
        double* col = A + (size_t)j * ld;
        col_axpy(-tau * col_dot(v, col, len), v, col, len);
    }
}

// w = A[:, 0:nc] x (x[j] = the right reflector's entries).
CTK_HOT void gemv_cols(const double* A, int ld, int nc, int len, const double* x, double* w) {
    for (int r = 0; r < len; ++r) w[r] = 0.0;
    int j = 0;
    for (; j + 4 <= nc; j += 4) {
        const double* c0 = A + (size_t)j * ld;
        const double *c1 = c0 + ld, *c2 = c1 + ld, *c3 = c2 + ld;
        const double x0 = x[j], x1 = x[j + 1], x2 = x[j + 2], x3 = x[j + 3];
        for (int r = 0; r < len; ++r) w[r] += (x0 * c0[r] + x1 * c1[r]) + (x2 * c2[r] + x3 * c3[r]);
    }
    for (; j < nc; ++j) col_axpy(x[j], A + (size_t)j * ld, w, len);
}

// A[:, j] -= tau x[j] w for j < nc.
CTK_HOT void rank1_cols(double* A, int ld, int nc, int len, const double* x, const double* w,
                        double tau) {
    int j = 0;
    for (; j + 4 <= nc; j += 4) {
        double* c0 = A + (size_t)j * ld;
        double *c1 = c0 + ld, *c2 = c1 + ld, *c3 = c2 + ld;
        const double a0 = -tau * x[j], a1 = -tau * x[j + 1], a2 = -tau * x[j + 2],
                     a3 = -tau * x[j + 3];
        for (int r = 0; r < len; ++r) {
            const double ww = w[r];
            c0[r] += a0 * ww;
            c1[r] += a1 * ww;
            c2[r] += a2 * ww;
            c3[r] += a3 * ww;
        }
    }
    for (; j < nc; ++j) col_axpy(-tau * x[j], w, A + (size_t)j * ld, len);
}

struct Bidiag {
    int m = 0, n = 0;
    std::vector<double> A;      // m x n column-major, right reflectors stored in rows
    std::vector<double> d, e, taup, g;
    std::vector<double> tmp;    // the current right reflector, contiguous
};

// H (m x n row-major) -> B = diag d + superdiag e; g = Q^T (beta e1).
void bidiagonalize(const double* H, int m, int n, double beta, Bidiag& bd) {
    bd.m = m;
    bd.n = n;
    bd.A.assign((size_t)m * n, 0.0);
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < n; ++j) bd.A[(size_t)i + (size_t)j * m] = H[(size_t)i * n + j];
    bd.d.assign(n, 0.0);
    bd.e.assign(n > 1 ? n - 1 : 1, 0.0);
    bd.taup.assign(n, 0.0);
    bd.g.assign(m, 0.0);
    bd.g[0] = beta;
    double* A = bd.A.data();
    auto at = [&](int i, int j) -> double& { return A[(size_t)i + (size_t)j * m]; };
    std::vector<double> w(m > n ? m : n);
    for (int i = 0; i < n; ++i) {
        // left reflector on column i, rows i..m-1
        double tq, b;
        householder(&at(i, i), m - i, 1, &tq, &b);
        if (tq != 0.0) {
            const double* v = &at(i, i);
            left_update(v, &at(i, i + 1), m, n - i - 1, m - i, tq);
            col_axpy(-tq * col_dot(v, &bd.g[i], m - i), v, &bd.g[i], m - i);
        }
        bd.d[i] = b;
        if (i < n - 1) {
            // right reflector on row i, columns i+1..n-1 (stored in place)
            double tp, b2;
            householder(&at(i, i + 1), n - i - 1, m, &tp, &b2);
            bd.taup[i] = tp;
            bd.e[i] = b2;
            if (tp != 0.0) {
                // w = A(i+1:, i+1:) v by columns (contiguous), then the rank-1 update
                const int nc = n - i - 1, len = m - i - 1;
                std::vector<double>& x = bd.tmp;
                x.resize(nc);
                for (int j = 0; j < nc; ++j) x[j] = at(i, i + 1 + j);
                gemv_cols(&at(i + 1, i + 1), m, nc, len, x.data(), &w[i + 1]);
                rank1_cols(&at(i + 1, i + 1), m, nc, len, x.data(), &w[i + 1], tp);
            }
        }
    }
}

// y = P z = G_0 (G_1 (... G_{n-2} z)) with G_i = I - tau_i v_i v_i^T on coords i+1..n-1.
void apply_p(const Bidiag& bd, const double* z, double* y) {
    const int n = bd.n, m = bd.m;
    for (int j = 0; j < n; ++j) y[j] = z[j];
    for (int i = n - 2; i >= 0; --i) {
        const double tp = bd.taup[i];
        if (tp == 0.0) continue;
        double s = y[i + 1];                               // v[0] = 1
        for (int j = i + 2; j < n; ++j) s += bd.A[(size_t)i + (size_t)j * m] * y[j];
        s *= tp;
        y[i + 1] -= s;
        for (int j = i + 2; j < n; ++j) y[j] -= s * bd.A[(size_t)i + (size_t)j * m];
    }
}

// min ||B z - g||^2 + lam^2 ||z||^2 for upper bidiagonal B (d, e): QR of
// [B; lam I] by Givens rotations in O(n) (Elden's bidiagonal scheme): row i of
// B absorbs the running damping row (pivot delta at column i), whose fill-in
// -s e_i at column i+1 is folded into the next damping row lam e_{i+1}, so
// every row needs two rotations and the triangular factor stays bidiagonal.
// Returns false when lam == 0 and B is numerically singular.
bool damped_bidiag_solve(std::vector<double> d, std::vector<double> e, std::vector<double> g,
                         double lam, double smax, int m_rows, double* z) {
    const int n = (int)d.size();
    auto hyp = [](double a, double b) {
        const double ss = a * a + b * b;     // |a|, |b| are matrix-scale: no hypot needed
        return (ss > 1e-290 && ss < 1e290) ? sqrt(ss) : hypot(a, b);
    };
    if (lam > 0.0) {
        double delta = lam, rho = 0.0;       // running damping row: delta at column i, rhs rho
        for (int i = 0; i < n; ++i) {
            const double h = hyp(d[i], delta);
            const double cs = d[i] / h, sn = delta / h;
            d[i] = h;
            const double gi = g[i];
            g[i] = cs * gi + sn * rho;
            rho = -sn * gi + cs * rho;
            if (i + 1 < n) {
                const double f = -sn * e[i];  // fill-in of the damping row at column i+1
                e[i] = cs * e[i];
                const double h2 = hyp(lam, f);
                rho = (f / h2) * rho;         // merged with the damping row lam e_{i+1}
                delta = h2;
            }
        }
    } else {
        const double cutoff = std::numeric_limits<double>::epsilon() * std::max(m_rows, n) * smax;
        for (int c = 0; c < n; ++c)
            if (!(fabs(d[c]) > cutoff)) return false;
    }
    z[n - 1] = g[n - 1] / d[n - 1];
    for (int c = n - 2; c >= 0; --c) z[c] = (g[c] - e[c] * z[c + 1]) / d[c];
    return true;
}

// rotation (c, s, r) with c*y + s*z = r, -s*y + c*z = 0
inline void rot(double y, double z, double* c, double* s, double* r) {
    if (z == 0.0) {
        *c = 1.0;
        *s = 0.0;
        *r = y;
        return;
    }
    const double ss = y * y + z * z;
    const double h = (ss > 1e-290 && ss < 1e290) ? sqrt(ss) : hypot(y, z);
    const double inv = 1.0 / h;
    *c = y * inv;
    *s = z * inv;
    *r = h;
}
// Singular values of the upper bidiagonal B (d[0..n-1], e[0..n-2]) with the
// left rotations applied to one vector: on return d = singular values
// (descending), g = U^T g up to per-entry signs.  Golub-Kahan implicit-shift
// QR (Wilkinson shift from the trailing 2x2 of B^T B), bulge chased top to
// bottom, deflation when |e_i| <= eps (|d_i| + |d_i+1|), zero diagonals
// rotated out (Golub & Van Loan, Alg. 8.6.2).  It replaces LAPACK dbdsqr with
// ncc = 1, which spends most of its time in per-rotation dlartg/drot calls.
// Returns 0, or 1 if it did not converge (the caller falls back to dgesdd).
int bdsvd(int n, double* d, double* e, double* g) {
    const double eps = std::numeric_limits<double>::epsilon();
    double anorm = 0.0;
    for (int i = 0; i < n; ++i)
        anorm = std::max(anorm, fabs(d[i]) + (i + 1 < n ? fabs(e[i]) : 0.0));
    const double dtol = eps * anorm;
    int q = n - 1, iter = 0;
    const int maxit = 30 * n * n;
    while (q > 0) {
        if (++iter > maxit) return 1;
        // deflation at the bottom
        if (fabs(e[q - 1]) <= eps * (fabs(d[q - 1]) + fabs(d[q])) || fabs(e[q - 1]) <= 1e-300) {
            e[q - 1] = 0.0;
            --q;
            continue;
        }
        int p = q - 1;
        while (p > 0) {
            if (fabs(e[p - 1]) <= eps * (fabs(d[p - 1]) + fabs(d[p]))) {
                e[p - 1] = 0.0;
                break;
            }
            --p;
        }
        // zero diagonal inside the block
        int zi = -1;
        for (int i = p; i <= q; ++i)
            if (fabs(d[i]) <= dtol) {
                zi = i;
                break;
            }
        if (zi >= 0) {
            d[zi] = 0.0;
            if (zi < q) {       // chase e[zi] right with left rotations (rows j, zi)
                double f = e[zi]; e[zi] = 0.0;
                for (int j = zi + 1; j <= q && f != 0.0; ++j) {
                    double c, s, r; rot(d[j], f, &c, &s, &r);
                    d[j] = r;
                    const double gj = g[j], gi = g[zi];
                    g[j] = c * gj + s * gi; g[zi] = -s * gj + c * gi;
                    if (j < q) { f = -s * e[j]; e[j] = c * e[j]; }
                }
            } else {            // d[q] == 0: chase e[q-1] up with right rotations (columns k, q)
                double f = e[q - 1]; e[q - 1] = 0.0;
                for (int k = q - 1; k >= p && f != 0.0; --k) {
                    double c, s, r; rot(d[k], f, &c, &s, &r);
                    d[k] = r;
                    if (k > p) { f = -s * e[k - 1]; e[k - 1] = c * e[k - 1]; }
                }
            }
            continue;
        }
        // Wilkinson shift from the trailing 2x2 of B^T B
        const double dm = d[q - 1], em = e[q - 1], dq = d[q];
        const double t11 = dm * dm + (q - 1 > p ? e[q - 2] * e[q - 2] : 0.0);
        const double t12 = dm * em, t22 = dq * dq + em * em;
        const double dl = 0.5 * (t11 - t22);
        const double den = dl + copysign(sqrt(dl * dl + t12 * t12), dl);
        const double mu = den != 0.0 ? t22 - t12 * t12 / den : t22 - fabs(t12);
        double y = d[p] * d[p] - mu, z = d[p] * e[p];
        for (int k = p; k < q; ++k) {
            double c, s, r;
            rot(y, z, &c, &s, &r);                   // right: columns k, k+1
            if (k > p) e[k - 1] = r;
            double a = d[k], b = e[k];
            d[k] = c * a + s * b; e[k] = -s * a + c * b;
            const double bl = s * d[k + 1];
            d[k + 1] = c * d[k + 1];
            rot(d[k], bl, &c, &s, &r);              // left: rows k, k+1
            d[k] = r;
            a = e[k]; b = d[k + 1];
            e[k] = c * a + s * b; d[k + 1] = -s * a + c * b;
            if (k + 1 < q) { z = s * e[k + 1]; e[k + 1] = c * e[k + 1]; }
            y = e[k];
            const double g0 = g[k], g1 = g[k + 1];
            g[k] = c * g0 + s * g1; g[k + 1] = -s * g0 + c * g1;
        }
    }
    for (int i = 0; i < n; ++i) d[i] = fabs(d[i]);
    // sort descending (insertion sort; n is small), g alongside
    for (int i = 1; i < n; ++i) {
        const double dv = d[i], gv = g[i]; int j = i - 1;
        while (j >= 0 && d[j] < dv) { d[j + 1] = d[j]; g[j + 1] = g[j]; --j; }
        d[j + 1] = dv; g[j + 1] = gv;
    }
    return 0;
}
// 0 = done, 1 = fall back to the dgesdd path (lam == 0 and rank deficient, or
// dbdsqr unavailable / failed).
int projected_fast(const double* H, int k, double beta, int strategy, double fixed_value,
                   int grid_count, double fallback_lambda, double* out, double* y) {
    if (!g_dbdsqr) return 1;
    const int m = k + 1, n = k;
    Bidiag bd;
    bidiagonalize(H, m, n, beta, bd);
    std::vector<double> sv(bd.d), ee(bd.e), c(bd.g.begin(), bd.g.begin() + n);
    if (g_lapack_bdsqr) {
        std::vector<double> work(4 * (size_t)n + 4);
        char uplo = 'U';
        int nn = n, ncvt = 0, nru = 0, ncc = 1, ldvt = 1, ldu = 1, ldc = n, info = 0;
        double dummy = 0.0;
        g_dbdsqr(&uplo, &nn, &ncvt, &nru, &ncc, sv.data(), ee.data(), &dummy, &ldvt, &dummy,
                 &ldu, c.data(), &ldc, work.data(), &info);
        if (info != 0) return 1;
    } else if (bdsvd(n, sv.data(), ee.data(), c.data()) != 0) {
        return 1;
    }
    // c = U^T (beta e1) up to per-column signs, which the filter-factor
    // formulas square away: the same (s, c) as beta * U[0, :] of the reference SVD.
    double lam = 0.0;
    int degenerate = 0;
    if (strategy == S_FIXED) {
        lam = fixed_value;
    } else if (strategy == S_LCURVE || strategy == S_GCV) {
        if (select_sc(sv.data(), c, k, m, beta, strategy, grid_count, &lam)) {
            degenerate = 1;
            lam = fallback_lambda;
        }
    }
    out[0] = lam;
    out[2] = degenerate;
    out[3] = 0;
    if (isnan(lam)) {
        out[1] = 0.0;
        return 0;
    }
    std::vector<double> z(n);
    std::vector<double> gn(bd.g.begin(), bd.g.begin() + n);
    if (!damped_bidiag_solve(bd.d, std::vector<double>(bd.e.begin(), bd.e.begin() + (n > 1 ? n - 1 : 0)),
                             gn, lam, sv.empty() ? 0.0 : sv[0], m, z.data()))
        return 1;
    apply_p(bd, z.data(), y);
    double r2 = 0.0;
    for (int i = 0; i < m; ++i) {
        double a = (i == 0) ? -beta : 0.0;
        for (int j = 0; j < n; ++j) a += H[(size_t)i * n + j] * y[j];
        r2 += a * a;
    }
    out[1] = sqrt(r2);
    return 0;
}

}  // namespace

extern "C" int ctk_set_svd_path(int lapack_only) {
    g_fast = lapack_only == 0;
    return CTK_OK;
}

extern "C" int ctk_set_lapack_extra(void* dbdsqr) {
    g_dbdsqr = reinterpret_cast<dbdsqr_t>(dbdsqr);
    return CTK_OK;
}

extern "C" int ctk_set_lapack(void* dgesdd, void* ddot) {
    g_dgesdd = reinterpret_cast<dgesdd_t>(dgesdd);
    g_ddot = reinterpret_cast<ddot_t>(ddot);
    return g_dgesdd ? CTK_OK : ctk_fail(CTK_ERR_ARG, "null dgesdd");
}

extern "C" int ctk_projected_solve(const double* H, int k, double beta, int strategy,
                                   double fixed_value, int grid_count, double fallback_lambda,
                                   double* out, double* y) {
    if (!g_dgesdd) return ctk_fail(CTK_ERR_ARG, "LAPACK dgesdd not registered (ctk_set_lapack)");
    if (!H || !out || !y || k < 1 || grid_count < 1)
        return ctk_fail(CTK_ERR_ARG, "bad projected-solve arguments");
    if (g_fast && projected_fast(H, k, beta, strategy, fixed_value, grid_count, fallback_lambda,
                                 out, y) == 0)
        return CTK_OK;
    Svd v;
    const int info = svd_hessenberg(H, k + 1, k, v);
    if (info != 0) return ctk_fail(CTK_ERR_ARG, "dgesdd failed (info %d)", info);
    double lam = 0.0;
    int degenerate = 0;
    if (strategy == S_FIXED) {
        lam = fixed_value;
    } else if (strategy == S_LCURVE || strategy == S_GCV) {
        if (select(v, beta, strategy, grid_count, &lam)) {
            degenerate = 1;
            lam = fallback_lambda;
        }
    }
    double res = 0.0;
    int rank_def = 0;
    if (!isnan(lam)) tikhonov(H, v, beta, lam, y, &res, &rank_def);
    out[0] = lam;
    out[1] = res;
    out[2] = degenerate;
    out[3] = rank_def;
    return CTK_OK;
}
