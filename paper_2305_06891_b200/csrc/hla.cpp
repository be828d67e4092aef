// H-arithmetic on the host (see hla.h): the block H-LU of PAPER.md:751-779 and the solve forms.
//
// Case analysis of the recursive operations (Hackbusch 2015, as PAPER.md:777 refers to it), every
// matrix in F's block tree:
//   hmul    C += a op(A) B          A an H-block, B / C dense multi-vectors
//   solve   B <- T^-1 B, T^-T B     T a diagonal H-block holding packed unit-lower L / upper U
//   trsm    X <- L^-1 X, U^-1 X, X L^-1, X U^-1   X an H-block (dense / low rank / subdivided)
//   mm      C += a A B              C, A, B H-blocks; a low-rank result is added with truncation
//   addlr   C += U V^T              split along C's tree, truncated at every low-rank leaf
// Truncation (reading R5): QR of both factors, one-sided Jacobi SVD of the small
// core, keep the smallest rank whose Frobenius tail is <= eps of the block's Frobenius norm.
// Parallelism: OpenMP tasks over independent target blocks (the four quadrants of a product, the
// column halves of a left substitution, ...).  Every block's operations run in the same order
// whatever the schedule, so the factors are bitwise reproducible.
#include "hla.h"

#include <omp.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>

#include "hm_internal.h"

namespace hm {
namespace hla {

using Vec = std::vector<double>;

static std::atomic<int64_t> g_prof[24];
static std::atomic<int64_t> g_ns[24];
struct ProfT {
    int id;
    std::chrono::steady_clock::time_point t0;
    explicit ProfT(int i) : id(i), t0(std::chrono::steady_clock::now()) {}
    ~ProfT() {
        g_prof[id].fetch_add(1, std::memory_order_relaxed);
        g_ns[id].fetch_add(std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count(),
                           std::memory_order_relaxed);
    }
};
static std::atomic<int64_t> g_hist[5], g_histk[5];
void prof_dump() {
    for (int b = 0; b < 5; ++b)
        if (g_hist[b]) fprintf(stderr, "  addlr-lr max(m,n) bucket %d: %lld calls, mean update rank %.1f\n", b,
                               (long long)g_hist[b].load(), (double)g_histk[b].load() / g_hist[b].load());
    static const char* names[24] = {"trunc", "qr", "jacobi", "trunc-gemm", "addlr-lr", "agglom", "mm-lrlr", "mm-lrA",
                                    "mm-lrB", "hmul-dense", "hmul-lr", "solve-dense", "lu-dense", "mm-dd", "addlr-subtop", "compress-dense",
                                    "trsmR-dense", "mmLR-dd", "mmLR-dsub", "mmLR-subd", "mmLR-subsub", "addlr-dense", "form-leaf", "x"};
    for (int i = 0; i < 24; ++i)
        if (g_prof[i]) fprintf(stderr, "  %-12s %10lld calls %9.3f s\n", names[i], (long long)g_prof[i].load(), g_ns[i].load() * 1e-9);
}


// ============================================================================ dense kernels
// column-major; C(m x n) += alpha A(m x k) op(B), op(B)(l, j) = BT ? B[j + l ldb] : B[l + j ldb]
template <bool BT>
static void gemm_n(int64_t m, int64_t n, int64_t k, double alpha, const double* A, int64_t lda, const double* B,
                   int64_t ldb, double* C, int64_t ldc) {
    if (m <= 0 || n <= 0 || k <= 0 || alpha == 0.0) return;
    auto bv = [&](int64_t l, int64_t j) { return BT ? B[j + l * ldb] : B[l + j * ldb]; };
    int64_t i0 = 0;
    for (; i0 + 8 <= m; i0 += 8) {
        int64_t j0 = 0;
        // 8 x 6 register tile (12 accumulator vectors of 4 doubles; measured 23.5 vs 19.8 GFLOP/s per
        // core for the 8 x 4 tile on 80 x 80 x 80)
        for (; j0 + 6 <= n; j0 += 6) {
            double acc[6][8] = {};
            for (int64_t l = 0; l < k; ++l) {
                const double* a = A + i0 + l * lda;
                double b[6];
                for (int jj = 0; jj < 6; ++jj) b[jj] = bv(l, j0 + jj);
#pragma omp simd
                for (int ii = 0; ii < 8; ++ii)
                    for (int jj = 0; jj < 6; ++jj) acc[jj][ii] += a[ii] * b[jj];
            }
            for (int jj = 0; jj < 6; ++jj) {
                double* c = C + i0 + (j0 + jj) * ldc;
#pragma omp simd
                for (int ii = 0; ii < 8; ++ii) c[ii] += alpha * acc[jj][ii];
            }
        }
        for (; j0 < n; ++j0) {
            double acc[8] = {};
            for (int64_t l = 0; l < k; ++l) {
                const double* a = A + i0 + l * lda;
                const double b = bv(l, j0);
#pragma omp simd
                for (int ii = 0; ii < 8; ++ii) acc[ii] += a[ii] * b;
            }
            double* c = C + i0 + j0 * ldc;
            for (int ii = 0; ii < 8; ++ii) c[ii] += alpha * acc[ii];
        }
    }
    for (; i0 < m; ++i0)
        for (int64_t j = 0; j < n; ++j) {
            double s = 0.0;
            for (int64_t l = 0; l < k; ++l) s += A[i0 + l * lda] * bv(l, j);
            C[i0 + j * ldc] += alpha * s;
        }
}

static void gemm_nn(int64_t m, int64_t n, int64_t k, double alpha, const double* A, int64_t lda, const double* B,
                    int64_t ldb, double* C, int64_t ldc) {
    gemm_n<false>(m, n, k, alpha, A, lda, B, ldb, C, ldc);
}
static void gemm_nt(int64_t m, int64_t n, int64_t k, double alpha, const double* A, int64_t lda, const double* B,
                    int64_t ldb, double* C, int64_t ldc) {
    gemm_n<true>(m, n, k, alpha, A, lda, B, ldb, C, ldc);
}
// C(m x n) += alpha A^T B, A is k x m, B is k x n (dot products over the long dimension k)
static void gemm_tn(int64_t m, int64_t n, int64_t k, double alpha, const double* A, int64_t lda, const double* B,
                    int64_t ldb, double* C, int64_t ldc) {
    if (m <= 0 || n <= 0 || k <= 0 || alpha == 0.0) return;
    for (int64_t j = 0; j < n; ++j) {
        const double* b = B + j * ldb;
        int64_t i = 0;
        for (; i + 4 <= m; i += 4) {
            const double *a0 = A + i * lda, *a1 = a0 + lda, *a2 = a1 + lda, *a3 = a2 + lda;
            double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
#pragma omp simd reduction(+ : s0, s1, s2, s3)
            for (int64_t l = 0; l < k; ++l) {
                s0 += a0[l] * b[l];
                s1 += a1[l] * b[l];
                s2 += a2[l] * b[l];
                s3 += a3[l] * b[l];
            }
            C[i + j * ldc] += alpha * s0;
            C[i + 1 + j * ldc] += alpha * s1;
            C[i + 2 + j * ldc] += alpha * s2;
            C[i + 3 + j * ldc] += alpha * s3;
        }
        for (; i < m; ++i) {
            const double* a = A + i * lda;
            double s = 0;
#pragma omp simd reduction(+ : s)
            for (int64_t l = 0; l < k; ++l) s += a[l] * b[l];
            C[i + j * ldc] += alpha * s;
        }
    }
}

static Vec transpose(const double* A, int64_t m, int64_t n, int64_t lda) {   // (m x n) -> (n x m)
    Vec T((size_t)(m * n));
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) T[j + i * n] = A[i + j * lda];
    return T;
}

enum SolveKind : int { S_LL = 0, S_LU = 1, S_LLT = 2, S_LUT = 3 };
// B (m x r) <- op(T)^-1 B with T the packed LU of an m x m dense diagonal leaf (ld m)
static void trsm_dense1(int kind, const double* T, int64_t m, double* B, int64_t ldb, int64_t r);
static void trsm_dense(int kind, const double* T, int64_t m, double* B, int64_t ldb, int64_t r) {
    // the column forms (unit lower / upper, the common ones) four right-hand sides at a time: every
    // column of T is loaded once per four updates
    int64_t j = 0;
    if (kind == S_LL || kind == S_LU) {
        for (; j + 4 <= r; j += 4) {
            double* __restrict b0 = B + j * ldb;
            double* __restrict b1 = b0 + ldb;
            double* __restrict b2 = b1 + ldb;
            double* __restrict b3 = b2 + ldb;
            if (kind == S_LL) {
                for (int64_t l = 0; l < m; ++l) {
                    const double* __restrict t = T + l * m;
                    const double x0 = b0[l], x1 = b1[l], x2 = b2[l], x3 = b3[l];
#pragma omp simd
                    for (int64_t i = l + 1; i < m; ++i) {
                        const double ti = t[i];
                        b0[i] -= ti * x0;
                        b1[i] -= ti * x1;
                        b2[i] -= ti * x2;
                        b3[i] -= ti * x3;
                    }
                }
            } else {
                for (int64_t l = m - 1; l >= 0; --l) {
                    const double* __restrict t = T + l * m;
                    const double inv = 1.0 / t[l];
                    b0[l] *= inv;
                    b1[l] *= inv;
                    b2[l] *= inv;
                    b3[l] *= inv;
                    const double x0 = b0[l], x1 = b1[l], x2 = b2[l], x3 = b3[l];
#pragma omp simd
                    for (int64_t i = 0; i < l; ++i) {
                        const double ti = t[i];
                        b0[i] -= ti * x0;
                        b1[i] -= ti * x1;
                        b2[i] -= ti * x2;
                        b3[i] -= ti * x3;
                    }
                }
            }
        }
    }
    if (j < r) trsm_dense1(kind, T, m, B + j * ldb, ldb, r - j);
}

static void trsm_dense1(int kind, const double* T, int64_t m, double* B, int64_t ldb, int64_t r) {
    for (int64_t j = 0; j < r; ++j) {
        double* b = B + j * ldb;
        switch (kind) {
        case S_LL:   // unit lower
            for (int64_t l = 0; l < m; ++l) {
                const double x = b[l];
                if (x == 0.0) continue;
                const double* t = T + l * m;
#pragma omp simd
                for (int64_t i = l + 1; i < m; ++i) b[i] -= t[i] * x;
            }
            break;
        case S_LU:   // upper
            for (int64_t l = m - 1; l >= 0; --l) {
                const double* t = T + l * m;
                b[l] /= t[l];
                const double x = b[l];
                if (x == 0.0) continue;
#pragma omp simd
                for (int64_t i = 0; i < l; ++i) b[i] -= t[i] * x;
            }
            break;
        case S_LLT:  // (unit lower)^T = unit upper
            for (int64_t l = m - 1; l >= 0; --l) {
                const double* t = T + l * m;
                double s = 0.0;
#pragma omp simd reduction(+ : s)
                for (int64_t i = l + 1; i < m; ++i) s += t[i] * b[i];
                b[l] -= s;
            }
            break;
        case S_LUT:  // upper^T = lower
            for (int64_t l = 0; l < m; ++l) {
                const double* t = T + l * m;
                double s = 0.0;
#pragma omp simd reduction(+ : s)
                for (int64_t i = 0; i < l; ++i) s += t[i] * b[i];
                b[l] = (b[l] - s) / t[l];
            }
            break;
        }
    }
}

// in-place LU without pivoting of an m x m column-major block; false on a pivot below 1e-14 ||A||_max
static bool lu_dense(double* A, int64_t m) {
    double amax = 0.0;
    for (int64_t i = 0; i < m * m; ++i) amax = std::max(amax, std::fabs(A[i]));
    for (int64_t l = 0; l < m; ++l) {
        const double piv = A[l + l * m];
        if (!(std::fabs(piv) > 1e-14 * amax)) return false;
        const double inv = 1.0 / piv;
        for (int64_t i = l + 1; i < m; ++i) A[i + l * m] *= inv;
        const double* cl = A + l * m;
        for (int64_t j = l + 1; j < m; ++j) {
            double* cj = A + j * m;
            const double a = cj[l];
            if (a == 0.0) continue;
#pragma omp simd
            for (int64_t i = l + 1; i < m; ++i) cj[i] -= cl[i] * a;
        }
    }
    return true;
}

// packed LU -> packed inverse factors: strictly lower part of L^-1, upper part (with diagonal) of U^-1
static void invert_packed(double* A, int64_t m) {
    Vec Li((size_t)(m * m), 0.0), Ui((size_t)(m * m), 0.0);
    for (int64_t i = 0; i < m; ++i) Li[i + i * m] = Ui[i + i * m] = 1.0;
    trsm_dense(S_LL, A, m, Li.data(), m, m);
    trsm_dense(S_LU, A, m, Ui.data(), m, m);
    for (int64_t j = 0; j < m; ++j)
        for (int64_t i = 0; i < m; ++i) A[i + j * m] = i > j ? Li[i + j * m] : Ui[i + j * m];
}

// ---------------------------------------------------------------- QR (Householder) + Jacobi SVD
// A (m x K column-major) = Q R, R kq x K upper (kq = min(m, K)); Q kept as Householder reflectors
// (W below the diagonal, tau) and applied with apply_q (Q is never formed).
// H = I - tau v v^T (v = [1; x[j+1..m)]) applied to rows j.. of the nc columns Y (ld m), four at a
// time so every load of x feeds four dot products / updates
static inline void reflect(const double* __restrict x, int j, int64_t m, double tj, double* Y, int64_t ldy, int nc) {
    int c = 0;
    for (; c + 4 <= nc; c += 4) {
        double* __restrict y0 = Y + (int64_t)c * ldy;
        double* __restrict y1 = y0 + ldy;
        double* __restrict y2 = y1 + ldy;
        double* __restrict y3 = y2 + ldy;
        double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
#pragma omp simd reduction(+ : s0, s1, s2, s3)
        for (int64_t i = j + 1; i < m; ++i) {
            const double xi = x[i];
            s0 += xi * y0[i];
            s1 += xi * y1[i];
            s2 += xi * y2[i];
            s3 += xi * y3[i];
        }
        s0 = (s0 + y0[j]) * tj;
        s1 = (s1 + y1[j]) * tj;
        s2 = (s2 + y2[j]) * tj;
        s3 = (s3 + y3[j]) * tj;
        y0[j] -= s0;
        y1[j] -= s1;
        y2[j] -= s2;
        y3[j] -= s3;
#pragma omp simd
        for (int64_t i = j + 1; i < m; ++i) {
            const double xi = x[i];
            y0[i] -= s0 * xi;
            y1[i] -= s1 * xi;
            y2[i] -= s2 * xi;
            y3[i] -= s3 * xi;
        }
    }
    for (; c < nc; ++c) {
        double* __restrict y = Y + (int64_t)c * ldy;
        double s = 0.0;
#pragma omp simd reduction(+ : s)
        for (int64_t i = j + 1; i < m; ++i) s += x[i] * y[i];
        s = (s + y[j]) * tj;
        y[j] -= s;
#pragma omp simd
        for (int64_t i = j + 1; i < m; ++i) y[i] -= s * x[i];
    }
}

struct QR {
    int64_t m = 0;
    int K = 0, kq = 0;
    Vec W, tau, R;
};
static void qr(int64_t m, int K, const double* A, QR& f) {
    f.m = m;
    f.K = K;
    const int kq = f.kq = (int)std::min<int64_t>(m, K);
    f.W.assign(A, A + m * K);
    f.tau.assign((size_t)kq, 0.0);
    double* __restrict Wp = f.W.data();
    for (int j = 0; j < kq; ++j) {
        double* __restrict x = Wp + (int64_t)j * m;
        double nrm2 = 0.0;
        for (int64_t i = j; i < m; ++i) nrm2 += x[i] * x[i];
        const double nrm = std::sqrt(nrm2);
        if (nrm == 0.0) continue;
        const double a0 = x[j];
        const double beta = a0 >= 0.0 ? -nrm : nrm;
        const double sc = 1.0 / (a0 - beta);
        for (int64_t i = j + 1; i < m; ++i) x[i] *= sc;
        const double tj = f.tau[j] = (beta - a0) / beta;
        x[j] = beta;
        reflect(x, j, m, tj, Wp + (int64_t)(j + 1) * m, m, K - j - 1);
    }
    f.R.assign((size_t)kq * K, 0.0);
    for (int c = 0; c < K; ++c)
        for (int i = 0; i <= std::min(c, kq - 1); ++i) f.R[i + (int64_t)c * kq] = Wp[i + (int64_t)c * f.m];
}
// out (m x c) = Q [A; 0], A kq x c column-major (ld kq)
static void apply_q(const QR& f, const double* A, int c, double* out) {
    const int64_t m = f.m;
    const int kq = f.kq;
    std::fill(out, out + m * c, 0.0);
    for (int l = 0; l < c; ++l)
        for (int i = 0; i < kq; ++i) out[i + (int64_t)l * m] = A[i + (int64_t)l * kq];
    const double* __restrict Wp = f.W.data();
    for (int j = kq - 1; j >= 0; --j) {
        const double tj = f.tau[j];
        if (tj == 0.0) continue;
        reflect(Wp + (int64_t)j * m, j, m, tj, out, m, c);
    }
}

// One-sided (Hestenes) Jacobi: W (p x q) <- W Y with orthogonal columns, Y (q x q) orthogonal.
// W Y^T stays equal to the input whatever the convergence, so dropping columns of W later costs
// exactly their Frobenius norm: the orthogonality tolerance only affects how small the kept rank
// is.  Pairs whose smaller column is below `tiny` (squared norm, far under the truncation level)
// are not rotated.
static void jacobi(int p, int q, double* W, double* Y, double tiny) {
    std::fill(Y, Y + (int64_t)q * q, 0.0);
    for (int i = 0; i < q; ++i) Y[i + (int64_t)i * q] = 1.0;
    std::vector<double> nrm((size_t)q);
    for (int i = 0; i < q; ++i) {
        double a = 0;
        for (int r = 0; r < p; ++r) a += W[r + (int64_t)i * p] * W[r + (int64_t)i * p];
        nrm[i] = a;
    }
    for (int sweep = 0; sweep < 30; ++sweep) {
        bool rot = false;
        for (int i = 0; i < q - 1; ++i) {
            double* wi = W + (int64_t)i * p;
            for (int j = i + 1; j < q; ++j) {
                double* wj = W + (int64_t)j * p;
                const double a = nrm[i], b = nrm[j];
                if (a <= tiny || b <= tiny) continue;
                double g = 0;
#pragma omp simd reduction(+ : g)
                for (int r = 0; r < p; ++r) g += wi[r] * wj[r];
                if (std::fabs(g) <= 1e-11 * std::sqrt(a * b)) continue;
                rot = true;
                const double zeta = (b - a) / (2.0 * g);
                const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
#pragma omp simd
                for (int r = 0; r < p; ++r) {
                    const double x = wi[r], y = wj[r];
                    wi[r] = c * x - s * y;
                    wj[r] = s * x + c * y;
                }
                // updated squared norms (exact for the rotation angle chosen)
                nrm[i] = a - t * g;
                nrm[j] = b + t * g;
                double* yi = Y + (int64_t)i * q;
                double* yj = Y + (int64_t)j * q;
#pragma omp simd
                for (int r = 0; r < q; ++r) {
                    const double x = yi[r], y = yj[r];
                    yi[r] = c * x - s * y;
                    yj[r] = s * x + c * y;
                }
            }
        }
        if (!rot) break;
        for (int i = 0; i < q; ++i) {   // refresh the norms once per sweep (rounding drift)
            double a = 0;
            for (int r = 0; r < p; ++r) a += W[r + (int64_t)i * p] * W[r + (int64_t)i * p];
            nrm[i] = a;
        }
    }
}

int truncate(int64_t m, int64_t n, int K, Vec& U, Vec& V, double eps) {
    ProfT _p(0);
    if (K <= 0 || m <= 0 || n <= 0) {
        U.clear();
        V.clear();
        return 0;
    }
    QR fu, fv;
    {
        ProfT _q(1);
        qr(m, K, U.data(), fu);
        qr(n, K, V.data(), fv);
    }
    const int ku = fu.kq, kv = fv.kq;
    const Vec &Ru = fu.R, &Rv = fv.R;
    // core M = Ru Rv^T (ku x kv)
    Vec M((size_t)ku * kv, 0.0);
    gemm_nt(ku, kv, K, 1.0, Ru.data(), ku, Rv.data(), kv, M.data(), ku);
    // SVD by one-sided Jacobi on the orientation with fewer columns
    const bool tr = kv > ku;
    const int p = tr ? kv : ku, q = tr ? ku : kv;
    Vec W = tr ? transpose(M.data(), ku, kv, ku) : M;   // p x q
    Vec Y((size_t)q * q);
    {
        ProfT _j(2);
        double tot = 0.0;
        for (double w : W) tot += w * w;
        jacobi(p, q, W.data(), Y.data(), 1e-6 * eps * eps * tot);
    }
    std::vector<std::pair<double, int>> sv((size_t)q);
    double tot = 0.0;
    for (int i = 0; i < q; ++i) {
        double s2 = 0.0;
        for (int r = 0; r < p; ++r) s2 += W[r + (int64_t)i * p] * W[r + (int64_t)i * p];
        sv[i] = {s2, i};
        tot += s2;
    }
    std::sort(sv.begin(), sv.end(), [](const std::pair<double, int>& a, const std::pair<double, int>& b) {
        return a.first > b.first || (a.first == b.first && a.second < b.second);
    });
    int kn = 0;
    if (tot > 0.0) {
        double tail = tot;
        const double lim = eps * eps * tot;
        while (kn < q && tail > lim) tail -= sv[kn++].first;
    }
    if (kn == 0) {
        U.clear();
        V.clear();
        return 0;
    }
    // not tr: M Y = W  => M = W Y^T:  U' = Qu W_k, V' = Qv Y_k
    // tr:     M^T Y = W => M = Y W^T: U' = Qu Y_k, V' = Qv W_k
    Vec A((size_t)ku * kn), B((size_t)kv * kn);
    for (int c = 0; c < kn; ++c) {
        const int i = sv[c].second;
        const double* wc = W.data() + (int64_t)i * p;
        const double* yc = Y.data() + (int64_t)i * q;
        if (!tr) {
            std::copy(wc, wc + ku, A.begin() + (int64_t)c * ku);
            std::copy(yc, yc + kv, B.begin() + (int64_t)c * kv);
        } else {
            std::copy(yc, yc + ku, A.begin() + (int64_t)c * ku);
            std::copy(wc, wc + kv, B.begin() + (int64_t)c * kv);
        }
    }
    ProfT _g(3);
    // fresh exact-size factors (a resize would keep the m x K capacity of the untruncated sum alive in
    // every block: measured 2x host memory at C5)
    Vec Un((size_t)(m * kn)), Vn((size_t)(n * kn));
    apply_q(fu, A.data(), kn, Un.data());
    apply_q(fv, B.data(), kn, Vn.data());
    U.swap(Un);
    V.swap(Vn);
    return kn;
}

// Best rank-k approximation of a dense m x n block D at eps (Frobenius tail, reading R5): Householder QR
// with column pivoting stopped once the trailing columns hold <= (eps/2)^2 of ||D||_F^2, then the SVD
// truncation of the small r x n factor at the remaining budget -- O(m n r) instead of a full SVD.
int compress_dense(const double* D, int64_t m, int64_t n, double eps, Vec& U, Vec& V) {
    ProfT _p(15);
    QR f;
    f.m = m;
    f.K = (int)n;
    f.W.assign(D, D + m * n);
    const int kmax = (int)std::min<int64_t>(m, n);
    f.tau.assign((size_t)kmax, 0.0);
    std::vector<double> nrm((size_t)n), nrm0((size_t)n);
    std::vector<int> perm((size_t)n);
    double tot = 0.0;
    for (int64_t c = 0; c < n; ++c) {
        double a = 0.0;
        for (int64_t i = 0; i < m; ++i) a += f.W[i + c * m] * f.W[i + c * m];
        nrm[c] = nrm0[c] = a;
        tot += a;
        perm[c] = (int)c;
    }
    if (tot == 0.0) {
        U.clear();
        V.clear();
        return 0;
    }
    const double lim = 0.25 * eps * eps * tot;
    double* Wp = f.W.data();
    int r = 0;
    for (; r < kmax; ++r) {
        double rem = 0.0;
        int piv = r;
        for (int64_t c = r; c < n; ++c) {
            rem += nrm[c];
            if (nrm[c] > nrm[piv]) piv = (int)c;
        }
        if (rem <= lim) break;
        if (piv != r) {
            std::swap_ranges(Wp + (int64_t)piv * m, Wp + (int64_t)(piv + 1) * m, Wp + (int64_t)r * m);
            std::swap(nrm[piv], nrm[r]);
            std::swap(nrm0[piv], nrm0[r]);
            std::swap(perm[piv], perm[r]);
        }
        double* x = Wp + (int64_t)r * m;
        double nn2 = 0.0;
        for (int64_t i = r; i < m; ++i) nn2 += x[i] * x[i];
        const double nv = std::sqrt(nn2);
        if (nv == 0.0) break;
        const double a0 = x[r];
        const double beta = a0 >= 0.0 ? -nv : nv;
        const double sc = 1.0 / (a0 - beta);
        for (int64_t i = r + 1; i < m; ++i) x[i] *= sc;
        const double tj = f.tau[r] = (beta - a0) / beta;
        x[r] = beta;
        reflect(x, r, m, tj, Wp + (int64_t)(r + 1) * m, m, (int)(n - r - 1));
        for (int64_t c = r + 1; c < n; ++c) {   // downdate the trailing norms (recompute when they fade)
            const double w = Wp[r + c * m];
            nrm[c] -= w * w;
            if (nrm[c] <= 1e-10 * nrm0[c]) {
                double a = 0.0;
                for (int64_t i = r + 1; i < m; ++i) a += Wp[i + c * m] * Wp[i + c * m];
                nrm[c] = nrm0[c] = a;
            }
        }
    }
    f.kq = r;
    if (r == 0) {
        U.clear();
        V.clear();
        return 0;
    }
    // R~ = R P^T (r x n): SVD-truncate I_r R~ at the remaining budget (relative to ||R~|| ~ ||D||)
    Vec Ui((size_t)r * r, 0.0), Vt((size_t)(n * r), 0.0);
    for (int i = 0; i < r; ++i) Ui[i + (int64_t)i * r] = 1.0;
    for (int64_t c = 0; c < n; ++c)
        for (int i = 0; i <= std::min<int64_t>(c, r - 1); ++i) Vt[perm[c] + (int64_t)i * n] = Wp[i + c * m];
    const int k = truncate(r, n, r, Ui, Vt, std::sqrt(0.75) * eps);
    if (k == 0) {
        U.clear();
        V.clear();
        return 0;
    }
    Vec Un((size_t)(m * k));
    apply_q(f, Ui.data(), k, Un.data());
    U.swap(Un);
    Vt.resize((size_t)(n * k));
    Vt.shrink_to_fit();
    V.swap(Vt);
    return k;
}

// ============================================================================ H-arithmetic
struct Impl {
    const std::vector<Node>& nodes;
    double eps;
    std::atomic<int64_t> ntr{0}, rin{0}, rout{0};
    std::atomic<bool> singular{false};
    std::mutex mu;
    std::string where;
    int64_t task_min;   // spawn tasks only for blocks with at least this many entries
    // which admissible blocks are accumulated dense: -1 (default) those between two leaf clusters,
    // > 0 those of at most this many entries, 0 none (HM_HLU_ACC_MAX; measured on C2, 8 threads:
    // leaf pairs 8.3 s, <= 80 x 80 entries 10.9 s, none 12.0 s)
    int64_t acc_max = getenv("HM_HLU_ACC_MAX") ? atol(getenv("HM_HLU_ACC_MAX")) : -1;
    bool acc_block(const Mat& A) const {
        if (acc_max < 0) return nodes[A.rn].is_leaf() && nodes[A.cn].is_leaf();
        return A.m * A.n <= acc_max;
    }

    bool big(const Mat& M) const { return M.m * M.n >= task_min; }

    int trunc(Mat& C, int K) {   // C.U (m x K), C.V (n x K) -> truncated rank
        ntr.fetch_add(1, std::memory_order_relaxed);
        rin.fetch_add(K, std::memory_order_relaxed);
        const int k = truncate(C.m, C.n, K, C.U, C.V, eps);
        rout.fetch_add(k, std::memory_order_relaxed);
        return k;
    }

    // ---- C (rows of op(A)) += alpha op(A) B ; B has r columns
    void hmul(const Mat& A, bool tr, const double* B, int64_t ldb, int64_t r, double* C, int64_t ldc, double alpha) {
        if (r <= 0) return;
        if (A.type == T_DENSE) {
            ProfT _p(9);
            if (tr) gemm_tn(A.n, r, A.m, alpha, A.D.data(), A.m, B, ldb, C, ldc);
            else gemm_nn(A.m, r, A.n, alpha, A.D.data(), A.m, B, ldb, C, ldc);
        } else if (A.type == T_LR) {
            if (A.k == 0) return;
            ProfT _p(10);
            Vec t((size_t)A.k * r, 0.0);
            if (tr) {
                gemm_tn(A.k, r, A.m, 1.0, A.U.data(), A.m, B, ldb, t.data(), A.k);
                gemm_nn(A.n, r, A.k, alpha, A.V.data(), A.n, t.data(), A.k, C, ldc);
            } else {
                gemm_tn(A.k, r, A.n, 1.0, A.V.data(), A.n, B, ldb, t.data(), A.k);
                gemm_nn(A.m, r, A.k, alpha, A.U.data(), A.m, t.data(), A.k, C, ldc);
            }
        } else {
            const int64_t m0 = A.ch(0, 0)->m, n0 = A.ch(0, 0)->n;
            const bool par = big(A) && r * (A.m + A.n) >= 4096;
            for (int o = 0; o < 2; ++o) {
#pragma omp task default(shared) firstprivate(o) if (par)
                {
                    if (!tr) {
                        double* Co = C + (o ? m0 : 0);
                        for (int j = 0; j < 2; ++j) hmul(*A.ch(o, j), false, B + (j ? n0 : 0), ldb, r, Co, ldc, alpha);
                    } else {
                        double* Co = C + (o ? n0 : 0);
                        for (int i = 0; i < 2; ++i) hmul(*A.ch(i, o), true, B + (i ? m0 : 0), ldb, r, Co, ldc, alpha);
                    }
                }
            }
#pragma omp taskwait
        }
    }

    // ---- B (T.m x r) <- op(T)^-1 B, T a diagonal H-block holding the packed LU
    void solve(const Mat& T, int kind, double* B, int64_t ldb, int64_t r) {
        if (r <= 0) return;
        if (T.type == T_DENSE) {
            ProfT _p(11);
            trsm_dense(kind, T.D.data(), T.m, B, ldb, r);
            return;
        }
        // independent column groups of a wide right-hand side
        const int64_t cols = 32;
        if (r > cols && T.m * r >= task_min) {
            for (int64_t j0 = 0; j0 < r; j0 += cols) {
#pragma omp task default(shared) firstprivate(j0)
                solve(T, kind, B + j0 * ldb, ldb, std::min<int64_t>(cols, r - j0));
            }
#pragma omp taskwait
            return;
        }
        const int64_t m0 = T.ch(0, 0)->m;
        double *B0 = B, *B1 = B + m0;
        switch (kind) {
        case S_LL:
            solve(*T.ch(0, 0), kind, B0, ldb, r);
            hmul(*T.ch(1, 0), false, B0, ldb, r, B1, ldb, -1.0);
            solve(*T.ch(1, 1), kind, B1, ldb, r);
            break;
        case S_LU:
            solve(*T.ch(1, 1), kind, B1, ldb, r);
            hmul(*T.ch(0, 1), false, B1, ldb, r, B0, ldb, -1.0);
            solve(*T.ch(0, 0), kind, B0, ldb, r);
            break;
        case S_LLT:
            solve(*T.ch(1, 1), kind, B1, ldb, r);
            hmul(*T.ch(1, 0), true, B1, ldb, r, B0, ldb, -1.0);
            solve(*T.ch(0, 0), kind, B0, ldb, r);
            break;
        case S_LUT:
            solve(*T.ch(0, 0), kind, B0, ldb, r);
            hmul(*T.ch(0, 1), true, B0, ldb, r, B1, ldb, -1.0);
            solve(*T.ch(1, 1), kind, B1, ldb, r);
            break;
        }
    }

    // ---- X <- L^-1 X (kind S_LL) or U^-1 X (S_LU), T = (sigma, sigma), X = (sigma, tau)
    void trsm_left(const Mat& T, int kind, Mat& X) {
        if (X.type == T_DENSE) { solve(T, kind, X.D.data(), X.m, X.n); return; }
        if (X.type == T_LR) { solve(T, kind, X.U.data(), X.m, X.k); return; }
        if (T.type != T_SUB) throw std::logic_error("hla: subdivided block over a dense diagonal leaf");
        const bool par = big(X);
        for (int j = 0; j < 2; ++j) {
#pragma omp task default(shared) firstprivate(j) if (par)
            {
                if (kind == S_LL) {
                    trsm_left(*T.ch(0, 0), kind, *X.ch(0, j));
                    mm(*X.ch(1, j), *T.ch(1, 0), *X.ch(0, j), -1.0);
                    trsm_left(*T.ch(1, 1), kind, *X.ch(1, j));
                } else {
                    trsm_left(*T.ch(1, 1), kind, *X.ch(1, j));
                    mm(*X.ch(0, j), *T.ch(0, 1), *X.ch(1, j), -1.0);
                    trsm_left(*T.ch(0, 0), kind, *X.ch(0, j));
                }
            }
        }
#pragma omp taskwait
    }

    // ---- X <- X L^-1 (lower = true) or X U^-1, T = (tau, tau), X = (sigma, tau)
    void trsm_right(const Mat& T, bool lower, Mat& X) {
        const int kind = lower ? S_LLT : S_LUT;   // (X T^-1)^T = T^-T X^T
        if (X.type == T_DENSE) {
            ProfT _p(16);
            Vec Xt = transpose(X.D.data(), X.m, X.n, X.m);
            solve(T, kind, Xt.data(), X.n, X.m);
            for (int64_t j = 0; j < X.n; ++j)
                for (int64_t i = 0; i < X.m; ++i) X.D[i + j * X.m] = Xt[j + i * X.n];
            return;
        }
        if (X.type == T_LR) { solve(T, kind, X.V.data(), X.n, X.k); return; }
        if (T.type != T_SUB) throw std::logic_error("hla: subdivided block over a dense diagonal leaf");
        const bool par = big(X);
        for (int i = 0; i < 2; ++i) {
#pragma omp task default(shared) firstprivate(i) if (par)
            {
                if (!lower) {
                    trsm_right(*T.ch(0, 0), lower, *X.ch(i, 0));
                    mm(*X.ch(i, 1), *X.ch(i, 0), *T.ch(0, 1), -1.0);
                    trsm_right(*T.ch(1, 1), lower, *X.ch(i, 1));
                } else {
                    trsm_right(*T.ch(1, 1), lower, *X.ch(i, 1));
                    mm(*X.ch(i, 0), *X.ch(i, 1), *T.ch(1, 0), -1.0);
                    trsm_right(*T.ch(0, 0), lower, *X.ch(i, 0));
                }
            }
        }
#pragma omp taskwait
    }

    // ---- C += alpha U V^T, U (C.m x k, ldu), V (C.n x k, ldv)
    static thread_local int fan_depth;
    void addlr(Mat& C, const double* U, int64_t ldu, const double* V, int64_t ldv, int k, double alpha) {
        if (k <= 0) return;
        if (C.type == T_SUB && fan_depth == 0) g_prof[14].fetch_add(1);
        struct FD { bool on; FD(bool b) : on(b) { if (on) ++fan_depth; } ~FD() { if (on) --fan_depth; } } fd(C.type == T_SUB);
        if (C.type == T_DENSE) {
            ProfT _p(21);
            gemm_nt(C.m, C.n, k, alpha, U, ldu, V, ldv, C.D.data(), C.m);
        } else if (C.type == T_LR) {
            ProfT _p(4);
            {   // size histogram (diagnostics)
                const int64_t mn = std::max(C.m, C.n);
                int b = mn <= 64 ? 0 : mn <= 128 ? 1 : mn <= 256 ? 2 : mn <= 1024 ? 3 : 4;
                g_hist[b].fetch_add(1, std::memory_order_relaxed);
                g_histk[b].fetch_add(k, std::memory_order_relaxed);
            }
            const int K = C.k + k;
            Vec Un((size_t)(C.m * K)), Vn((size_t)(C.n * K));
            std::copy(C.U.begin(), C.U.begin() + C.m * C.k, Un.begin());
            std::copy(C.V.begin(), C.V.begin() + C.n * C.k, Vn.begin());
            for (int l = 0; l < k; ++l) {
                for (int64_t i = 0; i < C.m; ++i) Un[i + (C.k + l) * C.m] = alpha * U[i + l * ldu];
                for (int64_t j = 0; j < C.n; ++j) Vn[j + (C.k + l) * C.n] = V[j + l * ldv];
            }
            C.U.swap(Un);
            C.V.swap(Vn);
            C.k = trunc(C, K);
        } else {
            const int64_t m0 = C.ch(0, 0)->m, n0 = C.ch(0, 0)->n;
            const bool par = big(C);
            for (int q = 0; q < 4; ++q) {
#pragma omp task default(shared) firstprivate(q) if (par)
                {
                    const int i = q >> 1, j = q & 1;
                    addlr(*C.c[q], U + (i ? m0 : 0), ldu, V + (j ? n0 : 0), ldv, k, alpha);
                }
            }
#pragma omp taskwait
        }
    }

    static Vec identity(int64_t m) {
        Vec I((size_t)(m * m), 0.0);
        for (int64_t i = 0; i < m; ++i) I[i + i * m] = 1.0;
        return I;
    }

    // collapse a subdivided block whose leaves are all low rank into one low-rank block (truncated)
    void agglomerate(Mat& T, Vec& U, Vec& V, int& k) {
        if (T.type == T_DENSE) {   // a dense leaf-pair accumulator: compress it on its own first
            k = dense_to_lr(T.D.data(), T.m, T.n, U, V);
            return;
        }
        if (T.type == T_LR) {
            U = T.U;
            V = T.V;
            k = T.k;
            return;
        }
        const int64_t m0 = T.ch(0, 0)->m, n0 = T.ch(0, 0)->n;
        Vec Uq[4], Vq[4];
        int kq[4], K = 0;
        for (int q = 0; q < 4; ++q) {
            agglomerate(*T.c[q], Uq[q], Vq[q], kq[q]);
            K += kq[q];
        }
        U.assign((size_t)(T.m * K), 0.0);
        V.assign((size_t)(T.n * K), 0.0);
        int o = 0;
        for (int q = 0; q < 4; ++q) {
            const int i = q >> 1, j = q & 1;
            const Mat& Cq = *T.c[q];
            for (int l = 0; l < kq[q]; ++l) {
                std::copy(Uq[q].begin() + l * Cq.m, Uq[q].begin() + (l + 1) * Cq.m, U.begin() + (o + l) * T.m + (i ? m0 : 0));
                std::copy(Vq[q].begin() + l * Cq.n, Vq[q].begin() + (l + 1) * Cq.n, V.begin() + (o + l) * T.n + (j ? n0 : 0));
            }
            o += kq[q];
        }
        ProfT _p(5);
        Mat tmp;
        tmp.m = T.m;
        tmp.n = T.n;
        tmp.U.swap(U);
        tmp.V.swap(V);
        k = trunc(tmp, K);
        U.swap(tmp.U);
        V.swap(tmp.V);
    }

    // a temporary low-rank target with C's subdivision (all leaves rank 0)
    std::unique_ptr<Mat> lr_shape(const Mat& C) {
        auto T = std::make_unique<Mat>();
        T->m = C.m;
        T->n = C.n;
        T->r0 = C.r0;
        T->c0 = C.c0;
        T->rn = C.rn;
        T->cn = C.cn;
        T->type = T_SUB;
        const Node& R = nodes[C.rn];
        const Node& K = nodes[C.cn];
        for (int q = 0; q < 4; ++q) {
            const int i = q >> 1, j = q & 1;
            auto c = std::make_unique<Mat>();
            const Node& ri = nodes[R.child[i]];
            const Node& cj = nodes[K.child[j]];
            c->rn = R.child[i];
            c->cn = K.child[j];
            c->r0 = ri.begin;
            c->c0 = cj.begin;
            c->m = ri.size();
            c->n = cj.size();
            if (acc_block(*c)) {   // accumulate dense (see densify_leaf_pairs)
                c->type = T_DENSE;
                c->D.assign((size_t)(c->m * c->n), 0.0);
            } else {
                c->type = T_LR;
            }
            T->c[q] = std::move(c);
        }
        return T;
    }

    // ---- dense view C (m x n, ldc) += alpha A B, any operand types (a dense target with a block
    // structure below it -- an admissible block accumulated dense -- is split along the operands)
    void mm_dview(double* Cp, int64_t ldc, int64_t m, int64_t n, const Mat& A, const Mat& B, double alpha) {
        if (A.type == T_LR || B.type == T_LR) {
            if (A.type == T_LR && B.type == T_LR) {
                if (A.k == 0 || B.k == 0) return;
                Vec core((size_t)A.k * B.k, 0.0);
                gemm_tn(A.k, B.k, A.n, 1.0, A.V.data(), A.n, B.U.data(), B.m, core.data(), A.k);
                Vec Up((size_t)(A.m * B.k), 0.0);
                gemm_nn(A.m, B.k, A.k, 1.0, A.U.data(), A.m, core.data(), A.k, Up.data(), A.m);
                gemm_nt(m, n, B.k, alpha, Up.data(), A.m, B.V.data(), B.n, Cp, ldc);
            } else if (A.type == T_LR) {
                if (A.k == 0) return;
                Vec T((size_t)(B.n * A.k), 0.0);
                hmul(B, true, A.V.data(), A.n, A.k, T.data(), B.n, 1.0);
                gemm_nt(m, n, A.k, alpha, A.U.data(), A.m, T.data(), B.n, Cp, ldc);
            } else {
                if (B.k == 0) return;
                Vec Z((size_t)(A.m * B.k), 0.0);
                hmul(A, false, B.U.data(), B.m, B.k, Z.data(), A.m, 1.0);
                gemm_nt(m, n, B.k, alpha, Z.data(), A.m, B.V.data(), B.n, Cp, ldc);
            }
            return;
        }
        if (A.type == T_DENSE && B.type == T_DENSE) {
            gemm_nn(m, n, A.n, alpha, A.D.data(), A.m, B.D.data(), B.m, Cp, ldc);
        } else if (A.type == T_SUB && B.type == T_DENSE) {
            hmul(A, false, B.D.data(), B.m, B.n, Cp, ldc, alpha);
        } else if (A.type == T_DENSE && B.type == T_SUB) {
            Vec At = transpose(A.D.data(), A.m, A.n, A.m);   // sigma x rho
            Vec Z((size_t)(B.n * A.m), 0.0);                 // B^T A^T = (A B)^T
            hmul(B, true, At.data(), A.n, A.m, Z.data(), B.n, 1.0);
            for (int64_t j = 0; j < n; ++j)
                for (int64_t i = 0; i < m; ++i) Cp[i + j * ldc] += alpha * Z[j + i * B.n];
        } else {   // both subdivided: quadrants of the view
            const int64_t m0 = A.ch(0, 0)->m, n0 = B.ch(0, 0)->n;
            for (int q = 0; q < 4; ++q) {
                const int i = q >> 1, j = q & 1;
                double* Cq = Cp + (i ? m0 : 0) + (j ? n0 : 0) * ldc;
                const int64_t mq = i ? m - m0 : m0, nq = j ? n - n0 : n0;
                for (int l = 0; l < 2; ++l) mm_dview(Cq, ldc, mq, nq, *A.ch(i, l), *B.ch(l, j), alpha);
            }
        }
    }

    // an admissible block accumulated dense, as a temporary low-rank operand (for products whose
    // target is not dense: their update then has the block's rank, not its dimension)
    std::unique_ptr<Mat> acc_as_lr(const Mat& A) {
        auto T = std::make_unique<Mat>();
        T->m = A.m;
        T->n = A.n;
        T->r0 = A.r0;
        T->c0 = A.c0;
        T->rn = A.rn;
        T->cn = A.cn;
        T->type = T_LR;
        T->k = dense_to_lr(A.D.data(), A.m, A.n, T->U, T->V);
        return T;
    }

    // ---- C += alpha A B
    void mm(Mat& C, const Mat& A, const Mat& B, double alpha) {
        // (only when the other operand is not low rank: then the update has that operand's rank anyway)
        const bool ca = A.acc && A.type == T_DENSE && B.type != T_LR;
        const bool cb = B.acc && B.type == T_DENSE && A.type != T_LR;
        if (C.type != T_DENSE && (ca || cb)) {
            std::unique_ptr<Mat> a2, b2;
            if (ca) a2 = acc_as_lr(A);
            if (cb) b2 = acc_as_lr(B);
            mm(C, a2 ? *a2 : A, b2 ? *b2 : B, alpha);
            return;
        }
        if (A.type == T_LR || B.type == T_LR) {
            if (A.type == T_LR && B.type == T_LR) {
                if (A.k == 0 || B.k == 0) return;
                Vec core((size_t)A.k * B.k, 0.0);   // Va^T Ub
                gemm_tn(A.k, B.k, A.n, 1.0, A.V.data(), A.n, B.U.data(), B.m, core.data(), A.k);
                if (B.k <= A.k) {
                    Vec Up((size_t)(A.m * B.k), 0.0);
                    gemm_nn(A.m, B.k, A.k, 1.0, A.U.data(), A.m, core.data(), A.k, Up.data(), A.m);
                    addlr(C, Up.data(), A.m, B.V.data(), B.n, B.k, alpha);
                } else {
                    Vec Vp((size_t)(B.n * A.k), 0.0);   // Vb core^T
                    gemm_nt(B.n, A.k, B.k, 1.0, B.V.data(), B.n, core.data(), A.k, Vp.data(), B.n);
                    addlr(C, A.U.data(), A.m, Vp.data(), B.n, A.k, alpha);
                }
            } else if (A.type == T_LR) {
                if (A.k == 0) return;
                Vec T((size_t)(B.n * A.k), 0.0);   // B^T Va
                hmul(B, true, A.V.data(), A.n, A.k, T.data(), B.n, 1.0);
                addlr(C, A.U.data(), A.m, T.data(), B.n, A.k, alpha);
            } else {
                if (B.k == 0) return;
                Vec Z((size_t)(A.m * B.k), 0.0);   // A Ub
                hmul(A, false, B.U.data(), B.m, B.k, Z.data(), A.m, 1.0);
                addlr(C, Z.data(), A.m, B.V.data(), B.n, B.k, alpha);
            }
            return;
        }
        // A, B dense or subdivided
        if (C.type == T_DENSE) {
            ProfT _p(13);
            mm_dview(C.D.data(), C.m, C.m, C.n, A, B, alpha);
            return;
        }
        if (C.type == T_LR) {
            if (A.type == T_DENSE && B.type == T_DENSE) {
                ProfT _p(17);
                const int64_t rho = A.m, sig = A.n, tau = B.n;
                if (sig <= rho && sig <= tau) {
                    Vec Bt = transpose(B.D.data(), B.m, B.n, B.m);   // tau x sigma
                    addlr(C, A.D.data(), rho, Bt.data(), tau, (int)sig, alpha);
                } else {
                    Vec P((size_t)(rho * tau), 0.0);
                    gemm_nn(rho, tau, sig, 1.0, A.D.data(), rho, B.D.data(), B.m, P.data(), rho);
                    if (rho <= tau) {
                        Vec Pt = transpose(P.data(), rho, tau, rho);
                        Vec I = identity(rho);
                        addlr(C, I.data(), rho, Pt.data(), tau, (int)rho, alpha);
                    } else {
                        Vec I = identity(tau);
                        addlr(C, P.data(), rho, I.data(), tau, (int)tau, alpha);
                    }
                }
            } else if (A.type == T_DENSE && B.type == T_SUB) {
                ProfT _p(18);
                Vec At = transpose(A.D.data(), A.m, A.n, A.m);
                Vec Z((size_t)(B.n * A.m), 0.0);
                hmul(B, true, At.data(), A.n, A.m, Z.data(), B.n, 1.0);
                Vec I = identity(A.m);
                addlr(C, I.data(), A.m, Z.data(), B.n, (int)A.m, alpha);
            } else if (A.type == T_SUB && B.type == T_DENSE) {
                ProfT _p(19);
                Vec Z((size_t)(A.m * B.n), 0.0);
                hmul(A, false, B.D.data(), B.m, B.n, Z.data(), A.m, 1.0);
                Vec I = identity(B.n);
                addlr(C, Z.data(), A.m, I.data(), B.n, (int)B.n, alpha);
            } else {
                // both subdivided: form the product in C's subdivision, collapse it, add it
                ProfT _p(20);
                auto T = lr_shape(C);
                const bool par = big(C);
                for (int q = 0; q < 4; ++q) {
#pragma omp task default(shared) firstprivate(q) if (par)
                    {
                        const int i = q >> 1, j = q & 1;
                        for (int l = 0; l < 2; ++l) mm(*T->c[q], *A.ch(i, l), *B.ch(l, j), alpha);
                    }
                }
#pragma omp taskwait
                Vec U, V;
                int k = 0;
                agglomerate(*T, U, V, k);
                addlr(C, U.data(), C.m, V.data(), C.n, k, 1.0);
            }
            return;
        }
        // C subdivided
        if (A.type == T_SUB && B.type == T_SUB) {
            const bool par = big(C);
            for (int q = 0; q < 4; ++q) {
#pragma omp task default(shared) firstprivate(q) if (par)
                {
                    const int i = q >> 1, j = q & 1;
                    for (int l = 0; l < 2; ++l) mm(*C.c[q], *A.ch(i, l), *B.ch(l, j), alpha);
                }
            }
#pragma omp taskwait
        } else if (A.type == T_DENSE && B.type == T_DENSE) {
            Vec Bt = transpose(B.D.data(), B.m, B.n, B.m);
            addlr(C, A.D.data(), A.m, Bt.data(), B.n, (int)A.n, alpha);
        } else {
            throw std::logic_error("hla: subdivided target of a dense and a subdivided factor");
        }
    }

    void lu(Mat& A) {
        if (singular.load(std::memory_order_relaxed)) return;
        if (A.type == T_DENSE) {
            ProfT _p(12);
            if (!lu_dense(A.D.data(), A.m)) {
                std::lock_guard<std::mutex> g(mu);
                if (!singular) where = "rows [" + std::to_string(A.r0) + ", " + std::to_string(A.r0 + A.m) + ")";
                singular = true;
            }
            return;
        }
        if (A.type != T_SUB) throw std::logic_error("hla: low-rank diagonal block");
        lu(*A.ch(0, 0));
#pragma omp task default(shared)
        trsm_left(*A.ch(0, 0), S_LL, *A.ch(0, 1));
#pragma omp task default(shared)
        trsm_right(*A.ch(0, 0), false, *A.ch(1, 0));
#pragma omp taskwait
        mm(*A.ch(1, 1), *A.ch(1, 0), *A.ch(0, 1), -1.0);
        lu(*A.ch(1, 1));
    }

    static void negate(Mat& X) {
        if (X.type == T_DENSE) for (double& v : X.D) v = -v;
        else if (X.type == T_LR) for (double& v : X.U) v = -v;
        else for (auto& c : X.c) negate(*c);
    }

    void form(Mat& A, int cut) {
        if (A.type == T_DENSE) {
            ProfT _p(22);
            invert_packed(A.D.data(), A.m);
            return;
        }
        const int level = nodes[A.rn].level;
        Mat &A00 = *A.ch(0, 0), &A01 = *A.ch(0, 1), &A10 = *A.ch(1, 0), &A11 = *A.ch(1, 1);
        if (level < cut) {   // W^L_t = L21 L11^-1, W^U_t = U12 U22^-1
#pragma omp task default(shared)
            trsm_right(A00, true, A10);
#pragma omp task default(shared)
            trsm_right(A11, false, A01);
#pragma omp taskwait
        } else {             // (L^-1)21 = -L22^-1 L21 L11^-1, (U^-1)12 = -U11^-1 U12 U22^-1
#pragma omp task default(shared)
            {
                trsm_right(A00, true, A10);
                trsm_left(A11, S_LL, A10);
                negate(A10);
            }
#pragma omp task default(shared)
            {
                trsm_right(A11, false, A01);
                trsm_left(A00, S_LU, A01);
                negate(A01);
            }
#pragma omp taskwait
        }
#pragma omp task default(shared)
        form(A00, cut);
#pragma omp task default(shared)
        form(A11, cut);
#pragma omp taskwait
    }

    // admissible blocks between two leaf clusters: dense while the factorisation runs (R33:
    // most updates land on these small blocks; as dense targets they cost a GEMM each instead of a
    // QR + SVD truncation), compressed once at the end at eps -- the same or a smaller error than
    // truncating after every update
    void densify_leaf_pairs(Mat& A) {
        if (A.type == T_SUB) {
            for (auto& c : A.c) densify_leaf_pairs(*c);
            return;
        }
        if (A.type != T_LR || !acc_block(A)) return;
        A.D.assign((size_t)(A.m * A.n), 0.0);
        gemm_nt(A.m, A.n, A.k, 1.0, A.U.data(), A.m, A.V.data(), A.n, A.D.data(), A.m);
        A.U.clear();
        A.V.clear();
        A.U.shrink_to_fit();
        A.V.shrink_to_fit();
        A.k = 0;
        A.type = T_DENSE;
        A.acc = true;
    }
    void compress_acc(Mat& A) {
        if (A.type == T_SUB) {
            const bool par = big(A);
            for (int q = 0; q < 4; ++q) {
#pragma omp task default(shared) firstprivate(q) if (par)
                compress_acc(*A.c[q]);
            }
#pragma omp taskwait
            return;
        }
        if (!A.acc) return;
        A.k = dense_to_lr(A.D.data(), A.m, A.n, A.U, A.V);
        A.D.clear();
        A.D.shrink_to_fit();
        A.type = T_LR;
        A.acc = false;
    }
    int dense_to_lr(const double* D, int64_t m, int64_t n, Vec& U, Vec& V) {
        ntr.fetch_add(1, std::memory_order_relaxed);
        rin.fetch_add(std::min(m, n), std::memory_order_relaxed);
        const int k = compress_dense(D, m, n, eps, U, V);
        rout.fetch_add(k, std::memory_order_relaxed);
        return k;
    }

    void normalize(Mat& A) {
        if (A.type == T_SUB) { for (auto& c : A.c) normalize(*c); return; }
        if (A.type != T_DENSE) return;
        if (nodes[A.rn].is_leaf() || nodes[A.cn].is_leaf()) return;   // a genuine near-field leaf
        // admissible block stored dense (rank cap reached in F): low-rank form, exact up to eps
        A.k = dense_to_lr(A.D.data(), A.m, A.n, A.U, A.V);
        A.D.clear();
        A.D.shrink_to_fit();
        A.type = T_LR;
    }
};

thread_local int Impl::fan_depth = 0;

// ============================================================================ HFactor
namespace {
struct BuildCtx {
    const std::vector<Node>& nodes;
    std::map<std::pair<int, int>, int> leaf_id;
    std::vector<Mat*>& by_block;
};
std::unique_ptr<Mat> build(BuildCtx& b, int rn, int cn) {
    auto M = std::make_unique<Mat>();
    const Node& R = b.nodes[rn];
    const Node& C = b.nodes[cn];
    M->rn = rn;
    M->cn = cn;
    M->r0 = R.begin;
    M->c0 = C.begin;
    M->m = R.size();
    M->n = C.size();
    auto it = b.leaf_id.find({rn, cn});
    if (it != b.leaf_id.end()) {
        M->type = T_DENSE;
        b.by_block[it->second] = M.get();
        return M;
    }
    if (R.is_leaf() || C.is_leaf()) throw std::logic_error("hla: block partition does not cover a leaf pair");
    M->type = T_SUB;
    for (int q = 0; q < 4; ++q) M->c[q] = build(b, R.child[q >> 1], C.child[q & 1]);
    return M;
}
int64_t env_task_min() {
    const char* e = getenv("HM_HLU_TASK_MIN");
    const long v = e ? atol(e) : 0;
    return v > 0 ? v : 1 << 14;
}
}  // namespace

HFactor::HFactor(const std::vector<Node>& nodes, const std::vector<std::pair<int, int>>& leaf_blocks)
    : nodes_(nodes) {
    by_block_.assign(leaf_blocks.size(), nullptr);
    BuildCtx b{nodes, {}, by_block_};
    for (size_t q = 0; q < leaf_blocks.size(); ++q) b.leaf_id[leaf_blocks[q]] = (int)q;
    root_ = build(b, 0, 0);
    for (Mat* p : by_block_)
        if (!p) throw std::logic_error("hla: a partition block is not reachable from the root pair");
}

HFactor::~HFactor() = default;

int HFactor::threads() const { return omp_get_max_threads(); }

void parallel_for(int64_t n, const std::function<void(int64_t)>& f) {
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < n; ++i) f(i);
}

void HFactor::for_each_leaf(const std::function<void(int, Mat&)>& f) {
    const int64_t nb = (int64_t)by_block_.size();
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t b = 0; b < nb; ++b) f((int)b, *by_block_[b]);
}

template <class F>
static void run_tasks(Impl& I, F&& f) {
#pragma omp parallel
#pragma omp single
    f(I);
}

void HFactor::normalize(double eps) {
    Impl I{nodes_, eps};
    I.task_min = env_task_min();
    run_tasks(I, [&](Impl& im) { im.normalize(*root_); });
    stats_.truncations += I.ntr;
    stats_.trunc_rank_in += I.rin;
    stats_.trunc_rank_out += I.rout;
}

void HFactor::factor(double eps) {
    const auto t0 = std::chrono::steady_clock::now();
    Impl I{nodes_, eps};
    I.task_min = env_task_min();
    if (I.acc_max != 0) run_tasks(I, [&](Impl& im) { im.densify_leaf_pairs(*root_); });
    run_tasks(I, [&](Impl& im) { im.lu(*root_); });
    singular_ = I.singular;
    singular_where_ = I.where;
    stats_.truncations += I.ntr;
    stats_.trunc_rank_in += I.rin;
    stats_.trunc_rank_out += I.rout;
    stats_.seconds_lu = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void HFactor::solve_form(int cut, double eps) {
    const auto t0 = std::chrono::steady_clock::now();
    Impl I{nodes_, eps};
    I.task_min = env_task_min();
    run_tasks(I, [&](Impl& im) {
        im.form(*root_, cut);
        im.compress_acc(*root_);
    });
    stats_.truncations += I.ntr;
    stats_.trunc_rank_in += I.rin;
    stats_.trunc_rank_out += I.rout;
    stats_.seconds_form = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

static void visit_rec(const Mat& A, int side, int node, const std::function<void(const LeafView&)>& f) {
    if (A.type != T_SUB) {
        f(LeafView{&A, side, node});
        return;
    }
    if (side == 0) {   // a diagonal block at tree node A.rn
        visit_rec(*A.ch(0, 0), 0, -1, f);
        visit_rec(*A.ch(1, 0), 1, A.rn, f);
        visit_rec(*A.ch(0, 1), 2, A.rn, f);
        visit_rec(*A.ch(1, 1), 0, -1, f);
    } else {
        for (int q = 0; q < 4; ++q) visit_rec(*A.c[q], side, node, f);
    }
}

void HFactor::visit(const std::function<void(const LeafView&)>& f) const { visit_rec(*root_, 0, -1, f); }

}  // namespace hla
}  // namespace hm
