// Dense fp64 kernels for the one-time factorisation of C = I - Lambda F (SURVEY.md §8(a) rows
// s4-s6; timed separately from the hot path):
//   expand_C      -- C in dense form from the H-format F (row-scale by Lambda, +I)
//   dgemm         -- C = beta C + alpha op(A) op(B) on the FP64 tensor pipe (mma.sync m8n8k4
//                    f64 -> SASS DMMA; sm_100a has no tcgen05 f64 kind), with optional
//                    lower-unit / upper triangular masking of an operand
//   leaf_lu_inv   -- dense LU without pivoting of a <=64 diagonal block + both triangular inverses
//   cpaca_batch   -- truncation of dense factor blocks to eps_LU by cross approximation with
//                    full pivoting (the paper's ACA variant) with the exact
//                    Frobenius residual as stop test (eq:erel)
#include <cstdint>

#include "hm_internal.h"

namespace hm {
namespace {

// ---------------------------------------------------------------- DMMA GEMM (64x64x16 tiles)
constexpr int BM = 64, BN = 64, BK = 16, PADM = 4;

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

template <int TRIA, int TRIB>
__device__ __forceinline__ double mask(double v, int64_t r, int64_t c, bool isA) {
    const int tri = isA ? TRIA : TRIB;
    if (tri == 1) return c < r ? v : (c == r ? 1.0 : 0.0);  // lower, unit diagonal
    if (tri == 2) return c >= r ? v : 0.0;                   // upper incl. diagonal
    return v;
}

template <int TRIA, int TRIB>
__global__ void __launch_bounds__(128)
dgemm_kernel(int64_t M, int64_t N, int64_t K, double alpha, const double* __restrict__ A, int64_t lda,
             const double* __restrict__ B, int64_t ldb, double beta, double* __restrict__ C, int64_t ldc) {
    __shared__ double As[BK][BM + PADM];
    __shared__ double Bs[BK][BN + PADM];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp >> 1, wn = warp & 1;
    const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
    // K range with structural zeros of triangular operands skipped
    int64_t kbeg = 0, kend = K;
    if (TRIA == 1) kend = min(kend, m0 + BM);
    if (TRIA == 2) kbeg = max(kbeg, m0);
    if (TRIB == 1) kbeg = max(kbeg, n0);
    if (TRIB == 2) kend = min(kend, n0 + BN);
    kbeg = (kbeg / BK) * BK;
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    double ra[8], rb[8];
    auto load = [&](int64_t k0) {
#pragma unroll
        for (int p = 0; p < 8; ++p) {
            const int e = tid + p * 128;
            const int row = e >> 4, kk = e & 15;
            const int64_t gi = m0 + row, gk = k0 + kk;
            double v = 0.0;
            if (gi < M && gk < K) v = mask<TRIA, TRIB>(A[gi * lda + gk], gi, gk, true);
            ra[p] = v;
            const int kb = e >> 6, col = e & 63;
            const int64_t gk2 = k0 + kb, gj = n0 + col;
            double w = 0.0;
            if (gk2 < K && gj < N) w = mask<TRIA, TRIB>(B[gk2 * ldb + gj], gk2, gj, false);
            rb[p] = w;
        }
    };
    auto store = [&]() {
#pragma unroll
        for (int p = 0; p < 8; ++p) {
            const int e = tid + p * 128;
            As[e & 15][e >> 4] = ra[p];
            Bs[e >> 6][e & 63] = rb[p];
        }
    };
    if (kbeg < kend) {
        load(kbeg);
        for (int64_t k0 = kbeg; k0 < kend; k0 += BK) {
            __syncthreads();
            store();
            __syncthreads();
            if (k0 + BK < kend) load(k0 + BK);
#pragma unroll
            for (int ks = 0; ks < BK; ks += 4) {
                const int kk = ks + (lane & 3);
                double a[4], b[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    a[q] = As[kk][wm * 32 + q * 8 + (lane >> 2)];
                    b[q] = Bs[kk][wn * 32 + q * 8 + (lane >> 2)];
                }
#pragma unroll
                for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                    for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
            }
        }
    }
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t r = m0 + wm * 32 + mi * 8 + (lane >> 2);
                const int64_t c = n0 + wn * 32 + ni * 8 + 2 * (lane & 3) + h;
                if (r < M && c < N) {
                    double v = alpha * acc[mi][ni][h];
                    if (beta != 0.0) v += beta * C[r * ldc + c];
                    C[r * ldc + c] = v;
                }
            }
}

// ---------------------------------------------------------------- leaf LU + inverses (n <= 64)
constexpr int LS = 65;
__global__ void __launch_bounds__(256)
leaf_lu_inv_kernel(double* __restrict__ M, double* __restrict__ Minv, int64_t ld, int n, int32_t* err) {
    extern __shared__ double sm[];
    double* S = sm;
    double* X = sm + 64 * LS;
    double* Y = X + 64 * LS;
    __shared__ double s_max[8];
    const int tid = threadIdx.x;
    double mx = 0.0;
    for (int e = tid; e < n * n; e += blockDim.x) {
        const int i = e / n, j = e % n;
        const double v = M[(int64_t)i * ld + j];
        S[i * LS + j] = v;
        mx = fmax(mx, fabs(v));
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((tid & 31) == 0) s_max[tid >> 5] = mx;
    __syncthreads();
    mx = s_max[0];
    for (int q = 1; q < 8; ++q) mx = fmax(mx, s_max[q]);
    const double thr = 1e-14 * mx;
    for (int k = 0; k < n; ++k) {
        const double piv = S[k * LS + k];
        if (!(fabs(piv) > thr) && tid == 0 && err[0] == 0) err[0] = 2;
        for (int i = k + 1 + tid; i < n; i += blockDim.x) S[i * LS + k] /= piv;
        __syncthreads();
        const int w = n - k - 1;
        for (int e = tid; e < w * w; e += blockDim.x) {
            const int i = k + 1 + e / w, j = k + 1 + e % w;
            S[i * LS + j] -= S[i * LS + k] * S[k * LS + j];
        }
        __syncthreads();
    }
    for (int e = tid; e < n * n; e += blockDim.x) {
        const int i = e / n, j = e % n;
        M[(int64_t)i * ld + j] = S[i * LS + j];
    }
    if (tid < n) {  // column j of L^-1 (unit lower)
        const int j = tid;
        for (int i = 0; i < j; ++i) X[i * LS + j] = 0.0;
        X[j * LS + j] = 1.0;
        for (int i = j + 1; i < n; ++i) {
            double s = 0.0;
            for (int kk = j; kk < i; ++kk) s += S[i * LS + kk] * X[kk * LS + j];
            X[i * LS + j] = -s;
        }
    } else if (tid >= 64 && tid < 64 + n) {  // column j of U^-1 (upper)
        const int j = tid - 64;
        Y[j * LS + j] = 1.0 / S[j * LS + j];
        for (int i = j - 1; i >= 0; --i) {
            double s = 0.0;
            for (int kk = i + 1; kk <= j; ++kk) s += S[i * LS + kk] * Y[kk * LS + j];
            Y[i * LS + j] = -s / S[i * LS + i];
        }
    }
    __syncthreads();
    for (int e = tid; e < n * n; e += blockDim.x) {
        const int i = e / n, j = e % n;
        Minv[(int64_t)i * ld + j] = i > j ? X[i * LS + j] : Y[i * LS + j];
    }
}

__global__ void copy2d_kernel(const double* __restrict__ src, int64_t lds, double* __restrict__ dst, int64_t ldd,
                              int64_t rows, int64_t cols) {
    const int64_t tot = rows * cols;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / cols, j = e % cols;
        dst[i * ldd + j] = src[i * lds + j];
    }
}

__global__ void extract_tri_kernel(const double* __restrict__ Minv, int64_t ld, int64_t r0, int64_t m, int mode,
                                   double* __restrict__ dst) {
    for (int64_t e = threadIdx.x; e < m * m; e += blockDim.x) {
        const int64_t i = e / m, j = e % m;
        const double v = Minv[(r0 + i) * ld + r0 + j];
        dst[e] = mode == 1 ? (j < i ? v : (j == i ? 1.0 : 0.0)) : (j >= i ? v : 0.0);
    }
}

__global__ void expand_kernel(const int64_t* __restrict__ tasks, const double* __restrict__ arena,
                              const double* __restrict__ lam, double* __restrict__ M, int64_t ld) {
    const int64_t* t = tasks + 10 * blockIdx.x;
    const int64_t a_off = t[0], a_ld = t[1], v_off = t[2], v_ld = t[3], r0 = t[4], m = t[5], c0 = t[6], nc = t[7],
                  k = t[8];
    for (int64_t e = threadIdx.x; e < m * nc; e += blockDim.x) {
        const int64_t i = e / nc, j = e % nc;
        double v;
        if (v_off < 0) {
            v = arena[a_off + j * a_ld + i];
        } else {
            v = 0.0;
            for (int64_t l = 0; l < k; ++l) v += arena[a_off + l * a_ld + i] * arena[v_off + j * v_ld + l];
        }
        M[(r0 + i) * ld + c0 + j] = -lam[r0 + i] * v;
    }
}

__global__ void add_identity_kernel(double* M, int64_t ld, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) M[i * ld + i] += 1.0;
}

// ---------------------------------------------------------------- cross approximation with full pivoting
constexpr int kCT = 256;
struct AM {
    double v;
    int64_t i;
};
__device__ __forceinline__ AM amax(AM x, AM y) {
    if (y.v > x.v) return y;
    if (y.v == x.v && y.i < x.i) return y;
    return x;
}
__device__ void cta_reduce(double& s, AM& a, double* sd, AM* sa) {
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        AM b{__shfl_xor_sync(0xffffffffu, a.v, o), __shfl_xor_sync(0xffffffffu, a.i, o)};
        a = amax(a, b);
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) { sd[threadIdx.x >> 5] = s; sa[threadIdx.x >> 5] = a; }
    __syncthreads();
    s = sd[0];
    a = sa[0];
    for (int q = 1; q < kCT / 32; ++q) { s += sd[q]; a = amax(a, sa[q]); }
}

__global__ void __launch_bounds__(kCT)
cpaca_kernel(double* __restrict__ T, int64_t ldt, const int64_t* __restrict__ blk, const int32_t* __restrict__ kcap_arr,
             double eps, double* __restrict__ fac, int32_t* __restrict__ rank_out) {
    __shared__ double sd[kCT / 32];
    __shared__ AM sa[kCT / 32];
    const int64_t* bb = blk + 7 * blockIdx.x;
    const int64_t i0 = bb[0], m = bb[1], j0 = bb[2], n = bb[3];
    ldt = bb[6] > 0 ? bb[6] : ldt;   // per-block row stride (packed blocks) or the batch's
    double* U = fac + bb[4];
    double* V = fac + bb[5];
    double* X = T + i0 * ldt + j0;
    const int kcap = kcap_arr[blockIdx.x];
    const int64_t tot = m * n;
    double s = 0.0;
    AM a{-1.0, INT64_MAX};
    for (int64_t e = threadIdx.x; e < tot; e += kCT) {
        const double v = X[(e / n) * ldt + e % n];
        s += v * v;
        a = amax(a, AM{fabs(v), e});
    }
    cta_reduce(s, a, sd, sa);
    const double thr = eps * eps * s;
    double R2 = s;
    int k = 0;
    while (R2 > thr) {
        if (k == kcap) {  // not compressible within the cap: restore X = R + U V^T, store dense
            __syncthreads();
            for (int64_t e = threadIdx.x; e < tot; e += kCT) {
                const int64_t i = e / n, j = e % n;
                double v = X[i * ldt + j];
                for (int l = 0; l < k; ++l) v += U[(int64_t)l * m + i] * V[(int64_t)l * n + j];
                X[i * ldt + j] = v;
            }
            if (threadIdx.x == 0) rank_out[blockIdx.x] = -1;
            return;
        }
        const int64_t is = a.i / n, js = a.i % n;
        const double delta = X[is * ldt + js];
        double* u = U + (int64_t)k * m;
        double* v = V + (int64_t)k * n;
        for (int64_t i = threadIdx.x; i < m; i += kCT) u[i] = X[i * ldt + js];
        for (int64_t j = threadIdx.x; j < n; j += kCT) v[j] = X[is * ldt + j] / delta;
        __syncthreads();
        s = 0.0;
        a = AM{-1.0, INT64_MAX};
        for (int64_t e = threadIdx.x; e < tot; e += kCT) {
            const int64_t i = e / n, j = e % n;
            const double r = X[i * ldt + j] - u[i] * v[j];
            X[i * ldt + j] = r;
            s += r * r;
            a = amax(a, AM{fabs(r), e});
        }
        cta_reduce(s, a, sd, sa);
        R2 = s;
        ++k;
    }
    if (threadIdx.x == 0) rank_out[blockIdx.x] = k;
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

namespace k {

void dgemm(int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda, int triA, const double* B,
           int64_t ldb, int triB, double beta, double* C, int64_t ldc, cudaStream_t s) {
    if (M <= 0 || N <= 0) return;
    dim3 grid(nblk(N, BN), nblk(M, BM));
#define HM_GEMM(TA, TB) dgemm_kernel<TA, TB><<<grid, 128, 0, s>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc)
    if (triA == 0 && triB == 0) HM_GEMM(0, 0);
    else if (triA == 1 && triB == 0) HM_GEMM(1, 0);
    else if (triA == 2 && triB == 0) HM_GEMM(2, 0);
    else if (triA == 0 && triB == 1) HM_GEMM(0, 1);
    else if (triA == 0 && triB == 2) HM_GEMM(0, 2);
    else throw Error(HM_ERR_INVALID_ARG, "dgemm: unsupported triangular combination");
#undef HM_GEMM
    HM_CUDA(cudaGetLastError());
    debug_sync(s, "dgemm");
}

void leaf_lu_inv(double* M, double* Minv, int64_t ld, int n, int32_t* err, cudaStream_t s) {
    const size_t smem = 3 * 64 * LS * sizeof(double);
    static bool attr = false;
    if (!attr) {
        HM_CUDA(cudaFuncSetAttribute(leaf_lu_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    leaf_lu_inv_kernel<<<1, 256, smem, s>>>(M, Minv, ld, n, err);
    HM_CUDA(cudaGetLastError());
    debug_sync(s, "leaf_lu_inv");
}

void copy2d(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows, int64_t cols, cudaStream_t s) {
    if (rows <= 0 || cols <= 0) return;
    const int64_t tot = rows * cols;
    const unsigned g = (unsigned)std::min<int64_t>((tot + 255) / 256, 148 * 16);
    copy2d_kernel<<<g, 256, 0, s>>>(src, lds, dst, ldd, rows, cols);
    HM_CUDA(cudaGetLastError());
    debug_sync(s, "copy2d");
}

void extract_tri(const double* Minv, int64_t ld, int64_t r0, int64_t m, int mode, double* dst, cudaStream_t s) {
    extract_tri_kernel<<<1, 256, 0, s>>>(Minv, ld, r0, m, mode, dst);
    HM_CUDA(cudaGetLastError());
}

void expand_C(const int64_t* tasks, int nt, const double* arena, const double* lam, double* M, int64_t ld,
              cudaStream_t s) {
    if (nt == 0) return;
    expand_kernel<<<nt, 256, 0, s>>>(tasks, arena, lam, M, ld);
    HM_CUDA(cudaGetLastError());
    debug_sync(s, "expand_C");
}

void add_identity(double* M, int64_t ld, int64_t n, cudaStream_t s) {
    add_identity_kernel<<<nblk(n, 256), 256, 0, s>>>(M, ld, n);
    HM_CUDA(cudaGetLastError());
}

void cpaca_batch(double* T, int64_t ldt, const int64_t* blk, const int32_t* kcap, int nb, double eps, double* fac,
                 int32_t* rank_out, cudaStream_t s) {
    if (nb == 0) return;
    cpaca_kernel<<<nb, kCT, 0, s>>>(T, ldt, blk, kcap, eps, fac, rank_out);
    HM_CUDA(cudaGetLastError());
    debug_sync(s, "cpaca");
}

}  // namespace k
}  // namespace hm
