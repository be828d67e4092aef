// Recompression of ACA factor pairs (the ACA output "may be further postprocessed (or
// truncated)"; reading R32).  One CTA per low-rank block U V^T
// (U m x k, V n x k, both column-major in place, k <= 64), best rank-k' truncation at the Frobenius
// tolerance eps (reading A5):
//
//   G_U = U^T U = W diag(lam) W^T              (Gram matrix; Jacobi eigen-decomposition)
//   B   = diag(sqrt lam) W^T                    (U = Q_U B with Q_U = U W diag(lam^-1/2) orthonormal)
//   N   = B (V^T V) B^T = Xe diag(s^2) Xe^T     (N = M M^T for the core M = B V^T Q_V; Jacobi eigen)
//   k'  = smallest k' with sqrt(sum_{i >= k'} s_i^2) <= eps sqrt(sum s_i^2)    (s descending)
//   U'  = U W diag(lam^-1/2) Xe[:, :k'],  V' = V B^T Xe[:, :k']
//
// so U' V'^T = Q_U Xe_k Xe_k^T Q_U^T U V^T, the projection of U V^T onto its top k' left singular
// vectors (Eckart-Young).  The oracle (oracle/aca.py: recompress) takes the QR + SVD route; both
// give the same truncation up to rounding.  Directions of U with lam <= 1e-26 lam_max (relative
// singular value below ~1e-13) are dropped.  Setup only, not on the hot path.
#include <cstdint>

#include "hm_internal.h"

namespace hm {
namespace {

constexpr int kRThreads = 256;
constexpr int kRMax = 64;            // rank cap (hm_aca_params.k_max <= 64)
constexpr int kRRows = 32;           // rows per streamed chunk

struct RSmem {
    double A[kRMax * kRMax];         // matrix being diagonalised (row-major, stride kRMax)
    double W[kRMax * kRMax];         // eigenvectors of G_U (columns)
    double Xe[kRMax * kRMax];        // eigenvectors of N (columns)
    double T[kRMax * kRMax];         // scratch / transforms
    double chunk[kRRows * kRMax];
    double lam[kRMax], s2[kRMax];
    double rc[kRMax / 2], rs[kRMax / 2];
    int order[kRMax];
    double red[kRThreads / 32];
    int kk_new;
};

// G = F^T F for F (rows x k, column-major, ld = rows), fixed summation order
__device__ void gram(RSmem& S, const double* F, int64_t rows, int k) {
    double acc[(kRMax * kRMax) / kRThreads];
    constexpr int kPer = (kRMax * kRMax) / kRThreads;
#pragma unroll
    for (int j = 0; j < kPer; ++j) acc[j] = 0.0;
    for (int64_t i0 = 0; i0 < rows; i0 += kRRows) {
        const int nr = (int)(rows - i0 < kRRows ? rows - i0 : kRRows);
        __syncthreads();
        for (int e = threadIdx.x; e < nr * k; e += kRThreads) {
            const int a = e / nr, i = e - a * nr;
            S.chunk[i * kRMax + a] = F[(int64_t)a * rows + i0 + i];
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            const int idx = threadIdx.x + j * kRThreads;
            const int a = idx / kRMax, b = idx % kRMax;
            if (a < k && b < k) {
                double s = acc[j];
                for (int i = 0; i < nr; ++i) s += S.chunk[i * kRMax + a] * S.chunk[i * kRMax + b];
                acc[j] = s;
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        const int idx = threadIdx.x + j * kRThreads;
        const int a = idx / kRMax, b = idx % kRMax;
        if (a < k && b < k) S.A[a * kRMax + b] = acc[j];
    }
    __syncthreads();
}

// Parallel cyclic Jacobi (round-robin pairing: all pairs of a step are disjoint and commute) on the
// symmetric k x k matrix S.A; eigenvectors accumulate into V (columns); eigenvalues -> ev.
__device__ void jacobi_eig(RSmem& S, double* V, double* ev, int k) {
    const int kk = (k + 1) & ~1;     // even player count; index k (odd k) is a zero dummy
    const int np = kk / 2;
    for (int e = threadIdx.x; e < kRMax * kRMax; e += kRThreads) {
        const int a = e / kRMax, b = e % kRMax;
        V[e] = a == b ? 1.0 : 0.0;
        if (a >= k || b >= k) S.A[e] = 0.0;
    }
    __syncthreads();
    for (int sweep = 0; sweep < 20; ++sweep) {
        // convergence: off-diagonal mass vs diagonal mass
        double off = 0.0, dia = 0.0;
        for (int e = threadIdx.x; e < k * k; e += kRThreads) {
            const int a = e / k, b = e % k;
            const double v = S.A[a * kRMax + b];
            if (a == b) dia += v * v; else off += v * v;
        }
        for (int o = 16; o > 0; o >>= 1) {
            off += __shfl_xor_sync(0xffffffffu, off, o);
            dia += __shfl_xor_sync(0xffffffffu, dia, o);
        }
        __syncthreads();
        if ((threadIdx.x & 31) == 0) S.red[threadIdx.x >> 5] = off;
        __syncthreads();
        double offt = 0.0;
        for (int w = 0; w < kRThreads / 32; ++w) offt += S.red[w];
        __syncthreads();
        if ((threadIdx.x & 31) == 0) S.red[threadIdx.x >> 5] = dia;
        __syncthreads();
        double diat = 0.0;
        for (int w = 0; w < kRThreads / 32; ++w) diat += S.red[w];
        __syncthreads();
        if (!(offt > 1e-30 * diat)) break;   // off-diagonal <= 1e-15 relative; also stops on a zero matrix
        for (int step = 0; step < kk - 1; ++step) {
            if (threadIdx.x < np) {   // rotation of pair p (Numerical Recipes convention)
                const int p = threadIdx.x;
                int a, b;
                if (p == 0) { a = 0; b = 1 + step % (kk - 1); }
                else { a = 1 + (step + p) % (kk - 1); b = 1 + (step - p + kk - 1) % (kk - 1); }
                double c = 1.0, s = 0.0;
                if (a < k && b < k) {
                    const double apq = S.A[a * kRMax + b];
                    const double app = S.A[a * kRMax + a], aqq = S.A[b * kRMax + b];
                    if (apq != 0.0 && fabs(apq) > 1e-300) {
                        const double th = (aqq - app) / (2.0 * apq);
                        const double t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
                        c = 1.0 / sqrt(t * t + 1.0);
                        s = t * c;
                    }
                }
                S.rc[p] = c;
                S.rs[p] = s;
                S.order[2 * p] = a;
                S.order[2 * p + 1] = b;
            }
            __syncthreads();
            // columns: A[:, a], A[:, b] and V[:, a], V[:, b]
            for (int e = threadIdx.x; e < np * kk; e += kRThreads) {
                const int p = e / kk, r = e - p * kk;
                const double c = S.rc[p], s = S.rs[p];
                if (s == 0.0) continue;
                const int a = S.order[2 * p], b = S.order[2 * p + 1];
                const double x = S.A[r * kRMax + a], y = S.A[r * kRMax + b];
                S.A[r * kRMax + a] = c * x - s * y;
                S.A[r * kRMax + b] = s * x + c * y;
                const double vx = V[r * kRMax + a], vy = V[r * kRMax + b];
                V[r * kRMax + a] = c * vx - s * vy;
                V[r * kRMax + b] = s * vx + c * vy;
            }
            __syncthreads();
            // rows: A[a, :], A[b, :]
            for (int e = threadIdx.x; e < np * kk; e += kRThreads) {
                const int p = e / kk, r = e - p * kk;
                const double c = S.rc[p], s = S.rs[p];
                if (s == 0.0) continue;
                const int a = S.order[2 * p], b = S.order[2 * p + 1];
                const double x = S.A[a * kRMax + r], y = S.A[b * kRMax + r];
                S.A[a * kRMax + r] = c * x - s * y;
                S.A[b * kRMax + r] = s * x + c * y;
            }
            __syncthreads();
        }
    }
    for (int a = threadIdx.x; a < k; a += kRThreads) ev[a] = S.A[a * kRMax + a];
    __syncthreads();
}

// F (rows x k, column-major, ld = rows) <- F T[:, :kn] in place, row chunk by row chunk
__device__ void transform(RSmem& S, double* F, int64_t rows, int k, int kn) {
    for (int64_t i0 = 0; i0 < rows; i0 += kRRows) {
        const int nr = (int)(rows - i0 < kRRows ? rows - i0 : kRRows);
        __syncthreads();
        for (int e = threadIdx.x; e < nr * k; e += kRThreads) {
            const int a = e / nr, i = e - a * nr;
            S.chunk[i * kRMax + a] = F[(int64_t)a * rows + i0 + i];
        }
        __syncthreads();
        for (int e = threadIdx.x; e < nr * kn; e += kRThreads) {
            const int j = e / nr, i = e - j * nr;
            double s = 0.0;
            for (int a = 0; a < k; ++a) s += S.chunk[i * kRMax + a] * S.T[a * kRMax + j];
            F[(int64_t)j * rows + i0 + i] = s;
        }
    }
    __syncthreads();
}

// blk[5 q + 0..4] = uoff, m, voff, n, k (offsets into base)
__global__ void __launch_bounds__(kRThreads) recompress_kernel(double* base, const int64_t* __restrict__ blk,
                                                               double eps, int32_t* __restrict__ new_rank) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    RSmem& S = *reinterpret_cast<RSmem*>(smem_raw);
    const int64_t* b = blk + 5 * (int64_t)blockIdx.x;
    double* U = base + b[0];
    double* Vf = base + b[2];
    const int64_t m = b[1], n = b[3];
    const int k = (int)b[4];
    // 1. G_U = U^T U = W diag(lam) W^T
    gram(S, U, m, k);
    jacobi_eig(S, S.W, S.lam, k);
    double lmax = 0.0;
    for (int a = 0; a < k; ++a) lmax = fmax(lmax, S.lam[a]);
    // 2. N = B G_V B^T with B = diag(sqrt lam) W^T (dropped directions: zero rows)
    gram(S, Vf, n, k);                                   // S.A = G_V
    for (int e = threadIdx.x; e < k * k; e += kRThreads) {   // T = B G_V
        const int a = e / k, d = e % k;
        const double la = S.lam[a];
        double s = 0.0;
        if (la > 1e-26 * lmax) {
            for (int c = 0; c < k; ++c) s += S.W[c * kRMax + a] * S.A[c * kRMax + d];
            s *= sqrt(la);
        }
        S.T[a * kRMax + d] = s;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < k * k; e += kRThreads) {   // N = T B^T
        const int a = e / k, c = e % k;
        const double lc = S.lam[c];
        double s = 0.0;
        if (lc > 1e-26 * lmax) {
            for (int d = 0; d < k; ++d) s += S.T[a * kRMax + d] * S.W[d * kRMax + c];
            s *= sqrt(lc);
        }
        S.Xe[a * kRMax + c] = s;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < k * k; e += kRThreads) {   // symmetrise into A
        const int a = e / k, c = e % k;
        S.A[a * kRMax + c] = 0.5 * (S.Xe[a * kRMax + c] + S.Xe[c * kRMax + a]);
    }
    __syncthreads();
    jacobi_eig(S, S.Xe, S.s2, k);
    // 3. order by s^2 descending (ties: lower index first), truncation rank k'
    for (int a = threadIdx.x; a < k; a += kRThreads) {
        const double v = fmax(S.s2[a], 0.0);
        int r = 0;
        for (int c = 0; c < k; ++c) {
            const double w = fmax(S.s2[c], 0.0);
            r += (w > v) || (w == v && c < a);
        }
        S.order[r] = a;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double total = 0.0;
        for (int r = 0; r < k; ++r) total += fmax(S.s2[S.order[r]], 0.0);
        double tail = 0.0;
        int kn = k;
        // tail(i) = sum_{r >= i} s_r^2; smallest i with tail(i) <= eps^2 total
        double tails[kRMax + 1];
        tails[k] = 0.0;
        for (int r = k - 1; r >= 0; --r) { tail += fmax(S.s2[S.order[r]], 0.0); tails[r] = tail; }
        for (int i = 0; i <= k; ++i)
            if (tails[i] <= eps * eps * total) { kn = i; break; }
        S.kk_new = kn;
    }
    __syncthreads();
    const int kn = S.kk_new;
    // 4. T_U = W diag(lam^-1/2) Xe[:, order[:k']] -> U' = U T_U
    for (int e = threadIdx.x; e < k * kn; e += kRThreads) {
        const int a = e / kn, j = e % kn;
        const int col = S.order[j];
        double s = 0.0;
        for (int c = 0; c < k; ++c) {
            const double lc = S.lam[c];
            if (lc > 1e-26 * lmax) s += S.W[a * kRMax + c] * (S.Xe[c * kRMax + col] / sqrt(lc));
        }
        S.T[a * kRMax + j] = s;
    }
    __syncthreads();
    transform(S, U, m, k, kn);
    // 5. T_V = B^T Xe[:, order[:k']] = W diag(sqrt lam) Xe -> V' = V T_V
    for (int e = threadIdx.x; e < k * kn; e += kRThreads) {
        const int a = e / kn, j = e % kn;
        const int col = S.order[j];
        double s = 0.0;
        for (int c = 0; c < k; ++c) {
            const double lc = S.lam[c];
            if (lc > 1e-26 * lmax) s += S.W[a * kRMax + c] * (sqrt(lc) * S.Xe[c * kRMax + col]);
        }
        S.T[a * kRMax + j] = s;
    }
    __syncthreads();
    transform(S, Vf, n, k, kn);
    if (threadIdx.x == 0) new_rank[blockIdx.x] = kn;
}

}  // namespace

namespace k {
void recompress_batch(double* base, const int64_t* blk, int nb, double eps, int32_t* new_rank, cudaStream_t s) {
    if (nb <= 0) return;
    static bool attr = false;
    if (!attr) {
        HM_CUDA(cudaFuncSetAttribute(recompress_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(RSmem)));
        attr = true;
    }
    recompress_kernel<<<nb, kRThreads, sizeof(RSmem), s>>>(base, blk, eps, new_rank);
    HM_CUDA(cudaGetLastError());
    debug_sync(s, "recompress_kernel");
}
}  // namespace k

}  // namespace hm
