// Hot-path kernels: the two-phase streaming H-apply.
//
//   phase 1 (K6): t_b = V_b^T x_tau for every low-rank block b -- one warp per row of V_b^T,
//                 coalesced loads along the row, warp-shuffle reduction, no atomics.
//   phase 2 (K7): per leaf row r: out_r (op)= sum of the leaf row's column stream
//                 (dense near-field slices and U slices, contiguous in HBM, column-major) times
//                 the gathered inputs XT[colsrc[c]] (x for dense columns, t for U columns).
//                 One CTA per leaf row owns its outputs (deterministic, no atomics).
// The same two kernels run the F apply ("x -> F x ... recursively") and every
// level of the level-scheduled substitution (W^L / W^U updates, leaf inverses).
#include <cstdint>

#include "hm_internal.h"

namespace hm {
namespace {

constexpr int kP1Threads = 256;
constexpr int kP2Threads = 256;

__global__ void __launch_bounds__(kP1Threads)
phase1_kernel(const P1Task* __restrict__ tasks, int64_t ntasks, const double* __restrict__ arena,
              double* __restrict__ xt, int64_t n) {
    const int64_t w = ((int64_t)blockIdx.x * kP1Threads + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= ntasks) return;
    const P1Task t = tasks[w];
    const double* a = arena + t.off;
    const double* x = xt + t.x_off;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int c = lane;
    for (; c + 96 < t.n; c += 128) {
        const double a0 = __ldg(a + c), a1 = __ldg(a + c + 32), a2 = __ldg(a + c + 64), a3 = __ldg(a + c + 96);
        s0 = fma(a0, x[c], s0);
        s1 = fma(a1, x[c + 32], s1);
        s2 = fma(a2, x[c + 64], s2);
        s3 = fma(a3, x[c + 96], s3);
    }
    for (; c < t.n; c += 32) s0 = fma(__ldg(a + c), x[c], s0);
    double s = (s0 + s1) + (s2 + s3);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) xt[n + w] = s;
}

__device__ __forceinline__ double pow4(double T) {
    const double t2 = T * T;
    return t2 * t2;
}

__global__ void __launch_bounds__(kP2Threads)
phase2_kernel(const P2Row* __restrict__ rows, const int32_t* __restrict__ colsrc,
              const double* __restrict__ arena, const double* __restrict__ xt, double* __restrict__ out,
              int mode, const int32_t* __restrict__ perm, FluxEpi epi) {
    extern __shared__ double red[];
    const P2Row r = rows[blockIdx.x];
    const int m = r.m;
    const int G = kP2Threads / m;
    const int g = threadIdx.x / m;
    const int i = threadIdx.x - g * m;
    double acc = 0.0;
    if (g < G) {
        const double* a = arena + r.region + i;
        const int32_t* cs = colsrc + r.col0;
        double acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
        int c = g;
        for (; c + 3 * G < r.ncols; c += 4 * G) {
            const int32_t s0 = cs[c], s1 = cs[c + G], s2 = cs[c + 2 * G], s3 = cs[c + 3 * G];
            const double a0 = __ldg(a + (int64_t)c * m);
            const double a1 = __ldg(a + (int64_t)(c + G) * m);
            const double a2 = __ldg(a + (int64_t)(c + 2 * G) * m);
            const double a3 = __ldg(a + (int64_t)(c + 3 * G) * m);
            acc = fma(a0, xt[s0], acc);
            acc1 = fma(a1, xt[s1], acc1);
            acc2 = fma(a2, xt[s2], acc2);
            acc3 = fma(a3, xt[s3], acc3);
        }
        for (; c < r.ncols; c += G) acc = fma(__ldg(a + (int64_t)c * m), xt[cs[c]], acc);
        acc = (acc + acc1) + (acc2 + acc3);
        red[g * m + i] = acc;
    }
    __syncthreads();
    if (g == 0) {
        double s = red[i];
        for (int q = 1; q < G; ++q) s += red[q * m + i];
        const int64_t row = (int64_t)r.r0 + i;
        switch (mode) {
            case OUT_ASSIGN: out[row] = s; break;
            case OUT_SUB: out[row] -= s; break;
            case OUT_PERM: out[(int64_t)perm[row] * epi.ld + epi.col] = s; break;
            default: {  // OUT_FLUX
                const int64_t e = perm[row];
                const double eta = pow4(epi.T_ext[e * epi.ld + epi.col]);
                out[e * epi.ld + epi.col] =
                    epi.sigma * (epi.eps_int[row] / epi.area_int[row]) * (s - eta * epi.g_int[row]);
            }
        }
    }
}

__global__ void permute_in_kernel(const double* __restrict__ x_ext, int ld, int col, const int32_t* __restrict__ perm,
                                  double* __restrict__ x_int, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) x_int[i] = x_ext[(int64_t)perm[i] * ld + col];
}
__global__ void permute_out_kernel(const double* __restrict__ y_int, const int32_t* __restrict__ perm,
                                   double* __restrict__ y_ext, int ld, int col, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y_ext[(int64_t)perm[i] * ld + col] = y_int[i];
}
__global__ void flux_prologue_kernel(const double* __restrict__ T_ext, int ld, int col, const int32_t* __restrict__ perm,
                                     const double* __restrict__ eps_int, double* __restrict__ w, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) w[i] = eps_int[i] * pow4(T_ext[(int64_t)perm[i] * ld + col]);
}
__global__ void fill_value_kernel(double* p, int64_t n, double v) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}
// s_i = (F_H 1)_i / A_i (eq:rowsum), c_i = clamp(s_i, 0, 1) (eq:clamped_rowsum),
// cdiv_i = c_i if c_i != 0 else 1 (eqn:F_closed leaves rows with c_i = 0 untouched)
__global__ void row_sums_kernel(const double* __restrict__ y, const double* __restrict__ area, double* s,
                                double* c, double* cdiv, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double si = y[i] / area[i];
    const double ci = si < 0.0 ? 0.0 : (si > 1.0 ? 1.0 : si);
    s[i] = si;
    c[i] = ci;
    cdiv[i] = ci != 0.0 ? ci : 1.0;
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

namespace k {

void phase1(const P1Task* tasks, int64_t ntasks, const double* arena, double* xt, int64_t n, cudaStream_t s) {
    if (ntasks == 0) return;
    phase1_kernel<<<nblk(ntasks * 32, kP1Threads), kP1Threads, 0, s>>>(tasks, ntasks, arena, xt, n);
    HM_CUDA(cudaGetLastError());
    debug_sync(s, "phase1");
}

void phase2(const P2Row* rows, int64_t nrows, int max_m, const int32_t* colsrc, const double* arena,
            const double* xt, double* out, int mode, const int32_t* perm, const FluxEpi* epi, cudaStream_t s) {
    if (nrows == 0) return;
    FluxEpi e{};
    if (epi) e = *epi;
    if (e.ld == 0) e.ld = 1;
    phase2_kernel<<<(unsigned)nrows, kP2Threads, kP2Threads * sizeof(double), s>>>(rows, colsrc, arena, xt, out,
                                                                                    mode, perm, e);
    HM_CUDA(cudaGetLastError());
    debug_sync(s, "phase2");
    (void)max_m;
}

void permute_in(const double* x_ext, int ld, int col, const int32_t* perm, double* x_int, int64_t n, cudaStream_t s) {
    permute_in_kernel<<<nblk(n, 256), 256, 0, s>>>(x_ext, ld, col, perm, x_int, n);
    HM_CUDA(cudaGetLastError());
    debug_sync(s, "permute_in");
}
void permute_out(const double* y_int, const int32_t* perm, double* y_ext, int ld, int col, int64_t n, cudaStream_t s) {
    permute_out_kernel<<<nblk(n, 256), 256, 0, s>>>(y_int, perm, y_ext, ld, col, n);
    HM_CUDA(cudaGetLastError());
    debug_sync(s, "permute_out");
}
void flux_prologue(const double* T_ext, int ld, int col, const int32_t* perm, const double* eps_int, double* w_int,
                   int64_t n, cudaStream_t s) {
    flux_prologue_kernel<<<nblk(n, 256), 256, 0, s>>>(T_ext, ld, col, perm, eps_int, w_int, n);
    HM_CUDA(cudaGetLastError());
    debug_sync(s, "flux_prologue");
}
void fill_value(double* p, int64_t n, double v, cudaStream_t s) {
    if (n == 0) return;
    fill_value_kernel<<<nblk(n, 256), 256, 0, s>>>(p, n, v);
    HM_CUDA(cudaGetLastError());
}
void row_sums_clamp(const double* y, const double* area, double* sv, double* c, double* cdiv, int64_t n,
                    cudaStream_t s) {
    row_sums_kernel<<<nblk(n, 256), 256, 0, s>>>(y, area, sv, c, cdiv, n);
    HM_CUDA(cudaGetLastError());
}

}  // namespace k
}  // namespace hm
