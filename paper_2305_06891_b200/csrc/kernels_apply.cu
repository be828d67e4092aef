// Hot-path kernels: the two-phase streaming H-apply.
//
//   phase 1 (K6): t_b = V_b^T x_tau for every low-rank block b.  All blocks sharing a column
//                 cluster tau are stacked into one column-major panel (K_tau x n_tau), so the
//                 pass is a stream of contiguous columns times x_tau.
//   phase 2 (K7): per leaf row r: out_r (op)= the leaf row's column stream (dense near-field
//                 slices and U slices, contiguous in HBM, column-major) times the gathered
//                 inputs XT[colsrc[c]] (x for dense columns, t for U columns).
// Both run through ONE kernel over ~48 KB work units with 16-byte loads; split-K partials of a
// row tile are added by its last-arriving unit in fixed order (deterministic, no FP atomics).
// The same kernel runs the F apply ("x -> F x ... recursively") and every level
// of the level-scheduled substitution (W^L / W^U updates, leaf inverses).
#include <cstdint>

#include "hm_internal.h"

namespace hm {
namespace {

constexpr int kThreads = 256;
constexpr int kQ = 12;          // columns per thread per work unit (row tile <= 128 rows)

__device__ __forceinline__ double pow4(double T) {
    const double t2 = T * T;
    return t2 * t2;
}

__device__ __forceinline__ void emit(double* __restrict__ out, int64_t row, double s, int mode,
                                     const int32_t* __restrict__ perm, const FluxEpi& epi) {
    switch (mode) {
        case OUT_ASSIGN: out[row] = s; break;
        case OUT_SUB: out[row] -= s; break;
        case OUT_PERM: out[(int64_t)perm[row] * epi.ld + epi.col] = s; break;
        default: {  // OUT_FLUX: q = sigma (eps/A) (F z - eta g), eq:qi_new_location operator form
            const int64_t e = perm[row];
            const double eta = pow4(epi.T_ext[e * epi.ld + epi.col]);
            out[e * epi.ld + epi.col] = epi.sigma * (epi.eps_int[row] / epi.area_int[row]) * (s - eta * epi.g_int[row]);
        }
    }
}

// One CTA per work unit.  Rows are processed in pairs (16-byte loads); the chunk's columns are
// split over G = 256 / pairs thread groups so that every thread owns at most kQ columns.  Each
// thread issues all of its payload loads first (streaming hint: the factors are read once, the
// vectors stay in L2), the gathered inputs of the chunk are staged once in shared memory, then
// the FMAs run; partial sums are reduced through shared memory in fixed order.
__global__ void __launch_bounds__(kThreads, 3)
stream_kernel(const Unit* __restrict__ units, const int32_t* __restrict__ colsrc, const double* __restrict__ arena,
              const double* __restrict__ xt, double* __restrict__ out, int mode, const int32_t* __restrict__ perm,
              FluxEpi epi, double* __restrict__ part, int32_t* __restrict__ counters) {
    __shared__ double2 red[kThreads];
    __shared__ double xs[kThreads * kQ];
    __shared__ int s_last;
    // PDL: the next pass may start streaming its (constant) factor payload while this one drains
    asm volatile("griddepcontrol.launch_dependents;");
    const Unit u = units[blockIdx.x];
    const int P = (u.nrows + 1) >> 1;
    const int G = kThreads / P;
    const int g = threadIdx.x / P;
    const int p = threadIdx.x - g * P;
    const bool active = g < G;
    double2 av[kQ];
    {
        const double2* a = reinterpret_cast<const double2*>(arena + u.a_off + (int64_t)u.c0 * u.ld) + p;
        const int64_t ld2 = u.ld >> 1;
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
            const int c = g + q * G;
            av[q] = (active && c < u.ncols) ? __ldcs(a + (int64_t)c * ld2) : make_double2(0.0, 0.0);
        }
    }
    // everything above reads only constant operator data; vectors are produced by the previous pass
    asm volatile("griddepcontrol.wait;" ::: "memory");
    {
        const int32_t* cs = colsrc + u.cs_off + u.c0;
        for (int c = threadIdx.x; c < u.ncols; c += kThreads) xs[c] = xt[__ldg(cs + c)];
    }
    __syncthreads();
    double2 acc = make_double2(0.0, 0.0), acc2 = make_double2(0.0, 0.0);
    if (active) {
#pragma unroll
        for (int q = 0; q < kQ; q += 2) {
            const int c = g + q * G;
            if (c < u.ncols) {
                const double x = xs[c];
                acc.x = fma(av[q].x, x, acc.x);
                acc.y = fma(av[q].y, x, acc.y);
            }
            if (q + 1 < kQ && c + G < u.ncols) {
                const double x = xs[c + G];
                acc2.x = fma(av[q + 1].x, x, acc2.x);
                acc2.y = fma(av[q + 1].y, x, acc2.y);
            }
        }
        acc.x += acc2.x;
        acc.y += acc2.y;
        red[g * P + p] = acc;
    }
    __syncthreads();
    double2 s = make_double2(0.0, 0.0);
    const bool owner = threadIdx.x < P;
    if (owner) {
        s = red[p];
        for (int q = 1; q < G; ++q) {
            const double2 v = red[q * P + p];
            s.x += v.x;
            s.y += v.y;
        }
    }
    if (u.grp < 0) {
        if (owner) {
            const int r = 2 * p;
            emit(out, u.out0 + r, s.x, mode, perm, epi);
            if (r + 1 < u.nrows) emit(out, u.out0 + r + 1, s.y, mode, perm, epi);
        }
        return;
    }
    // split-K: publish the partial, the last unit of the group adds all partials in order
    if (owner) reinterpret_cast<double2*>(part + u.part_off)[p] = s;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const int prev = atomicAdd(counters + u.grp, 1);
        s_last = (prev == u.nseg - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (owner) {
        const int first = (int)blockIdx.x - u.seg;   // units of a group are consecutive
        double2 t = make_double2(0.0, 0.0);
        for (int q = 0; q < u.nseg; ++q) {
            const Unit& uq = units[first + q];
            const double2 v = __ldcg(reinterpret_cast<const double2*>(part + uq.part_off) + p);
            t.x += v.x;
            t.y += v.y;
        }
        const int r = 2 * p;
        emit(out, u.out0 + r, t.x, mode, perm, epi);
        if (r + 1 < u.nrows) emit(out, u.out0 + r + 1, t.y, mode, perm, epi);
    }
    if (threadIdx.x == 0) counters[u.grp] = 0;   // re-arm for the next launch (graph-replay safe)
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

void stream_pass(const StreamPass& p, const int32_t* colsrc, const double* arena, const double* xt, double* out,
                 int mode, const int32_t* perm, const FluxEpi* epi, cudaStream_t s) {
    if (p.n_units == 0) return;
    FluxEpi e{};
    if (epi) e = *epi;
    if (e.ld == 0) e.ld = 1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)p.n_units);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    HM_CUDA(cudaLaunchKernelEx(&cfg, stream_kernel, p.units.p, colsrc, arena, xt, out, mode, perm, e, p.part.p,
                               p.counters.p));
    debug_sync(s, "stream_kernel");
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
