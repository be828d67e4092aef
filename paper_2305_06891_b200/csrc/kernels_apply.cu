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

// Facet <- node projection (eqn:P_fi_definition), one facet row per thread:
// mode 0: eta_i = sum_M P_iM T_M^4 (eqn:flux_residual_3 input); mode 1: eta_i = sum_M P_iM 4 T_M^3 x_M
// (eq:Jcav input).  T, x: n_nodes x ld, column col.
__global__ void proj_facets_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col_idx,
                                   const double* __restrict__ val, const double* __restrict__ T,
                                   const double* __restrict__ x, int mode, int ld, int col, double* __restrict__ eta,
                                   int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;
    for (int64_t q = rp[i]; q < rp[i + 1]; ++q) {
        const int64_t M = col_idx[q];
        const double t = T[M * ld + col];
        const double t3 = t * t * t;
        s += val[q] * (mode == 0 ? t3 * t : 4.0 * t3 * x[M * ld + col]);
    }
    eta[i] = s;
}
// Node <- facet transpose (P^T, eqn:S_def_matrix): Q_M = sum_{i ~ M} P_iM y_i in fixed facet order
// (deterministic, no atomics); Q: n_nodes x ld, column col.
__global__ void proj_nodes_kernel(const int64_t* __restrict__ tp, const int32_t* __restrict__ tidx,
                                  const double* __restrict__ tval, const double* __restrict__ y, int ld, int col,
                                  double* __restrict__ Q, int64_t n_nodes) {
    const int64_t M = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (M >= n_nodes) return;
    double s = 0.0;
    for (int64_t q = tp[M]; q < tp[M + 1]; ++q) s += tval[q] * y[tidx[q]];
    Q[M * ld + col] = s;
}

__global__ void sum_segments_kernel(const double* __restrict__ buf, int world, int64_t count, int64_t n, int ld,
                                    int col, double* __restrict__ out) {
    const int64_t N = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (N >= n) return;
    double s = 0.0;
    for (int r = 0; r < world; ++r) s += buf[(int64_t)r * count + N];
    out[N * ld + col] = s;
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

namespace k {

void sum_segments(const double* buf, int world, int64_t count, int64_t n, int ld, int col, double* out, cudaStream_t s) {
    sum_segments_kernel<<<nblk(n, 256), 256, 0, s>>>(buf, world, count, n, ld, col, out);
    HM_CUDA(cudaGetLastError());
    debug_sync(s, "sum_segments");
}

void proj_facets(const int64_t* rp, const int32_t* col_idx, const double* val, const double* T, const double* x,
                 int mode, int ld, int col, double* eta, int64_t n, cudaStream_t s) {
    if (n == 0) return;
    proj_facets_kernel<<<nblk(n, 256), 256, 0, s>>>(rp, col_idx, val, T, x, mode, ld, col, eta, n);
    HM_CUDA(cudaGetLastError());
    debug_sync(s, "proj_facets");
}
void proj_nodes(const int64_t* tp, const int32_t* tidx, const double* tval, const double* y, int ld, int col, double* Q,
                int64_t n_nodes, cudaStream_t s) {
    if (n_nodes == 0) return;
    proj_nodes_kernel<<<nblk(n_nodes, 256), 256, 0, s>>>(tp, tidx, tval, y, ld, col, Q, n_nodes);
    HM_CUDA(cudaGetLastError());
    debug_sync(s, "proj_nodes");
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
