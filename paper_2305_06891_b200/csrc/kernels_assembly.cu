// Setup kernels that produce the hot path's data:
//   K1 vf_entry     -- view-factor entry, eq:Fdef_new_location: one-point centroid
//                      rule, or the adaptive Gauss quadrature of PAPER.md:156 (reading R35) for near pairs
//   K2 fill_entries -- dense near-field blocks
//   K3 aca_batch    -- adaptive cross approximation with partial pivoting,
//                      one CTA per admissible block, reading R10 step by step
//   pack / scale_rows -- arena layout and closed-cavity row scaling (eqn:F_closed)
// Entry and ACA arithmetic use explicit __dmul_rn/__dadd_rn/__dsub_rn/__ddiv_rn (never
// contracted into FMA), so entries, pivots and factors are the exact IEEE sequence of R22.
#include <cstdint>

#include "hm_internal.h"

namespace hm {
namespace {

constexpr double kPi = 3.141592653589793;  // the double nearest to pi

struct GeoView {
    const double *cx, *cy, *cz, *nx, *ny, *nz, *A;
    const double* Q;   // adaptive quadrature table (reading R35), internal order, kQStride per facet; or null
    __device__ GeoView(const double* g, int64_t n, const double* q)
        : cx(g), cy(g + n), cz(g + 2 * n), nx(g + 3 * n), ny(g + 4 * n), nz(g + 5 * n), A(g + 6 * n), Q(q) {}
};

// ---------------------------------------------------------------- adaptive Gauss quadrature (R35)
// the rule's order grows as facets get closer.  Table row of a facet (built on the host,
// api.cpp quad_table): the 3 points of the degree-2 rule, the 6 of Dunavant's degree-4 rule, the 24 of
// that rule on the 4 midpoint sub-triangles (x, y, z each), then the squared longest edge.
__device__ __forceinline__ double tier_weight(int tier, int p) {
    constexpr double w3 = 1.0 / 3.0;
    constexpr double wa = 0.223381589678011, wb = 0.109951743655322;   // Dunavant degree 4
    if (tier == 1) return w3;
    const double w = (p % 6) < 3 ? wa : wb;
    return tier == 2 ? w : __dmul_rn(0.25, w);
}
// F_ab = A_a A_b sum_p sum_q w_p w_q cos_p cos_q / (pi r_pq^2), points p on facet a, q on facet b (a < b),
// p-major; a point pair facing away (R3) adds nothing
__device__ double quad_entry(const GeoView& g, int64_t a, int64_t b, int tier, int32_t* err) {
    const int off = tier == 1 ? kQOff1 : tier == 2 ? kQOff2 : kQOff3;
    const int np = tier == 1 ? 3 : tier == 2 ? 6 : 24;
    const double* Pa = g.Q + a * kQStride + off;
    const double* Pb = g.Q + b * kQStride + off;
    const double nax = g.nx[a], nay = g.ny[a], naz = g.nz[a], nbx = g.nx[b], nby = g.ny[b], nbz = g.nz[b];
    double s = 0.0;
    for (int p = 0; p < np; ++p) {
        const double xa = Pa[3 * p], ya = Pa[3 * p + 1], za = Pa[3 * p + 2];
        const double wp = tier_weight(tier, p);
        for (int q = 0; q < np; ++q) {
            const double dx = __dsub_rn(Pb[3 * q], xa);
            const double dy = __dsub_rn(Pb[3 * q + 1], ya);
            const double dz = __dsub_rn(Pb[3 * q + 2], za);
            const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
            if (r2 == 0.0) {
                if (atomicCAS(err, 0, 1) == 0) { err[1] = (int32_t)a; err[2] = (int32_t)b; }
                return 0.0;
            }
            const double ca = __dadd_rn(__dadd_rn(__dmul_rn(nax, dx), __dmul_rn(nay, dy)), __dmul_rn(naz, dz));
            const double cb = -__dadd_rn(__dadd_rn(__dmul_rn(nbx, dx), __dmul_rn(nby, dy)), __dmul_rn(nbz, dz));
            if (!(ca > 0.0 && cb > 0.0)) continue;
            const double t = __ddiv_rn(__dmul_rn(__dmul_rn(wp, tier_weight(tier, q)), __dmul_rn(ca, cb)),
                                       __dmul_rn(__dmul_rn(kPi, r2), r2));
            s = __dadd_rn(s, t);
        }
    }
    return __dmul_rn(__dmul_rn(g.A[a], g.A[b]), s);
}

// K1: F_ij = (A_i A_j cos(phi_i) cos(phi_j)) / (pi R^2) by the centroid rule, canonical
// pair (a,b) = (min,max); back-facing pairs -> 0 (R3); F_ii = 0.
__device__ __forceinline__ double vf_entry(const GeoView& g, int64_t i, int64_t j, int32_t* err) {
    if (i == j) return 0.0;
    const int64_t a = i < j ? i : j;
    const int64_t b = i < j ? j : i;
    const double dx = __dsub_rn(g.cx[b], g.cx[a]);
    const double dy = __dsub_rn(g.cy[b], g.cy[a]);
    const double dz = __dsub_rn(g.cz[b], g.cz[a]);
    const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    const double ca = __dadd_rn(__dadd_rn(__dmul_rn(g.nx[a], dx), __dmul_rn(g.ny[a], dy)), __dmul_rn(g.nz[a], dz));
    const double cb = -__dadd_rn(__dadd_rn(__dmul_rn(g.nx[b], dx), __dmul_rn(g.ny[b], dy)), __dmul_rn(g.nz[b], dz));
    if (r2 == 0.0) {
        if (atomicCAS(err, 0, 1) == 0) { err[1] = (int32_t)a; err[2] = (int32_t)b; }
        return 0.0;
    }
    if (g.Q) {   // reading R35: pairs closer than 10 h take a quadrature tier (tau^2 = 100, 16, 2.25)
        const double h2 = fmax(g.Q[a * kQStride + kQH2], g.Q[b * kQStride + kQH2]);
        if (!(r2 >= __dmul_rn(100.0, h2)))
            return quad_entry(g, a, b, r2 >= __dmul_rn(16.0, h2) ? 1 : r2 >= __dmul_rn(2.25, h2) ? 2 : 3, err);
    }
    if (!(ca > 0.0 && cb > 0.0)) return 0.0;
    const double num = __dmul_rn(__dmul_rn(g.A[a], g.A[b]), __dmul_rn(ca, cb));
    const double den = __dmul_rn(__dmul_rn(kPi, r2), r2);
    return __ddiv_rn(num, den);
}

// ---------------------------------------------------------------- deterministic CTA reductions
constexpr int kAcaThreads = 256;
constexpr int kAcaWarps = kAcaThreads / 32;

struct ArgMax {
    double v;   // |value|; -1 marks "none"
    int64_t i;
};
__device__ __forceinline__ ArgMax better(ArgMax x, ArgMax y) {  // larger |v|, lower index on ties
    if (y.v > x.v) return y;
    if (y.v == x.v && y.i < x.i && y.v >= 0.0) return y;
    return x;
}
__device__ ArgMax cta_argmax(ArgMax a, ArgMax* sm) {
    for (int o = 16; o > 0; o >>= 1) {
        ArgMax b;
        b.v = __shfl_xor_sync(0xffffffffu, a.v, o);
        b.i = __shfl_xor_sync(0xffffffffu, a.i, o);
        a = better(a, b);
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sm[w] = a;
    __syncthreads();
    ArgMax r = sm[0];
    for (int q = 1; q < kAcaWarps; ++q) r = better(r, sm[q]);
    return r;
}
// sums NV values per thread at once (fixed order: lane tree, then warps ascending)
template <int NV>
__device__ void cta_sum(double (&v)[NV], double* sm /* kAcaWarps*NV */) {
    for (int q = 0; q < NV; ++q)
        for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0)
        for (int q = 0; q < NV; ++q) sm[w * NV + q] = v[q];
    __syncthreads();
    for (int q = 0; q < NV; ++q) {
        double s = sm[q];
        for (int ww = 1; ww < kAcaWarps; ++ww) s += sm[ww * NV + q];
        v[q] = s;
    }
}

__device__ __forceinline__ bool bit_get(const uint32_t* b, int64_t i) { return (b[i >> 5] >> (i & 31)) & 1u; }

// K3: one CTA per admissible block (rows r0..r0+m, cols c0..c0+n of the internal order).
// U slot l at U[l*m + i], V slot l at V[l*n + j]; slot k doubles as the residual buffer.
__global__ void __launch_bounds__(kAcaThreads)
aca_kernel(const double* __restrict__ geo, int64_t ntot, const int64_t* __restrict__ blk,
           const int64_t* __restrict__ uoff, const int64_t* __restrict__ voff,
           const int32_t* __restrict__ kcap_arr, double eps, double* __restrict__ scratch,
           int32_t* __restrict__ rank_out, double* __restrict__ margin_out, int32_t* err, int probes,
           const double* __restrict__ quad) {
    __shared__ int64_t s_probe;
    extern __shared__ uint32_t smem_bits[];
    __shared__ ArgMax s_am[kAcaWarps];
    __shared__ double s_red[kAcaWarps * 8];
    __shared__ double s_urow[64], s_vcol[64];
    __shared__ double s_xu[64], s_xv[64];

    const int b = blockIdx.x;
    const int64_t r0 = blk[4 * b], m = blk[4 * b + 1], c0 = blk[4 * b + 2], n = blk[4 * b + 3];
    double* U = scratch + uoff[b];
    double* V = scratch + voff[b];
    const int kcap = kcap_arr[b];
    const GeoView g(geo, ntot, quad);
    uint32_t* used_r = smem_bits;
    uint32_t* used_c = smem_bits + ((m + 31) >> 5);
    const int tid = threadIdx.x;
    for (int64_t q = tid; q < ((m + 31) >> 5) + ((n + 31) >> 5); q += blockDim.x) smem_bits[q] = 0u;
    __syncthreads();

    const double eps2 = __dmul_rn(eps, eps);
    double S2 = 0.0;
    double margin = INFINITY;
    int k = 0;
    int64_t istar = 0;
    int64_t n_used_r = 0;
    int probe_q = 0;
    while (true) {
        // (a) row residual r_j = X(i*,j) - sum_{l<k} U[i*,l] V[j,l] into V slot k
        if (tid < k) s_urow[tid] = U[(int64_t)tid * m + istar];
        __syncthreads();
        double* r = V + (int64_t)k * n;
        ArgMax am{-1.0, INT64_MAX};
        for (int64_t j = tid; j < n; j += blockDim.x) {
            double x = vf_entry(g, r0 + istar, c0 + j, err);
            for (int l = 0; l < k; ++l) x = __dsub_rn(x, __dmul_rn(s_urow[l], V[(int64_t)l * n + j]));
            r[j] = x;
            if (!bit_get(used_c, j)) am = better(am, ArgMax{fabs(x), j});
        }
        // (b) j* = argmax over unused columns, lowest index on ties
        am = cta_argmax(am, s_am);
        const int64_t jstar = am.i;
        const double delta = (am.v >= 0.0) ? r[jstar] : 0.0;  // r visible: cta_argmax synced
        if (delta == 0.0) {  // (c)
            __syncthreads();
            if (tid == 0) used_r[istar >> 5] |= 1u << (istar & 31);
            __syncthreads();
            ++n_used_r;
            if (n_used_r >= m) break;
            int64_t nxt = 0;
            while (bit_get(used_r, nxt)) ++nxt;  // smallest unused row
            istar = nxt;
            continue;
        }
        // (d) v = r / delta ; (e) column residual u_i into U slot k
        if (tid < k) s_vcol[tid] = V[(int64_t)tid * n + jstar];
        __syncthreads();
        double* u = U + (int64_t)k * m;
        double part[2] = {0.0, 0.0};  // nu2, nv2
        for (int64_t j = tid; j < n; j += blockDim.x) {
            const double v = __ddiv_rn(r[j], delta);
            r[j] = v;
            part[1] += v * v;
        }
        ArgMax ai{-1.0, INT64_MAX};
        for (int64_t i = tid; i < m; i += blockDim.x) {
            double x = vf_entry(g, r0 + i, c0 + jstar, err);
            for (int l = 0; l < k; ++l) x = __dsub_rn(x, __dmul_rn(U[(int64_t)l * m + i], s_vcol[l]));
            u[i] = x;
            part[0] += x * x;
            if (!bit_get(used_r, i) && i != istar) ai = better(ai, ArgMax{fabs(x), i});
        }
        // (f) nu2, nv2 and X = sum_l (u.U_l)(v.V_l), reduced 8 values at a time
        cta_sum<2>(part, s_red);
        const double nu2 = part[0], nv2 = part[1];
        for (int l0 = 0; l0 < k; l0 += 4) {
            double d[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            for (int64_t i = tid; i < m; i += blockDim.x) {
                const double ui = u[i];
                for (int q = 0; q < 4 && l0 + q < k; ++q) d[q] += ui * U[(int64_t)(l0 + q) * m + i];
            }
            for (int64_t j = tid; j < n; j += blockDim.x) {
                const double vj = r[j];
                for (int q = 0; q < 4 && l0 + q < k; ++q) d[4 + q] += vj * V[(int64_t)(l0 + q) * n + j];
            }
            cta_sum<8>(d, s_red);
            if (tid == 0)
                for (int q = 0; q < 4 && l0 + q < k; ++q) { s_xu[l0 + q] = d[q]; s_xv[l0 + q] = d[4 + q]; }
        }
        __syncthreads();
        double X2 = 0.0;
        for (int l = 0; l < k; ++l) X2 += s_xu[l] * s_xv[l];
        const double S2n = (S2 + nu2 * nv2) + 2.0 * X2;
        const double lhs = nu2 * nv2, rhs = eps2 * S2n;
        if (rhs > 0.0) margin = fmin(margin, fabs(lhs / rhs - 1.0));
        if (lhs <= rhs) {  // (g) stop, discard this cross
            if (probe_q < probes) {
                // R30: before stopping, probe the smallest unused row at or after m (q+1)/(probes+1)
                // (wrapping to the smallest unused row) as the next pivot row
                const int64_t pos = (m * (probe_q + 1)) / (probes + 1);
                ++probe_q;
                __syncthreads();
                if (tid == 0) {
                    int64_t p = -1, first = -1;
                    for (int64_t i = 0; i < m; ++i) {
                        if (bit_get(used_r, i)) continue;
                        if (first < 0) first = i;
                        if (i >= pos) { p = i; break; }
                    }
                    s_probe = p >= 0 ? p : first;
                }
                __syncthreads();
                if (s_probe < 0) break;
                istar = s_probe;
                __syncthreads();
                continue;
            }
            break;
        }
        // (h) append
        ++k;
        S2 = S2n;
        __syncthreads();
        if (tid == 0) {
            if (!bit_get(used_r, istar)) { used_r[istar >> 5] |= 1u << (istar & 31); }
            used_c[jstar >> 5] |= 1u << (jstar & 31);
        }
        __syncthreads();
        ++n_used_r;
        if (k >= kcap) break;        // (i) k (m+n) >= m n or the rank cap -> stored dense
        if (n_used_r >= m) break;
        // (j) i* = argmax over unused rows of |u_i|
        ai = cta_argmax(ai, s_am);
        istar = ai.i;
        __syncthreads();
    }
    if (tid == 0) {
        rank_out[b] = k;
        margin_out[b] = margin;
    }
}

__global__ void fill_kernel(const double* __restrict__ geo, int64_t ntot, const int64_t* __restrict__ tasks,
                            double* __restrict__ arena, int32_t* err, const double* __restrict__ quad) {
    const int64_t* t = tasks + 6 * blockIdx.x;
    const int64_t dst = t[0], r0 = t[1], rows = t[2], c0 = t[3], cols = t[4], dld = t[5];
    const GeoView g(geo, ntot, quad);
    for (int64_t e = threadIdx.x; e < rows * cols; e += blockDim.x) {
        const int64_t i = e % rows, j = e / rows;  // column-major slice
        arena[dst + j * dld + i] = vf_entry(g, r0 + i, c0 + j, err);
    }
}

__global__ void pack_kernel(const int64_t* __restrict__ tasks, double* __restrict__ arena) {
    const int64_t* t = tasks + 7 * blockIdx.x;
    const int64_t dst = t[0];
    const double* src = reinterpret_cast<const double*>(t[1]);
    const int64_t rows = t[2], cols = t[3], rs = t[4], cs = t[5], dld = t[6];
    for (int64_t e = threadIdx.x; e < rows * cols; e += blockDim.x) {
        const int64_t i = e % rows, j = e / rows;
        arena[dst + j * dld + i] = src[i * rs + j * cs];
    }
}

__global__ void scale_rows_kernel(const int64_t* __restrict__ tasks, double* __restrict__ arena,
                                  const double* __restrict__ cdiv) {
    const int64_t* t = tasks + 5 * blockIdx.x;
    const int64_t a_off = t[0], ld = t[1], m = t[2], ncols = t[3], r0 = t[4];
    for (int64_t e = threadIdx.x; e < m * ncols; e += blockDim.x) {
        const int64_t i = e % m, j = e / m;
        arena[a_off + j * ld + i] = arena[a_off + j * ld + i] / cdiv[r0 + i];
    }
}

}  // namespace

namespace k {

void aca_batch(const double* geo, int64_t n, const int64_t* blk, const int64_t* uoff, const int64_t* voff, int probes,
               const int32_t* kcap, int nb, double eps, double* scratch, int32_t* rank_out, double* margin_out,
               int32_t* err, cudaStream_t s, int64_t max_m, int64_t max_n, const double* quad) {
    if (nb == 0) return;
    const size_t smem = sizeof(uint32_t) * (size_t)(((max_m + 31) >> 5) + ((max_n + 31) >> 5));
    if (smem > 48 * 1024)
        HM_CUDA(cudaFuncSetAttribute(aca_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    aca_kernel<<<nb, kAcaThreads, smem, s>>>(geo, n, blk, uoff, voff, kcap, eps, scratch, rank_out, margin_out,
                                             err, probes, quad);
    HM_CUDA(cudaGetLastError());
    debug_sync(s, "aca_kernel");
}

void fill_entries(const double* geo, int64_t n, const int64_t* tasks, int nt, double* arena, int32_t* err,
                  cudaStream_t s, const double* quad) {
    if (nt == 0) return;
    fill_kernel<<<nt, 256, 0, s>>>(geo, n, tasks, arena, err, quad);
    HM_CUDA(cudaGetLastError());
    debug_sync(s, "fill_kernel");
}

void pack(const int64_t* tasks, int nt, double* arena, cudaStream_t s) {
    if (nt == 0) return;
    pack_kernel<<<nt, 256, 0, s>>>(tasks, arena);
    HM_CUDA(cudaGetLastError());
    debug_sync(s, "pack_kernel");
}

void scale_rows(const int64_t* tasks, int nt, double* arena, const double* cdiv, cudaStream_t s) {
    if (nt == 0) return;
    scale_rows_kernel<<<nt, 256, 0, s>>>(tasks, arena, cdiv);
    HM_CUDA(cudaGetLastError());
    debug_sync(s, "scale_rows");
}

}  // namespace k
}  // namespace hm
