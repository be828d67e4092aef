// C ABI of include/hm.h: context, geometry/trees, ACA assembly, hot-path entry points.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>

#include "hla.h"
#include "hm_internal.h"

namespace hm {

double now_seconds() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e == cudaSuccess) return;
    const char* base = strrchr(file, '/');
    std::string msg = std::string(cudaGetErrorString(e)) + " in " + what + " (" + (base ? base + 1 : file) + ":" +
                      std::to_string(line) + ")";
    if (e == cudaErrorMemoryAllocation) throw Error(HM_ERR_OOM, msg);
    throw Error(HM_ERR_CUDA, msg);
}

static bool g_debug = false;
void debug_sync(cudaStream_t s, const char* what) {
    if (!g_debug) return;
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) throw Error(HM_ERR_CUDA, std::string("kernel fault after ") + what + ": " + cudaGetErrorString(e));
}

void* dmalloc(Ctx* ctx, size_t bytes, const char* what) {
    void* p = nullptr;
    if (ctx && ctx->alloc_fn) {
        p = ctx->alloc_fn(bytes, ctx->stream, ctx->alloc_user);
        if (!p) throw Error(HM_ERR_OOM, std::string("allocator hook failed: ") + std::to_string(bytes) + " bytes for " + what);
        return p;
    }
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw Error(HM_ERR_OOM, std::string("cudaMalloc of ") + std::to_string(bytes) + " bytes for " + what + ": " +
                                    cudaGetErrorString(e));
    }
    return p;
}

void dfree(Ctx* ctx, void* p) {
    if (!p) return;
    if (ctx && ctx->free_fn) {
        ctx->free_fn(p, ctx->stream, ctx->alloc_user);
        return;
    }
    cudaFree(p);
}

// implemented in hlu.cpp
void factor_hlu(HLU& L, const double* emissivity);

// Reading R35: the adaptive-quadrature table, internal order -- per facet the points of
// the 3-point degree-2 rule, of Dunavant's 6-point degree-4 rule and of that rule on the 4 midpoint
// sub-triangles (v0, m01, m20), (m01, v1, m12), (m20, m12, v2), (m12, m20, m01), each point
// x = (b0 v0 + b1 v1) + b2 v2 (no contraction: the oracle forms the same doubles), then the squared
// longest edge.  vertices_ext: n x 9, external order.
std::vector<double> quad_table(const Geom& g, const double* V) {
    const int64_t n = g.n;
    std::vector<double> Q((size_t)n * kQStride, 0.0);
    const double t = 2.0 / 3.0, u = 1.0 / 6.0;
    const double b3[3][3] = {{t, u, u}, {u, t, u}, {u, u, t}};
    const double A = 0.445948490915965, B = 0.108103018168070, Cc = 0.091576213509771, D = 0.816847572980459;
    const double b6[6][3] = {{B, A, A}, {A, B, A}, {A, A, B}, {D, Cc, Cc}, {Cc, D, Cc}, {Cc, Cc, D}};
    for (int64_t i = 0; i < n; ++i) {
        const double* v0 = V + 9 * (int64_t)g.perm[i];
        const double* v1 = v0 + 3;
        const double* v2 = v0 + 6;
        double* row = Q.data() + i * kQStride;
        int k = 0;
        auto put = [&](const double* b, const double* p0, const double* p1, const double* p2) {
            for (int c = 0; c < 3; ++c) row[3 * k + c] = (b[0] * p0[c] + b[1] * p1[c]) + b[2] * p2[c];
            ++k;
        };
        for (int p = 0; p < 3; ++p) put(b3[p], v0, v1, v2);
        for (int p = 0; p < 6; ++p) put(b6[p], v0, v1, v2);
        double m01[3], m12[3], m20[3];
        for (int c = 0; c < 3; ++c) {
            m01[c] = (v0[c] + v1[c]) * 0.5;
            m12[c] = (v1[c] + v2[c]) * 0.5;
            m20[c] = (v2[c] + v0[c]) * 0.5;
        }
        const double* sub[4][3] = {{v0, m01, m20}, {m01, v1, m12}, {m20, m12, v2}, {m12, m20, m01}};
        for (int q = 0; q < 4; ++q)
            for (int p = 0; p < 6; ++p) put(b6[p], sub[q][0], sub[q][1], sub[q][2]);
        double h2 = 0.0;
        const double* ed[3][2] = {{v0, v1}, {v1, v2}, {v2, v0}};
        for (int e = 0; e < 3; ++e) {
            const double ex = ed[e][1][0] - ed[e][0][0], ey = ed[e][1][1] - ed[e][0][1], ez = ed[e][1][2] - ed[e][0][2];
            const double l2 = (ex * ex + ey * ey) + ez * ez;
            h2 = e == 0 ? l2 : std::max(h2, l2);
        }
        row[kQH2] = h2;
    }
    return Q;
}

}  // namespace hm

using namespace hm;

namespace {

template <class F>
hm_status guarded(Ctx* ctx, F&& f) {
    try {
        f();
        return HM_OK;
    } catch (const Error& e) {
        if (ctx) ctx->last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        if (ctx) ctx->last_error = "host allocation failed";
        return HM_ERR_OOM;
    } catch (const std::exception& e) {
        if (ctx) ctx->last_error = e.what();
        return HM_ERR_CUDA;
    }
}

bool is_device_ptr(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Output target of a hot-path call: device memory as is; pinned host memory through its device alias,
// so the kernels' emits write it directly (no staging buffer, no device-to-host copy after the
// program); pageable host memory through a staging buffer and a copy.  kind: 0 device, 1 pinned host,
// 2 staged.
double* out_target(Ctx* ctx, DBuf<double>& stage, double* p, size_t count, int& kind) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        a.type = cudaMemoryTypeUnregistered;
    }
    if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) {
        kind = 0;
        return p;
    }
    if (a.type == cudaMemoryTypeHost && a.devicePointer) {
        kind = 1;
        return static_cast<double*>(a.devicePointer);
    }
    kind = 2;
    if (stage.n < count) stage.alloc(ctx, count, "host staging (out)");
    return stage.p;
}

// Device alias of a pinned host input (nullptr for device, managed or pageable memory).
const double* pinned_alias(const double* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return a.type == cudaMemoryTypeHost ? static_cast<const double*>(a.devicePointer) : nullptr;
}

// Stage host arrays through device buffers; returns the device pointer to use.
const double* stage_in(Ctx* ctx, DBuf<double>& buf, const double* p, size_t count, cudaStream_t s, bool& host) {
    host = !is_device_ptr(p);
    if (!host) return p;
    if (buf.n < count) buf.alloc(ctx, count, "host staging (in)");
    HM_CUDA(cudaMemcpyAsync(buf.p, p, count * sizeof(double), cudaMemcpyHostToDevice, s));
    return buf.p;
}

}  // namespace

// ============================================================================ lifetime
extern "C" {

const char* hm_status_string(hm_status s) {
    switch (s) {
        case HM_OK: return "ok";
        case HM_ERR_INVALID_ARG: return "invalid argument";
        case HM_ERR_CUDA: return "CUDA error";
        case HM_ERR_OOM: return "out of device memory";
        case HM_ERR_NCCL: return "NCCL error";
        case HM_ERR_DEGENERATE_GEOMETRY: return "degenerate geometry";
        case HM_ERR_SINGULAR: return "singular leaf block";
        case HM_ERR_NOT_READY: return "not ready";
        case HM_ERR_UNSUPPORTED: return "unsupported configuration";
    }
    return "unknown status";
}

const char* hm_last_error(const hm_ctx* ctx) { return ctx ? ctx->c.last_error.c_str() : "null context"; }

hm_status hm_init(int device, int rank, int world, const void* comm_id, uint32_t flags, hm_ctx** out) {
    if (!out) return HM_ERR_INVALID_ARG;
    *out = nullptr;
    if (world < 1 || (world & (world - 1)) || rank < 0 || rank >= world) return HM_ERR_INVALID_ARG;
    auto* c = new hm_ctx;
    c->c.device = device;
    c->c.rank = rank;
    c->c.world = world;
    c->c.flags = flags;
    c->c.host_only = device < 0;
    const char* dbg = getenv("HM_DEBUG");
    g_debug = c->c.debug = dbg && dbg[0] == '1';
    if (c->c.host_only) {   // trees and shard plans only: no CUDA, no exchange
        *out = c;
        return HM_OK;
    }
    int cnt = 0;
    if (cudaGetDeviceCount(&cnt) != cudaSuccess || cnt == 0 || device >= cnt) {
        cudaGetLastError();
        delete c;
        return HM_ERR_CUDA;
    }
    hm_status st = guarded(&c->c, [&] {
        HM_CUDA(cudaSetDevice(device));
        HM_CUDA(cudaStreamCreateWithFlags(&c->c.stream, cudaStreamNonBlocking));
        c->c.ex = make_exchanger(device, rank, world, comm_id, flags).release();
    });
    if (st != HM_OK) {
        if (c->c.stream) cudaStreamDestroy(c->c.stream);
        delete c;
        return st;
    }
    *out = c;
    return HM_OK;
}

void hm_finalize(hm_ctx* ctx) {
    if (!ctx) return;
    delete ctx->c.ex;
    if (ctx->c.stream) cudaStreamDestroy(ctx->c.stream);
    delete ctx;
}

hm_status hm_set_flags(hm_ctx* ctx, uint32_t flags) {
    if (!ctx || (flags & ~HM_FLAG_ASYNC_PINNED)) return HM_ERR_INVALID_ARG;   // only the call-mode flag changes
    ctx->c.flags = (ctx->c.flags & ~HM_FLAG_ASYNC_PINNED) | flags;
    return HM_OK;
}

hm_status hm_set_allocator(hm_ctx* ctx, void* (*alloc_fn)(size_t, void*, void*), void (*free_fn)(void*, void*, void*),
                           void* user) {
    if (!ctx || (!alloc_fn) != (!free_fn)) return HM_ERR_INVALID_ARG;
    ctx->c.alloc_fn = alloc_fn;
    ctx->c.free_fn = free_fn;
    ctx->c.alloc_user = user;
    return HM_OK;
}

// ============================================================================ geometry
hm_status hm_build_geometry(hm_ctx* ctx, int64_t n, const double* xyz, const double* nrm, const double* area,
                            const double* facet_aabb, const hm_tree_params* params, hm_geom** out) {
    if (!ctx || !out) return HM_ERR_INVALID_ARG;
    *out = nullptr;
    Ctx* c = &ctx->c;
    return guarded(c, [&] {
        if (n < 1 || n >= INT32_MAX / 2 || !xyz || !nrm || !area || !params)
            throw Error(HM_ERR_INVALID_ARG, "hm_build_geometry: need n >= 1 and non-null xyz, nrm, area, params");
        if (params->n_min < 1 || params->n_min > 256)
            throw Error(HM_ERR_INVALID_ARG, "hm_build_geometry: n_min must be in [1, 256]");
        if (!(params->eta > 0.0) || !std::isfinite(params->eta))
            throw Error(HM_ERR_INVALID_ARG, "hm_build_geometry: eta must be finite and > 0");
        if (params->adm_mode != 0 && params->adm_mode != 1)
            throw Error(HM_ERR_INVALID_ARG, "hm_build_geometry: adm_mode must be 0 or 1");
        if (params->adm_mode == 1 && !facet_aabb)
            throw Error(HM_ERR_INVALID_ARG, "hm_build_geometry: adm_mode 1 needs facet_aabb");
        for (int64_t i = 0; i < n; ++i) {
            for (int k = 0; k < 3; ++k)
                if (!std::isfinite(xyz[3 * i + k]) || !std::isfinite(nrm[3 * i + k]))
                    throw Error(HM_ERR_DEGENERATE_GEOMETRY, "non-finite coordinate or normal at facet " + std::to_string(i));
            if (!(area[i] > 0.0) || !std::isfinite(area[i]))
                throw Error(HM_ERR_DEGENERATE_GEOMETRY, "area <= 0 or non-finite at facet " + std::to_string(i));
            const double l2 = nrm[3 * i] * nrm[3 * i] + nrm[3 * i + 1] * nrm[3 * i + 1] + nrm[3 * i + 2] * nrm[3 * i + 2];
            if (std::fabs(l2 - 1.0) > 1e-6)
                throw Error(HM_ERR_INVALID_ARG, "normal of facet " + std::to_string(i) + " is not unit length");
        }
        auto* G = new hm_geom;
        std::unique_ptr<hm_geom> guard(G);
        Geom& g = G->g;
        g.ctx = c;
        g.n = n;
        g.params = *params;
        const double t0 = now_seconds();
        build_trees(g, xyz, nrm, area, facet_aabb);
        make_shard(g, c->rank, c->world);
        if (c->host_only) {
            g.setup_seconds = now_seconds() - t0;
            *out = guard.release();
            return;
        }
        std::vector<double> soa(7 * (size_t)n);
        std::copy(g.cx.begin(), g.cx.end(), soa.begin());
        std::copy(g.cy.begin(), g.cy.end(), soa.begin() + n);
        std::copy(g.cz.begin(), g.cz.end(), soa.begin() + 2 * n);
        std::copy(g.nx.begin(), g.nx.end(), soa.begin() + 3 * n);
        std::copy(g.ny.begin(), g.ny.end(), soa.begin() + 4 * n);
        std::copy(g.nz.begin(), g.nz.end(), soa.begin() + 5 * n);
        std::copy(g.area.begin(), g.area.end(), soa.begin() + 6 * n);
        g.d_geo.upload(c, soa, "facet data", c->stream);
        g.d_perm.upload(c, g.perm, "permutation", c->stream);
        HM_CUDA(cudaStreamSynchronize(c->stream));
        g.setup_seconds = now_seconds() - t0;
        *out = guard.release();
    });
}

void hm_destroy_geom(hm_geom* g) { delete g; }

hm_status hm_export_perm(const hm_geom* geom, int32_t* perm) {
    if (!geom || !perm) return HM_ERR_INVALID_ARG;
    std::copy(geom->g.perm.begin(), geom->g.perm.end(), perm);
    return HM_OK;
}

hm_status hm_export_partition(const hm_geom* geom, const hm_hmat* F, int64_t* n_blocks, int64_t* rows) {
    if (!geom || !n_blocks) return HM_ERR_INVALID_ARG;
    const Geom& g = geom->g;
    *n_blocks = (int64_t)g.blocks.size();
    if (!rows) return HM_OK;
    for (size_t b = 0; b < g.blocks.size(); ++b) {
        const Blk& B = g.blocks[b];
        int64_t* r = rows + 8 * b;
        r[0] = B.level; r[1] = B.r0; r[2] = B.r1; r[3] = B.c0; r[4] = B.c1; r[5] = B.adm;
        r[6] = F ? F->h.blk_kind[b] : (B.adm ? 1 : 0);
        r[7] = F ? F->h.blk_rank[b] : 0;
    }
    return HM_OK;
}

hm_status hm_local_range(const hm_geom* geom, int rank, int world, int64_t* begin, int64_t* end) {
    if (!geom || !begin || !end || world < 1 || rank < 0 || rank >= world || (world & (world - 1)))
        return HM_ERR_INVALID_ARG;
    local_range(geom->g, rank, world, begin, end);   // node `rank` at tree level log2(world)
    return HM_OK;
}

// ============================================================================ ACA assembly
hm_status hm_assemble_aca(hm_ctx* ctx, const hm_geom* geom, const hm_aca_params* params, hm_hmat** F_out) {
    if (!ctx || !geom || !params || !F_out) return HM_ERR_INVALID_ARG;
    *F_out = nullptr;
    if (ctx->c.host_only) {
        ctx->c.last_error = "host-only context (device < 0): trees and shard plans only";
        return HM_ERR_NOT_READY;
    }
    Ctx* c = &ctx->c;
    return guarded(c, [&] {
        if (!(params->eps_aca > 0.0) || params->eps_aca >= 1.0)
            throw Error(HM_ERR_INVALID_ARG, "eps_aca must be in (0, 1)");
        if (params->k_max < 0 || params->k_max > 64) throw Error(HM_ERR_INVALID_ARG, "k_max must be in [0, 64]");
        if (params->probes < 0 || params->probes > 16) throw Error(HM_ERR_INVALID_ARG, "probes must be in [0, 16]");
        if (params->pivoting != 0 && params->pivoting != 1) throw Error(HM_ERR_INVALID_ARG, "pivoting must be 0 or 1");
        if (params->recompress != 0 && params->recompress != 1) throw Error(HM_ERR_INVALID_ARG, "recompress must be 0 or 1");
        if (params->quadrature != 0 && params->quadrature != 1) throw Error(HM_ERR_INVALID_ARG, "quadrature must be 0 or 1");
        if (params->quadrature == 1 && !params->vertices)
            throw Error(HM_ERR_INVALID_ARG, "quadrature = 1 (adaptive) needs the facets' triangle vertices");
        const Geom& g = geom->g;
        const cudaStream_t s = c->stream;
        const int64_t n = g.n;
        auto* H = new hm_hmat;
        std::unique_ptr<hm_hmat> guard(H);
        HMat& F = H->h;
        F.ctx = c;
        F.geom = &g;
        F.params = *params;
        F.params.vertices = nullptr;   // the caller's array is read during this call only
        DBuf<double> dquad;            // reading R35 table (assembly only)
        if (params->quadrature == 1) dquad.upload(c, quad_table(g, params->vertices), "quadrature table", s);
        const double* quad = dquad.p;
        const int KMAX = params->k_max > 0 ? params->k_max : 48;
        const size_t nb = g.blocks.size();
        F.blk_kind.assign(nb, KIND_DENSE);
        F.blk_rank.assign(nb, 0);

        // ---- batched partial-pivot ACA over admissible blocks (scratch bounded per batch)
        double t0 = now_seconds();
        struct AcaRec { int batch; int64_t uoff, voff; int kcap; };
        std::vector<AcaRec> rec(nb, AcaRec{-1, 0, 0, 0});
        std::vector<DBuf<double>> batches;
        const int64_t budget = int64_t(1) << 28;  // doubles of scratch per batch (2 GiB)
        DBuf<int32_t> err;
        err.alloc(c, 4, "err");
        HM_CUDA(cudaMemsetAsync(err.p, 0, 4 * sizeof(int32_t), s));
        size_t b = 0;
        while (params->pivoting == 1 && b < nb) {
            // full pivoting (the paper's ACA variant, NEXT-3): evaluate the admissible
            // blocks of a batch densely (row-major X[i][j] = F(r0+i, c0+j), filled through the bitwise
            // symmetry of the unscaled entry, reading R3), then cross approximation with full pivoting
            // and the exact Frobenius residual as stop test (eq:erel): ||X - U V^T||_F <= eps ||X||_F
            std::vector<int64_t> hblk, hfill;
            std::vector<int32_t> hkcap;
            std::vector<size_t> ids;
            int64_t cur = 0, fac = 0;
            for (; b < nb; ++b) {
                const Blk& B = g.blocks[b];
                if (!B.adm) continue;
                const int64_t m = B.r1 - B.r0, nn = B.c1 - B.c0;
                const int64_t klim = (m * nn + m + nn - 1) / (m + nn);
                const int kc = (int)std::min<int64_t>(KMAX, klim);
                const int64_t need = m * nn + ((m * kc + 1) & ~1LL) + ((nn * kc + 1) & ~1LL);
                if (!ids.empty() && (cur + fac + need > budget || ids.size() >= 1000000)) break;
                hfill.insert(hfill.end(), {cur, B.c0, nn, B.r0, m, nn});   // X^T column-major = X row-major
                hblk.insert(hblk.end(), {0, m, cur, nn, 0, 0, nn});        // X = T + cur, row stride nn
                hkcap.push_back(kc);
                ids.push_back(b);
                cur += m * nn;
                fac += ((m * kc + 1) & ~1LL) + ((nn * kc + 1) & ~1LL);
            }
            if (ids.empty()) break;
            int64_t fo = 0;
            for (size_t q = 0; q < ids.size(); ++q) {   // factor slots after the dense blocks
                const Blk& B = g.blocks[ids[q]];
                const int64_t m = B.r1 - B.r0, nn = B.c1 - B.c0, kc = hkcap[q];
                hblk[7 * q + 4] = cur + fo;
                fo += (m * kc + 1) & ~1LL;
                hblk[7 * q + 5] = cur + fo;
                fo += (nn * kc + 1) & ~1LL;
            }
            DBuf<double> scratch;
            scratch.alloc(c, (size_t)std::max<int64_t>(cur + fo, 2), "full-pivot ACA scratch");
            DBuf<int64_t> dfill, dblk;
            DBuf<int32_t> dkcap, drank;
            dfill.upload(c, hfill, "fp-aca fill", s);
            dblk.upload(c, hblk, "fp-aca blocks", s);
            dkcap.upload(c, hkcap, "fp-aca kcap", s);
            drank.alloc(c, ids.size(), "fp-aca ranks");
            k::fill_entries(g.d_geo.p, n, dfill.p, (int)ids.size(), scratch.p, err.p, s, quad);
            k::cpaca_batch(scratch.p, 1, dblk.p, dkcap.p, (int)ids.size(), params->eps_aca, scratch.p, drank.p, s);
            std::vector<int32_t> hrank(ids.size());
            HM_CUDA(cudaMemcpyAsync(hrank.data(), drank.p, ids.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
            HM_CUDA(cudaStreamSynchronize(s));
            std::vector<int64_t> ctasks;
            int64_t ctot = 0;
            for (size_t q = 0; q < ids.size(); ++q) {
                const size_t bb = ids[q];
                const Blk& B = g.blocks[bb];
                const int64_t m = B.r1 - B.r0, nn = B.c1 - B.c0;
                const int kq = hrank[q];
                F.blk_rank[bb] = kq < 0 ? hkcap[q] : kq;
                F.blk_kind[bb] = kq < 0 ? KIND_ADM_DENSE : KIND_LR;
                if (F.blk_kind[bb] != KIND_LR) continue;
                const int64_t uo = ctot, vo = ctot + ((m * kq + 1) & ~1LL);
                ctot = vo + ((nn * kq + 1) & ~1LL);
                if (kq > 0) {
                    ctasks.insert(ctasks.end(), {uo, (int64_t)(uintptr_t)(scratch.p + hblk[7 * q + 4]), m * kq, 1, 1, 0, m * kq});
                    ctasks.insert(ctasks.end(), {vo, (int64_t)(uintptr_t)(scratch.p + hblk[7 * q + 5]), nn * kq, 1, 1, 0, nn * kq});
                }
                rec[bb] = AcaRec{(int)batches.size(), uo, vo, hkcap[q]};
            }
            DBuf<double> compact;
            compact.alloc(c, (size_t)std::max<int64_t>(ctot, 2), "ACA factors");
            if (!ctasks.empty()) {
                DBuf<int64_t> dct;
                dct.upload(c, ctasks, "compaction tasks", s);
                k::pack(dct.p, (int)(ctasks.size() / 7), compact.p, s);
                HM_CUDA(cudaStreamSynchronize(s));
            }
            scratch.reset();
            batches.push_back(std::move(compact));
        }
        while (params->pivoting == 0 && b < nb) {
            std::vector<int64_t> hblk, huoff, hvoff;
            std::vector<int32_t> hkcap;
            std::vector<size_t> ids;
            int64_t cur = 0, max_m = 1, max_n = 1;
            for (; b < nb; ++b) {
                const Blk& B = g.blocks[b];
                if (!B.adm) continue;
                const int64_t m = B.r1 - B.r0, nn = B.c1 - B.c0;
                const int64_t klim = (m * nn + m + nn - 1) / (m + nn);  // smallest k with k(m+n) >= mn
                const int kc = (int)std::min<int64_t>(KMAX, klim);
                const int64_t need = ((m * kc + 1) & ~1LL) + ((nn * kc + 1) & ~1LL);
                if (!ids.empty() && (cur + need > budget || ids.size() >= 1000000)) break;
                hblk.insert(hblk.end(), {B.r0, m, B.c0, nn});
                huoff.push_back(cur);
                cur += (m * kc + 1) & ~1LL;
                hvoff.push_back(cur);
                cur += (nn * kc + 1) & ~1LL;
                hkcap.push_back(kc);
                ids.push_back(b);
                max_m = std::max(max_m, m);
                max_n = std::max(max_n, nn);
            }
            if (ids.empty()) break;
            DBuf<int64_t> dblk, duoff, dvoff;
            DBuf<int32_t> dkcap, drank;
            DBuf<double> dmargin, scratch;
            dblk.upload(c, hblk, "aca blocks", s);
            duoff.upload(c, huoff, "aca uoff", s);
            dvoff.upload(c, hvoff, "aca voff", s);
            dkcap.upload(c, hkcap, "aca kcap", s);
            drank.alloc(c, ids.size(), "aca ranks");
            dmargin.alloc(c, ids.size(), "aca margins");
            scratch.alloc(c, (size_t)std::max<int64_t>(cur, 2), "aca scratch");
            k::aca_batch(g.d_geo.p, n, dblk.p, duoff.p, dvoff.p, params->probes, dkcap.p, (int)ids.size(), params->eps_aca, scratch.p,
                         drank.p, dmargin.p, err.p, s, max_m, max_n, quad);
            std::vector<int32_t> hrank(ids.size());
            HM_CUDA(cudaMemcpyAsync(hrank.data(), drank.p, ids.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
            HM_CUDA(cudaStreamSynchronize(s));
            // compact the batch: keep only the first k columns of U and V of the low-rank blocks
            // (scratch is sized for the rank cap; stored factors are a small fraction of it)
            std::vector<int64_t> ctasks;
            int64_t ctot = 0;
            for (size_t q = 0; q < ids.size(); ++q) {
                const size_t bb = ids[q];
                const Blk& B = g.blocks[bb];
                const int64_t m = B.r1 - B.r0, nn = B.c1 - B.c0, kq = hrank[q];
                F.blk_rank[bb] = hrank[q];
                F.blk_kind[bb] = hrank[q] >= hkcap[q] ? KIND_ADM_DENSE : KIND_LR;
                if (F.blk_kind[bb] != KIND_LR) continue;
                const int64_t uo = ctot, vo = ctot + ((m * kq + 1) & ~1LL);
                ctot = vo + ((nn * kq + 1) & ~1LL);
                if (kq > 0) {
                    ctasks.insert(ctasks.end(), {uo, (int64_t)(uintptr_t)(scratch.p + huoff[q]), m * kq, 1, 1, 0, m * kq});
                    ctasks.insert(ctasks.end(), {vo, (int64_t)(uintptr_t)(scratch.p + hvoff[q]), nn * kq, 1, 1, 0, nn * kq});
                }
                rec[bb] = AcaRec{(int)batches.size(), uo, vo, hkcap[q]};
            }
            DBuf<double> compact;
            compact.alloc(c, (size_t)std::max<int64_t>(ctot, 2), "ACA factors");
            if (!ctasks.empty()) {
                DBuf<int64_t> dct;
                dct.upload(c, ctasks, "compaction tasks", s);
                k::pack(dct.p, (int)(ctasks.size() / 7), compact.p, s);
                HM_CUDA(cudaStreamSynchronize(s));
            }
            scratch.reset();
            batches.push_back(std::move(compact));
        }
        // ---- optional recompression of the low-rank factors (reading R32): per batch, in place
        if (params->recompress) {
            for (size_t bi = 0; bi < batches.size(); ++bi) {
                std::vector<int64_t> hb;
                std::vector<size_t> ids;
                for (size_t q = 0; q < nb; ++q) {
                    if (F.blk_kind[q] != KIND_LR || rec[q].batch != (int)bi || F.blk_rank[q] < 2) continue;
                    const Blk& B = g.blocks[q];
                    hb.insert(hb.end(), {rec[q].uoff, B.r1 - B.r0, rec[q].voff, B.c1 - B.c0, (int64_t)F.blk_rank[q]});
                    ids.push_back(q);
                }
                if (ids.empty()) continue;
                DBuf<int64_t> dblk;
                DBuf<int32_t> drank;
                dblk.upload(c, hb, "recompression blocks", s);
                drank.alloc(c, ids.size(), "recompressed ranks");
                for (size_t q0 = 0; q0 < ids.size(); q0 += 1000000)
                    k::recompress_batch(batches[bi].p, dblk.p + 5 * q0, (int)std::min<size_t>(1000000, ids.size() - q0),
                                        params->eps_aca, drank.p + q0, s);
                std::vector<int32_t> hr(ids.size());
                HM_CUDA(cudaMemcpyAsync(hr.data(), drank.p, ids.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
                HM_CUDA(cudaStreamSynchronize(s));
                for (size_t q = 0; q < ids.size(); ++q) F.blk_rank[ids[q]] = hr[q];
            }
        }
        int32_t herr[4];
        HM_CUDA(cudaMemcpy(herr, err.p, sizeof(herr), cudaMemcpyDeviceToHost));
        if (herr[0])
            throw Error(HM_ERR_DEGENERATE_GEOMETRY, "coincident collocation points for facets " +
                                                        std::to_string(g.perm[herr[1]]) + "," + std::to_string(g.perm[herr[2]]));
        F.setup_seconds[0] = now_seconds() - t0;

        // ---- near field + factors into the stream layout
        t0 = now_seconds();
        std::vector<SrcBlock> src(nb);
        for (size_t q = 0; q < nb; ++q) {
            const Blk& B = g.blocks[q];
            SrcBlock& S = src[q];
            S.r0 = B.r0; S.m = B.r1 - B.r0; S.c0 = B.c0; S.n = B.c1 - B.c0;
            if (F.blk_kind[q] == KIND_LR) {
                S.kind = KIND_LR;
                S.k = F.blk_rank[q];
                const double* base = batches[rec[q].batch].p;
                S.U = base + rec[q].uoff;
                S.u_ld = S.m;
                S.V = base + rec[q].voff;
                S.v_ld = S.n;
            } else {
                S.kind = KIND_DENSE;
                S.fill_entries = true;
            }
        }
        F.op.p1_by_key = true;   // phase 1 in cluster order (row-group links of the flux program)
        build_hop(c, g, src, F.op, s, nullptr, 0, quad);
        if (g.shard.sharded()) build_hop(c, g, src, F.op_loc, s, &g.shard, 0, quad);   // this rank's block rows
        batches.clear();
        F.setup_seconds[1] = now_seconds() - t0;

        // ---- row sums s = F_H 1 / A (eq:rowsum), clamp (eq:clamped_rowsum), scaling (eqn:F_closed)
        t0 = now_seconds();
        F.xt.alloc(c, (size_t)(n + F.op.n_t), "F xt");
        F.y.alloc(c, (size_t)n, "F y");
        DBuf<double> sv, cv, cdiv;
        sv.alloc(c, n, "row sums");
        cv.alloc(c, n, "clamped row sums");
        cdiv.alloc(c, n, "row divisors");
        {   // F_H 1 with the engine (setup program, internal order)
            Program rs;
            rs.add_stream(F.op.p1, F.op, F.xt.p, F.xt.p, OUT_ASSIGN);
            rs.add_stream(F.op.p2, F.op, F.xt.p, F.y.p, OUT_ASSIGN, DEP_BARRIER, nullptr, IN_PLAIN, -1);
            rs.finalize(c, s);
            k::fill_value(F.xt.p, n, 1.0, s);
            rs.launch(ProgArgs{}, s);
            HM_CUDA(cudaStreamSynchronize(s));
        }
        k::row_sums_clamp(F.y.p, g.d_geo.p + 6 * n, sv.p, cv.p, cdiv.p, n, s);
        if (params->closed_cavity) {
            std::vector<int64_t> tasks;
            for (const Panel& pn : F.op.p2.panels) tasks.insert(tasks.end(), {pn.a_off, pn.ld, pn.nrows, pn.ncols, pn.out0});
            DBuf<int64_t> dt;
            dt.upload(c, tasks, "scale tasks", s);
            k::scale_rows(dt.p, (int)F.op.p2.panels.size(), F.op.arena.p, cdiv.p, s);
            HM_CUDA(cudaStreamSynchronize(s));
        }
        std::vector<double> hs(n), hc(n);
        HM_CUDA(cudaMemcpyAsync(hs.data(), sv.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
        HM_CUDA(cudaMemcpyAsync(hc.data(), cv.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
        HM_CUDA(cudaStreamSynchronize(s));
        if (g.shard.sharded()) {
            // the local operator: same closed-cavity scaling, rows indexed in the padded layout
            const Shard& S = g.shard;
            if (params->closed_cavity) {
                std::vector<double> cdiv_pad(S.n_pad(), 1.0);
                for (int64_t i = S.lb(); i < S.le(); ++i) cdiv_pad[S.pad(i)] = hc[i] != 0.0 ? hc[i] : 1.0;
                DBuf<double> dcp;
                dcp.upload(c, cdiv_pad, "row divisors (padded)", s);
                std::vector<int64_t> tasks;
                for (const Panel& pn : F.op_loc.p2.panels)
                    tasks.insert(tasks.end(), {pn.a_off, pn.ld, pn.nrows, pn.ncols, pn.out0});
                DBuf<int64_t> dt;
                dt.upload(c, tasks, "scale tasks (local)", s);
                if (!tasks.empty()) k::scale_rows(dt.p, (int)F.op_loc.p2.panels.size(), F.op_loc.arena.p, dcp.p, s);
                HM_CUDA(cudaStreamSynchronize(s));
            }
            F.xt_loc.alloc(c, (size_t)(S.n_pad() + F.op_loc.n_t), "F xt (local)");
            Program& P = F.sp_apply.add(F.xt_loc.p, true);
            P.n_x = S.n_pad();
            P.add_stream(F.op_loc.p1, F.op_loc, F.xt_loc.p, F.xt_loc.p, OUT_ASSIGN);
            P.add_stream(F.op_loc.p2, F.op_loc, F.xt_loc.p, nullptr, OUT_LOCAL, DEP_BARRIER, nullptr, IN_PLAIN, -1);
            F.sp_apply.finalize(c, s, &g);
            // multi-RHS (C5's sharded 64-RHS apply): allgather of the n_pad x 64 block, DMMA engine
            F.xt_loc_m.alloc(c, (size_t)(S.n_pad() + F.op_loc.n_t) * kMrhsMax, "F xt (local, multi-RHS)");
            F.sp_apply_m.mrhs = true;
            Program& Pm = F.sp_apply_m.add(F.xt_loc_m.p, true);
            Pm.mrhs = true;
            Pm.n_x = S.n_pad();
            Pm.add_stream(F.op_loc.p1m, F.op_loc, F.xt_loc_m.p, F.xt_loc_m.p, OUT_ASSIGN);
            Pm.add_stream(F.op_loc.p2m, F.op_loc, F.xt_loc_m.p, nullptr, OUT_LOCAL, DEP_BARRIER, nullptr, IN_PLAIN, -1);
            F.sp_apply_m.finalize(c, s, &g);
        }
        F.s_ext.resize(n);
        F.c_ext.resize(n);
        for (int64_t i = 0; i < n; ++i) {
            F.s_ext[g.perm[i]] = hs[i];
            F.c_ext[g.perm[i]] = hc[i];
        }
        // hot-path program: phase 1 -> phase 2, permute-in fused into the gathers, permute-out into
        // the emit
        F.prog_apply.n_x = n;
        F.prog_apply.add_stream(F.op.p1, F.op, F.xt.p, F.xt.p, OUT_ASSIGN, DEP_BARRIER, nullptr, IN_PERM);
        F.prog_apply.add_stream(F.op.p2, F.op, F.xt.p, nullptr, OUT_PERM, DEP_BARRIER, nullptr, IN_PERM, -1);
        F.prog_apply.finalize(c, s);
        {   // pinned host x: copy-in pass first; phase 1 and the x-only phase-2 pieces wait for it
            F.x_dev.alloc(c, (size_t)n, "apply x (pinned host copy-in)");
            Program& P = F.prog_apply_h;
            P.n_x = n;
            P.add_elementwise(UNIT_COPYIN, n, F.x_dev.p, copyin_rows(n));
            P.add_stream(F.op.p1, F.op, F.xt.p, F.xt.p, OUT_ASSIGN, DEP_BARRIER, nullptr, IN_PERM);
            P.add_stream(F.op.p2, F.op, F.xt.p, nullptr, OUT_PERM, DEP_BARRIER, nullptr, IN_PERM, 0);
            P.finalize(c, s);
        }
        if (!g.shard.sharded()) {   // multi-RHS program: blocks of kMrhsMax columns, DMMA engine
            F.xt_m.alloc(c, (size_t)(n + F.op.n_t) * kMrhsMax, "F xt (multi-RHS)");
            F.y_m.alloc(c, (size_t)n * kMrhsMax, "F y (multi-RHS)");
            Program& P = F.prog_apply_m;
            P.mrhs = true;
            P.n_x = n;
            P.add_elementwise(UNIT_PERMUTE, n, F.xt_m.p, elementwise_rows(n));   // x -> internal n x 64 (coalesced)
            const int xin = (int)P.h_passes.size() - 1;   // x-only phase-2 tasks wait for it (no phase 1: no LR block)
            P.add_stream(F.op.p1m, F.op, F.xt_m.p, F.xt_m.p, OUT_ASSIGN);
            // HM_MRHS_FUSED_EPI=1: phase 2 emits the permuted result itself (no epilogue pass)
            const bool fused = mrhs_fused_epilogue();
            P.add_stream(F.op.p2m, F.op, F.xt_m.p, F.y_m.p, fused ? OUT_PERM : OUT_ASSIGN, DEP_BARRIER, nullptr, IN_PLAIN, xin);
            if (!fused) P.add_elementwise(UNIT_EPILOGUE, n, nullptr, elementwise_rows(n), F.y_m.p, OUT_PERM);
            P.finalize(c, s);
        }
        HM_CUDA(cudaStreamSynchronize(s));
        F.setup_seconds[2] = now_seconds() - t0;
        *F_out = guard.release();
    });
}

void hm_destroy_hmat(hm_hmat* F) { delete F; }

hm_status hm_hmat_from_host(hm_ctx* ctx, const hm_geom* geom, const int32_t* kind, const int32_t* rank,
                            const int64_t* offset, const double* data, hm_hmat** F_out) {
    if (!ctx || !geom || !kind || !rank || !offset || !data || !F_out) return HM_ERR_INVALID_ARG;
    *F_out = nullptr;
    Ctx* c = &ctx->c;
    if (!c->host_only) {
        c->last_error = "hm_hmat_from_host: host-only contexts (device < 0) only";
        return HM_ERR_UNSUPPORTED;
    }
    return guarded(c, [&] {
        const Geom& g = geom->g;
        auto* H = new hm_hmat;
        std::unique_ptr<hm_hmat> guard(H);
        HMat& F = H->h;
        F.ctx = c;
        F.geom = &g;
        F.params = hm_aca_params{};
        const size_t nb = g.blocks.size();
        F.blk_kind.assign(nb, KIND_DENSE);
        F.blk_rank.assign(nb, 0);
        F.host_blocks.resize(nb);
        for (size_t b = 0; b < nb; ++b) {
            const Blk& B = g.blocks[b];
            const int64_t m = B.r1 - B.r0, nn = B.c1 - B.c0;
            HostBlock& Hb = F.host_blocks[b];
            const double* p = data + offset[b];
            if (kind[b] == 1) {
                if (!B.adm || rank[b] < 0 || rank[b] > std::min<int64_t>(m, nn))
                    throw Error(HM_ERR_INVALID_ARG, "block " + std::to_string(b) + ": low rank needs an admissible block and 0 <= k <= min(m, n)");
                Hb.kind = KIND_LR;
                Hb.k = rank[b];
                Hb.U.assign(p, p + m * Hb.k);
                Hb.V.assign(p + m * Hb.k, p + m * Hb.k + nn * Hb.k);
                F.blk_kind[b] = KIND_LR;
                F.blk_rank[b] = Hb.k;
            } else if (kind[b] == 0) {
                Hb.kind = KIND_DENSE;
                Hb.D.assign(p, p + m * nn);
                F.blk_kind[b] = B.adm ? KIND_ADM_DENSE : KIND_DENSE;
            } else {
                throw Error(HM_ERR_INVALID_ARG, "block " + std::to_string(b) + ": kind must be 0 or 1");
            }
        }
        *F_out = guard.release();
    });
}

hm_status hm_export_factors(const hm_hmat* Fh, const hm_hlu* LUh, int32_t op, int64_t* n_items, int64_t* n_doubles,
                            int64_t* meta, double* data) {
    if (!n_items || !n_doubles || op < 0 || (!Fh && !LUh)) return HM_ERR_INVALID_ARG;
    Ctx* c = Fh ? Fh->h.ctx : LUh->h.ctx;
    return guarded(c, [&] {
        struct Item { int64_t r0, m, c0, n, kind, k; };
        std::vector<Item> items;
        const bool fill = meta != nullptr;
        if (fill && !data) throw Error(HM_ERR_INVALID_ARG, "data is NULL");
        int64_t nd = 0;
        auto emit_meta = [&](const Item& it) {
            if (fill) {
                int64_t* r = meta + 6 * (int64_t)items.size();
                r[0] = it.r0; r[1] = it.m; r[2] = it.c0; r[3] = it.n; r[4] = it.kind; r[5] = it.k;
            }
            items.push_back(it);
        };
        if (c->host_only) {
            if (op == HM_OP_F) {
                if (!Fh || Fh->h.host_blocks.empty()) throw Error(HM_ERR_INVALID_ARG, "F holds no host blocks");
                const Geom& g = *Fh->h.geom;
                for (size_t b = 0; b < g.blocks.size(); ++b) {
                    const Blk& B = g.blocks[b];
                    const HostBlock& H = Fh->h.host_blocks[b];
                    const int64_t m = B.r1 - B.r0, nn = B.c1 - B.c0;
                    const bool lr = H.kind == KIND_LR;
                    emit_meta(Item{B.r0, m, B.c0, nn, lr ? 1 : 0, lr ? H.k : 0});
                    if (fill) {
                        if (lr) {
                            std::copy(H.U.begin(), H.U.end(), data + nd);
                            std::copy(H.V.begin(), H.V.end(), data + nd + m * H.k);
                        } else {
                            std::copy(H.D.begin(), H.D.end(), data + nd);
                        }
                    }
                    nd += lr ? H.k * (m + nn) : m * nn;
                }
            } else {
                if (!LUh || !LUh->h.host_factor) throw Error(HM_ERR_INVALID_ARG, "LU holds no host factors");
                const HLU& L = LUh->h;
                const Geom& g = *L.F->geom;
                const int Lc = L.cut_level;
                const int side_want = op == HM_OP_LINV ? 1 : op == HM_OP_UINV ? 2 : ((op - 3) % 2 == 0 ? 1 : 2);
                const int lvl_want = op >= 3 ? (op - 3) / 2 : -1;
                if (lvl_want >= Lc) throw Error(HM_ERR_INVALID_ARG, "no W blocks at that level (cut level " + std::to_string(Lc) + ")");
                L.host_factor->visit([&](const hla::LeafView& v) {
                    const hla::Mat& M = *v.M;
                    if (v.side == 0) {
                        if (lvl_want >= 0) return;
                        const int64_t m = M.m;
                        emit_meta(Item{M.r0, m, M.c0, m, 0, 0});
                        if (fill)
                            for (int64_t j = 0; j < m; ++j)
                                for (int64_t i = 0; i < m; ++i) {
                                    const double a = M.D[i + j * m];
                                    double x = 0.0;
                                    if (side_want == 1) x = i > j ? a : (i == j ? 1.0 : 0.0);
                                    else x = i <= j ? a : 0.0;
                                    data[nd + i + j * m] = x;
                                }
                        nd += m * m;
                        return;
                    }
                    if (v.side != side_want) return;
                    const int lvl = g.nodes[v.node].level;
                    if (lvl_want >= 0 ? lvl != lvl_want : lvl < Lc) return;
                    const bool lr = M.type == hla::T_LR;
                    emit_meta(Item{M.r0, M.m, M.c0, M.n, lr ? 1 : 0, lr ? M.k : 0});
                    if (fill) {
                        if (lr) {
                            std::copy(M.U.begin(), M.U.begin() + M.m * M.k, data + nd);
                            std::copy(M.V.begin(), M.V.begin() + M.n * M.k, data + nd + M.m * M.k);
                        } else {
                            std::copy(M.D.begin(), M.D.end(), data + nd);
                        }
                    }
                    nd += lr ? M.k * (M.m + M.n) : M.m * M.n;
                });
            }
        } else {
            const HOp* hop = nullptr;
            if (op == HM_OP_F) {
                if (!Fh) throw Error(HM_ERR_INVALID_ARG, "F is NULL");
                hop = &Fh->h.op;
            } else {
                if (!LUh) throw Error(HM_ERR_INVALID_ARG, "LU is NULL");
                const HLU& L = LUh->h;
                if (op == HM_OP_LINV) hop = &L.leafL;
                else if (op == HM_OP_UINV) hop = &L.leafU;
                else {
                    const int lv = (op - 3) / 2;
                    if (lv >= L.cut_level) throw Error(HM_ERR_INVALID_ARG, "no W blocks at that level");
                    hop = (op - 3) % 2 == 0 ? &L.fwd[lv] : &L.bwd[lv];
                }
            }
            int64_t tot = 0;
            std::vector<int64_t> at(hop->items.size());
            for (size_t q = 0; q < hop->items.size(); ++q) {
                const HOp::ItemRec& it = hop->items[q];
                const bool lr = it.v_off >= 0;
                emit_meta(Item{it.r0, it.m, it.c0, it.ncols, lr ? 1 : 0, lr ? it.k : 0});
                at[q] = tot;
                tot += lr ? it.k * (it.m + it.ncols) : it.m * it.ncols;
            }
            nd = tot;
            if (fill)
                read_items(c, *hop, [](size_t) { return true; }, [&](size_t q, const double* pay, const double* V) {
                    const HOp::ItemRec& it = hop->items[q];
                    const bool lr = it.v_off >= 0;
                    double* dst = data + at[q];
                    if (lr) {
                        std::copy(pay, pay + it.m * it.k, dst);
                        if (it.k > 0) std::copy(V, V + it.ncols * it.k, dst + it.m * it.k);
                    } else {
                        std::copy(pay, pay + it.m * it.ncols, dst);
                    }
                });
        }
        *n_items = (int64_t)items.size();
        *n_doubles = nd;
    });
}

hm_status hm_set_ambient(hm_ctx* ctx, hm_hlu* LUh, int32_t enable, double T_inf) {
    if (!ctx || !LUh) return HM_ERR_INVALID_ARG;
    Ctx* c = &ctx->c;
    return guarded(c, [&] {
        HLU& L = LUh->h;
        if (!enable) {
            L.ambient = false;
            return;
        }
        if (c->host_only) throw Error(HM_ERR_NOT_READY, "host-only context: no hot path");
        if (!(T_inf >= 0.0) || !std::isfinite(T_inf)) throw Error(HM_ERR_INVALID_ARG, "T_inf must be finite and >= 0");
        const HMat& F = *L.F;
        if (F.params.closed_cavity)
            throw Error(HM_ERR_INVALID_ARG, "the ambient term belongs to open cavities (PAPER.md:886-891); F was "
                                            "assembled with closed-cavity row scaling");
        const Geom& g = *F.geom;
        const int64_t n = g.n;
        std::vector<double> a(n);
        for (int64_t i = 0; i < n; ++i) a[i] = g.area[i] * (1.0 - F.c_ext[g.perm[i]]);   // A_i (1 - c_i)
        const cudaStream_t s = c->stream;
        L.amb_int.upload(c, a, "ambient A(1-c)", s);
        if (g.shard.sharded()) {
            const Shard& S = g.shard;
            std::vector<double> ap(S.n_pad(), 0.0);
            for (int64_t i = 0; i < n; ++i) ap[S.pad(i)] = a[i];
            L.amb_pad.upload(c, ap, "ambient A(1-c) (padded)", s);
        }
        HM_CUDA(cudaStreamSynchronize(s));
        const double t2 = T_inf * T_inf;
        L.t_inf4 = t2 * t2;
        L.ambient = true;
    });
}

hm_status hm_export_row_sums(const hm_hmat* F, double* s, double* c) {
    if (!F) return HM_ERR_INVALID_ARG;
    if (s) std::copy(F->h.s_ext.begin(), F->h.s_ext.end(), s);
    if (c) std::copy(F->h.c_ext.begin(), F->h.c_ext.end(), c);
    return HM_OK;
}

// ============================================================================ hot path
hm_status hm_apply_F(hm_ctx* ctx, const hm_hmat* Fh, int32_t nrhs, const double* x, double* y, void* stream) {
    if (!ctx || !Fh || !x || !y || nrhs < 1) return HM_ERR_INVALID_ARG;
    Ctx* c = &ctx->c;
    return guarded(c, [&] {
        HMat& F = const_cast<HMat&>(Fh->h);
        const size_t cnt = (size_t)vec_rows(*F.geom) * nrhs;
        cudaStream_t s = (cudaStream_t)stream;
        int ok_ = 0;
        double* yd = out_target(c, F.host_stage_out, y, cnt, ok_);
        const bool hout = ok_ == 2, hsync = ok_ != 0;
        // HM_FLAG_ASYNC_PINNED: a pinned host output written in place by the program needs no sync
        const bool async_ok = ok_ == 1 && (c->flags & HM_FLAG_ASYNC_PINNED);
        if (nrhs == 1 && F.prog_apply_h.ready && !F.geom->shard.sharded()) {
            if (const double* xa = pinned_alias(x)) {   // pinned host x: the program's copy-in pass
                ProgArgs a = base_args(*F.geom, F.x_dev.p, yd, 1, 0);
                a.host_in = xa;
                F.prog_apply_h.launch(a, s);
                if (hout) HM_CUDA(cudaMemcpyAsync(y, yd, cnt * sizeof(double), cudaMemcpyDeviceToHost, s));
                if (!async_ok) HM_CUDA(cudaStreamSynchronize(s));
                return;
            }
        }
        bool hin = false;
        const double* xd = stage_in(c, F.host_stage_in, x, cnt, s, hin);
        if (nrhs >= 2 && F.prog_apply_m.ready) {   // multi-RHS engine, kMrhsMax columns per launch
            for (int c0 = 0; c0 < nrhs; c0 += kMrhsMax) {
                ProgArgs a = base_args(*F.geom, xd + c0, yd + c0, nrhs, 0);
                a.nrhs = std::min(kMrhsMax, nrhs - c0);
                F.prog_apply_m.launch(a, s);
            }
        } else if (nrhs >= 2 && !F.sp_apply_m.empty()) {   // sharded multi-RHS: allgather + DMMA engine
            for (int c0 = 0; c0 < nrhs; c0 += kMrhsMax) {
                ProgArgs a = base_args(*F.geom, xd, yd + c0, nrhs, c0);
                a.nrhs = std::min(kMrhsMax, nrhs - c0);
                F.sp_apply_m.launch(c, *F.geom, a, s);
            }
        } else {
            for (int col = 0; col < nrhs; ++col) launch_apply(c, F, xd, yd, nrhs, col, s);
        }
        if (hout) HM_CUDA(cudaMemcpyAsync(y, yd, cnt * sizeof(double), cudaMemcpyDeviceToHost, s));
        if (hin || (hsync && !async_ok)) HM_CUDA(cudaStreamSynchronize(s));
    });
}

hm_status hm_solve_C(hm_ctx* ctx, const hm_hlu* LUh, int32_t nrhs, const double* b, double* z, void* stream) {
    if (!ctx || !LUh || !b || !z || nrhs < 1) return HM_ERR_INVALID_ARG;
    Ctx* c = &ctx->c;
    return guarded(c, [&] {
        HLU& L = const_cast<HLU&>(LUh->h);
        const size_t cnt = (size_t)vec_rows(*L.F->geom) * nrhs;
        cudaStream_t s = (cudaStream_t)stream;
        int ok_ = 0;
        double* zd = out_target(c, L.host_stage_out, z, cnt, ok_);
        const bool hout = ok_ == 2, hsync = ok_ != 0;
        // HM_FLAG_ASYNC_PINNED: a pinned host output written in place by the program needs no sync
        const bool async_ok = ok_ == 1 && (c->flags & HM_FLAG_ASYNC_PINNED);
        if (nrhs == 1 && L.prog_solve_h.ready && !L.F->geom->shard.sharded()) {
            if (const double* ba = pinned_alias(b)) {   // pinned host b: the program's copy-in pass
                ProgArgs a = base_args(*L.F->geom, L.T_dev.p, zd, 1, 0);
                a.host_in = ba;
                L.prog_solve_h.launch(a, s);
                if (hout) HM_CUDA(cudaMemcpyAsync(z, zd, cnt * sizeof(double), cudaMemcpyDeviceToHost, s));
                if (!async_ok) HM_CUDA(cudaStreamSynchronize(s));
                return;
            }
        }
        bool hin = false;
        const double* bd = stage_in(c, L.host_stage_in, b, cnt, s, hin);
        if (nrhs >= 2 && L.prog_solve_m.ready) {
            for (int c0 = 0; c0 < nrhs; c0 += kMrhsMax) {
                ProgArgs a = base_args(*L.F->geom, bd + c0, zd + c0, nrhs, 0);
                a.nrhs = std::min(kMrhsMax, nrhs - c0);
                L.prog_solve_m.launch(a, s);
            }
        } else if (nrhs >= 2 && !L.sp_solve_m.empty()) {   // sharded multi-RHS
            for (int c0 = 0; c0 < nrhs; c0 += kMrhsMax) {
                ProgArgs a = base_args(*L.F->geom, bd, zd + c0, nrhs, c0);
                a.nrhs = std::min(kMrhsMax, nrhs - c0);
                L.sp_solve_m.launch(c, *L.F->geom, a, s);
            }
        } else {
            for (int col = 0; col < nrhs; ++col) launch_solve(c, L, bd, zd, nrhs, col, s);
        }
        if (hout) HM_CUDA(cudaMemcpyAsync(z, zd, cnt * sizeof(double), cudaMemcpyDeviceToHost, s));
        if (hin || (hsync && !async_ok)) HM_CUDA(cudaStreamSynchronize(s));
    });
}

}  // extern "C"

namespace hm {
// Rows of the caller's vectors: n (external order) or, sharded, this rank's slice (internal order).
int64_t vec_rows(const Geom& g) { return g.shard.sharded() ? g.shard.le() - g.shard.lb() : g.n; }

ProgArgs base_args(const Geom& g, const double* in, double* out, int ld, int col) {
    ProgArgs a{};
    a.perm = g.d_perm.p;
    a.user_in = in;
    a.user_out = out;
    a.ld = ld;
    a.col = col;
    a.local0 = g.shard.base();
    return a;
}

void launch_apply(Ctx* c, HMat& F, const double* xd, double* yd, int ld, int col, cudaStream_t s) {
    const Geom& g = *F.geom;
    ProgArgs a = base_args(g, xd, yd, ld, col);
    if (g.shard.sharded()) F.sp_apply.launch(c, g, a, s);
    else F.prog_apply.launch(a, s);
}

void launch_solve(Ctx* c, HLU& L, const double* bd, double* zd, int ld, int col, cudaStream_t s) {
    const Geom& g = *L.F->geom;
    ProgArgs a = base_args(g, bd, zd, ld, col);
    if (g.shard.sharded()) L.sp_solve.launch(c, g, a, s);
    else L.prog_solve.launch(a, s);
}

// One flux evaluation (engine program(s)) for column `col` (device pointers).
void launch_flux(Ctx* c, HLU& L, const double* Td, double* qd, int ld, int col, cudaStream_t s,
                 unsigned long long* trace) {
    const Geom& g = *L.F->geom;
    ProgArgs a = base_args(g, Td, qd, ld, col);
    a.sigma = 5.670374419e-8;  // DESIGN.md reading R2
    a.trace = trace;
    if (g.shard.sharded()) {
        a.eps_int = L.eps_pad.p;
        a.area_int = L.area_pad.p;
        a.g_int = L.g_pad.p;
        a.amb = L.ambient ? L.amb_pad.p : nullptr;
        a.t_inf4 = L.t_inf4;
        a.T_pad = L.T_pad;
        L.sp_flux.launch(c, g, a, s);
    } else {
        a.eps_int = L.eps_int.p;
        a.eps_ext = L.eps_ext.p;
        a.area_int = g.d_geo.p + 6 * g.n;
        a.g_int = L.g_int.p;
        a.amb = L.ambient ? L.amb_int.p : nullptr;
        a.t_inf4 = L.t_inf4;
        L.prog_flux.launch(a, s);
    }
}

// Multi-RHS flux: r <= kMrhsMax columns starting at Td / qd (caller's arrays, row stride ld).
void launch_flux_m(HLU& L, const double* Td, double* qd, int ld, int r, cudaStream_t s) {
    const Geom& g = *L.F->geom;
    ProgArgs a = base_args(g, Td, qd, ld, 0);
    a.nrhs = r;
    a.sigma = 5.670374419e-8;  // DESIGN.md reading R2
    a.eps_int = L.eps_int.p;
    a.eps_ext = L.eps_ext.p;
    a.area_int = g.d_geo.p + 6 * g.n;
    a.g_int = L.g_int.p;
    a.amb = L.ambient ? L.amb_int.p : nullptr;
    a.t_inf4 = L.t_inf4;
    L.prog_flux_m.launch(a, s);
}

}  // namespace hm

extern "C" {

hm_status hm_radiative_flux(hm_ctx* ctx, const hm_hmat* Fh, const hm_hlu* LUh, int32_t nrhs, const double* T, double* q,
                            void* stream) {
    if (!ctx || !Fh || !LUh || !T || !q || nrhs < 1) return HM_ERR_INVALID_ARG;
    if (LUh->h.F != &Fh->h) {
        ctx->c.last_error = "hm_radiative_flux: LU was not factored from this F";
        return HM_ERR_NOT_READY;
    }
    Ctx* c = &ctx->c;
    return guarded(c, [&] {
        HLU& L = const_cast<HLU&>(LUh->h);
        const size_t cnt = (size_t)vec_rows(*L.F->geom) * nrhs;
        cudaStream_t s = (cudaStream_t)stream;
        int ok_ = 0;
        double* qd = out_target(c, L.host_stage_out, q, cnt, ok_);
        const bool hout = ok_ == 2, hsync = ok_ != 0;
        // HM_FLAG_ASYNC_PINNED: a pinned host output written in place by the program needs no sync
        const bool async_ok = ok_ == 1 && (c->flags & HM_FLAG_ASYNC_PINNED);
        // single vector, pinned host T: the program's copy-in pass reads it (no separate H2D copy
        // before the kernel: the payload stream starts while T crosses the bus)
        if (nrhs == 1 && L.prog_flux_h.ready && !L.F->geom->shard.sharded()) {
            cudaPointerAttributes pa;
            if (cudaPointerGetAttributes(&pa, T) != cudaSuccess) {
                cudaGetLastError();
                pa.type = cudaMemoryTypeUnregistered;
            }
            if (pa.type == cudaMemoryTypeHost && pa.devicePointer) {
                const Geom& g = *L.F->geom;
                ProgArgs a = base_args(g, L.T_dev.p, qd, 1, 0);
                a.host_in = static_cast<const double*>(pa.devicePointer);
                a.sigma = 5.670374419e-8;   // DESIGN.md reading R2
                a.eps_int = L.eps_int.p;
                a.eps_ext = L.eps_ext.p;
                a.area_int = g.d_geo.p + 6 * g.n;
                a.g_int = L.g_int.p;
                a.amb = L.ambient ? L.amb_int.p : nullptr;
                a.t_inf4 = L.t_inf4;
                L.prog_flux_h.launch(a, s);
                if (hout) HM_CUDA(cudaMemcpyAsync(q, qd, cnt * sizeof(double), cudaMemcpyDeviceToHost, s));
                if (!async_ok) HM_CUDA(cudaStreamSynchronize(s));
                return;
            }
        }
        bool hin = false;
        const double* Td = stage_in(c, L.host_stage_in, T, cnt, s, hin);
        if (nrhs >= 2 && L.prog_flux_m.ready) {
            for (int c0 = 0; c0 < nrhs; c0 += kMrhsMax) launch_flux_m(L, Td + c0, qd + c0, nrhs, std::min(kMrhsMax, nrhs - c0), s);
        } else if (nrhs >= 2 && !L.sp_flux_m.empty()) {   // sharded multi-RHS flux
            const Geom& g = *L.F->geom;
            for (int c0 = 0; c0 < nrhs; c0 += kMrhsMax) {
                ProgArgs a = base_args(g, Td, qd + c0, nrhs, c0);
                a.nrhs = std::min(kMrhsMax, nrhs - c0);
                a.sigma = 5.670374419e-8;   // DESIGN.md reading R2
                a.eps_int = L.eps_pad.p;
                a.area_int = L.area_pad.p;
                a.g_int = L.g_pad.p;
                a.amb = L.ambient ? L.amb_pad.p : nullptr;
                a.t_inf4 = L.t_inf4;
                a.T_pad = L.T_loc_m.p;
                L.sp_flux_m.launch(c, g, a, s);
            }
        } else {
            for (int col = 0; col < nrhs; ++col) launch_flux(c, L, Td, qd, nrhs, col, s);
        }
        if (hout) HM_CUDA(cudaMemcpyAsync(q, qd, cnt * sizeof(double), cudaMemcpyDeviceToHost, s));
        if (hin || (hsync && !async_ok)) HM_CUDA(cudaStreamSynchronize(s));
    });
}

hm_status hm_profile_flux(hm_ctx* ctx, const hm_hmat* Fh, const hm_hlu* LUh, const double* T, double* q, int32_t iters,
                          double* ms_out, int64_t* launches_out, void* stream) {
    if (!ctx || !Fh || !LUh || !T || !q || iters < 1 || !ms_out) return HM_ERR_INVALID_ARG;
    Ctx* c = &ctx->c;
    return guarded(c, [&] {
        HLU& L = const_cast<HLU&>(LUh->h);
        HMat& F = const_cast<HMat&>(Fh->h);
        cudaStream_t s = (cudaStream_t)stream;
        cudaEvent_t e0, e1;
        HM_CUDA(cudaEventCreate(&e0));
        HM_CUDA(cudaEventCreate(&e1));
        auto timeit = [&](auto&& fn) {
            fn();
            HM_CUDA(cudaEventRecord(e0, s));
            for (int it = 0; it < iters; ++it) fn();
            HM_CUDA(cudaEventRecord(e1, s));
            HM_CUDA(cudaEventSynchronize(e1));
            float ms = 0;
            HM_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            return (double)ms / iters;
        };
        ms_out[0] = timeit([&] { launch_flux(c, L, T, q, 1, 0, s); });
        ms_out[1] = timeit([&] { launch_apply(c, F, T, q, 1, 0, s); });
        ms_out[2] = timeit([&] { launch_solve(c, L, T, q, 1, 0, s); });
        for (int i = 3; i < 6; ++i) ms_out[i] = 0.0;
        if (F.geom->shard.sharded()) {   // the same segments with their allgathers skipped: comm share
            c->skip_exchange = true;
            try {
                ms_out[3] = timeit([&] { launch_flux(c, L, T, q, 1, 0, s); });
            } catch (...) {
                c->skip_exchange = false;
                throw;
            }
            c->skip_exchange = false;
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (launches_out) {
            const bool sh = F.geom->shard.sharded();
            launches_out[0] = sh ? (int64_t)L.sp_flux.segs.size() : 1;
            launches_out[1] = sh ? (int64_t)F.sp_apply.segs.size() : 1;
            launches_out[2] = sh ? (int64_t)L.sp_solve.segs.size() : 1;
            int64_t passes = 0, units = 0;
            if (sh) {
                for (auto& P : L.sp_flux.segs) { passes += (int64_t)P->h_passes.size(); units += (int64_t)P->h_units.size(); }
            } else {
                passes = (int64_t)L.prog_flux.h_passes.size();
                units = (int64_t)L.prog_flux.h_units.size();
            }
            launches_out[3] = passes;
            launches_out[4] = units;
            launches_out[5] = engine_grid();
        }
    });
}

hm_status hm_trace_flux(hm_ctx* ctx, const hm_hmat* Fh, const hm_hlu* LUh, const double* T, double* q,
                        int32_t max_passes, int32_t* n_passes, double* t_begin_us, double* t_end_us,
                        int64_t* pass_bytes, void* stream) {
    if (!ctx || !Fh || !LUh || !T || !q || !n_passes) return HM_ERR_INVALID_ARG;
    Ctx* c = &ctx->c;
    return guarded(c, [&] {
        HLU& L = const_cast<HLU&>(LUh->h);
        Program& P = L.prog_flux;
        cudaStream_t s = (cudaStream_t)stream;
        const size_t np = P.h_passes.size();
        *n_passes = (int32_t)np;
        std::vector<unsigned long long> init(2 * np);
        for (size_t i = 0; i < np; ++i) { init[2 * i] = ~0ull; init[2 * i + 1] = 0ull; }
        if (P.trace.n < 2 * np) P.trace.alloc(c, 2 * np, "engine trace");
        HM_CUDA(cudaMemcpyAsync(P.trace.p, init.data(), 2 * np * sizeof(unsigned long long), cudaMemcpyHostToDevice, s));
        if (L.F->geom->shard.sharded()) throw Error(HM_ERR_UNSUPPORTED, "hm_trace_flux: world == 1 only");
        launch_flux(c, L, T, q, 1, 0, s, P.trace.p);
        std::vector<unsigned long long> tr(2 * np);
        HM_CUDA(cudaMemcpyAsync(tr.data(), P.trace.p, 2 * np * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
        HM_CUDA(cudaStreamSynchronize(s));
        unsigned long long t0 = ~0ull;
        for (size_t i = 0; i < np; ++i) t0 = std::min(t0, tr[2 * i]);
        std::vector<int64_t> bytes(np, 0);
        for (const Unit& u : P.h_units) bytes[u.pass] += u.type == UNIT_STREAM ? 8LL * u.ncols * u.ld : 0;
        for (size_t i = 0; i < np && (int32_t)i < max_passes; ++i) {
            if (t_begin_us) t_begin_us[i] = (tr[2 * i] == ~0ull) ? -1.0 : (double)(tr[2 * i] - t0) * 1e-3;
            if (t_end_us) t_end_us[i] = (double)(tr[2 * i + 1] - t0) * 1e-3;
            if (pass_bytes) pass_bytes[i] = bytes[i];
        }
    });
}

hm_status hm_storage_report(const hm_hmat* Fh, const hm_hlu* LUh, hm_storage* out) {
    if (!Fh || !out) return HM_ERR_INVALID_ARG;
    std::memset(out, 0, sizeof(*out));
    const HMat& F = Fh->h;
    const Geom& g = *F.geom;
    out->n = g.n;
    out->n_leaves = (int64_t)g.leaves.size();
    out->depth = g.depth;
    out->n_blocks = (int64_t)g.blocks.size();
    int64_t lr = 0, ksum = 0;
    for (size_t b = 0; b < g.blocks.size(); ++b) {
        if (F.blk_kind[b] == KIND_DENSE) out->n_dense++;
        else if (F.blk_kind[b] == KIND_LR) { lr++; ksum += F.blk_rank[b]; out->rank_max = std::max<int64_t>(out->rank_max, F.blk_rank[b]); }
        else out->n_adm_dense++;
    }
    out->n_lowrank = lr;
    out->rank_mean = lr ? double(ksum) / lr : 0.0;
    out->bytes_F_phase1 = 8 * F.op.p1_doubles();
    out->bytes_F_phase2 = 8 * F.op.p2_doubles();
    out->bytes_F = out->bytes_F_phase1 + out->bytes_F_phase2;
    out->launches_apply_F = g.shard.sharded() ? (int64_t)F.sp_apply.segs.size() : 1;  // persistent engine launches
    out->rank = g.shard.rank;
    out->world = g.shard.world;
    out->bytes_F_local = g.shard.sharded() ? 8 * (F.op_loc.p1_doubles() + F.op_loc.p2_doubles()) : out->bytes_F;
    for (int q = 0; q < 3; ++q) out->setup_seconds[q] = F.setup_seconds[q];
    out->setup_seconds[0] += g.setup_seconds;
    if (LUh) {
        const HLU& L = LUh->h;
        out->bytes_C = 8 * L.bytes;
        out->bytes_C_leaf = 8 * L.bytes_leaf;
        out->n_blocks_C = L.n_blocks;
        out->n_lowrank_C = L.n_lr;
        out->rank_max_C = L.rank_max;
        out->rank_mean_C = L.n_lr ? double(L.rank_sum) / L.n_lr : 0.0;
        out->lu_method = L.params.method;
        out->lu_truncations = L.hlu_truncations;
        out->lu_threads = (int64_t)L.hlu_threads;
        out->launches_solve_C = g.shard.sharded() ? (int64_t)L.sp_solve.segs.size() : 1;
        out->bytes_C_local = g.shard.sharded() ? 8 * (L.leafL_loc.p1_doubles() + L.leafL_loc.p2_doubles() +
                                                      L.leafU_loc.p1_doubles() + L.leafU_loc.p2_doubles())
                                               : out->bytes_C;
        for (int q = 0; q < 4; ++q) out->setup_seconds[4 + q] = L.setup_seconds[q];
    }
    return HM_OK;
}

}  // extern "C"

// ============================================================================ cavity operator (NEXT-1)
namespace {
// y_facets = A o q(eta) = Rbar eta (eq:Rbardef) by the flux program with the eta input / Rbar output
// modes, then Q_nodes = P^T y (eqn:S_def_matrix)
void cavity_column(Ctx* c, HLU& L, Proj& P, const double* Tn, const double* xn, int mode, int ld, int col, double* Qn,
                   cudaStream_t s) {
    const Geom& g = *L.F->geom;
    k::proj_facets(P.rp.p, P.ci.p, P.cv.p, Tn, xn, mode, ld, col, P.eta.p, P.n_facets, s);
    ProgArgs a = base_args(g, P.eta.p, P.rbar.p, 1, 0);
    a.sigma = 5.670374419e-8;  // DESIGN.md reading R2
    a.eps_int = L.eps_int.p;
    a.eps_ext = L.eps_ext.p;
    a.area_int = g.d_geo.p + 6 * g.n;
    a.g_int = L.g_int.p;
    a.amb = L.ambient ? L.amb_int.p : nullptr;
    a.t_inf4 = (mode == 0 ? L.t_inf4 : 0.0);   // Jacobian mode: d/dT of the constant T_inf^4 is 0
    a.eta_in = 1;
    a.rbar_out = 1;
    L.prog_flux.launch(a, s);
    k::proj_nodes(P.tp.p, P.ti.p, P.tv.p, P.rbar.p, ld, col, Qn, P.n_nodes, s);
}

// Sharded (world > 1): node vectors are replicated on every rank; each rank projects onto its own facets,
// runs the sharded flux program with the eta-input / Rbar-output modes on its slice, projects back onto
// the nodes its facets touch, and the per-rank node partials are allgathered and summed in rank order.
void cavity_column_sharded(Ctx* c, HLU& L, Proj& P, const double* Tn, const double* xn, int mode, int ld, int col,
                           double* Qn, cudaStream_t s) {
    const Geom& g = *L.F->geom;
    const Shard& S = g.shard;
    k::proj_facets(P.rp_loc.p, P.ci_loc.p, P.cv_loc.p, Tn, xn, mode, ld, col, P.eta_loc.p, P.n_loc, s);
    ProgArgs a = base_args(g, P.eta_loc.p, P.rbar_loc.p, 1, 0);
    a.sigma = 5.670374419e-8;  // DESIGN.md reading R2
    a.eps_int = L.eps_pad.p;
    a.area_int = L.area_pad.p;
    a.g_int = L.g_pad.p;
    a.amb = L.ambient ? L.amb_pad.p : nullptr;
    a.t_inf4 = (mode == 0 ? L.t_inf4 : 0.0);   // Jacobian mode: d/dT of the constant T_inf^4 is 0
    a.T_pad = L.T_pad;
    a.eta_in = 1;
    a.rbar_out = 1;
    L.sp_flux.launch(c, g, a, s);
    k::proj_nodes(P.tp_loc.p, P.ti_loc.p, P.tv_loc.p, P.rbar_loc.p, 1, 0, P.qpart.p + (int64_t)S.rank * P.qcount,
                  P.n_nodes, s);
    if (!c->ex) throw Error(HM_ERR_NOT_READY, "sharded cavity operator without an exchanger");
    c->ex->allgather(P.qpart.p, P.qcount, s);
    k::sum_segments(P.qpart.p, S.world, P.qcount, P.n_nodes, ld, col, Qn, s);
}

hm_status cavity_call(hm_ctx* ctx, const hm_hmat* Fh, const hm_hlu* LUh, hm_proj* Ph, int32_t nrhs, const double* T,
                      const double* x, double* out, void* stream, int mode) {
    if (!ctx || !Fh || !LUh || !Ph || !T || !out || nrhs < 1 || (mode == 1 && !x)) return HM_ERR_INVALID_ARG;
    if (LUh->h.F != &Fh->h || Ph->p.geom != Fh->h.geom) {
        ctx->c.last_error = "cavity operator: LU / projection not built for this F";
        return HM_ERR_NOT_READY;
    }
    Ctx* c = &ctx->c;
    return guarded(c, [&] {
        HLU& L = const_cast<HLU&>(LUh->h);
        Proj& P = Ph->p;
        const size_t cnt = (size_t)P.n_nodes * nrhs;
        cudaStream_t s = (cudaStream_t)stream;
        bool h1 = false, h2 = false;
        const double* Td = stage_in(c, P.host_in, T, cnt, s, h1);
        const double* xd = mode == 1 ? stage_in(c, P.host_in2, x, cnt, s, h2) : nullptr;
        const bool hout = !is_device_ptr(out);
        double* od = out;
        if (hout) {
            if (P.host_out.n < cnt) P.host_out.alloc(c, cnt, "host staging (out)");
            od = P.host_out.p;
        }
        const bool sharded = Fh->h.geom->shard.sharded();
        for (int col = 0; col < nrhs; ++col) {
            if (sharded) cavity_column_sharded(c, L, P, Td, xd, mode, nrhs, col, od, s);
            else cavity_column(c, L, P, Td, xd, mode, nrhs, col, od, s);
        }
        if (hout) HM_CUDA(cudaMemcpyAsync(out, od, cnt * sizeof(double), cudaMemcpyDeviceToHost, s));
        if (h1 || h2 || hout) HM_CUDA(cudaStreamSynchronize(s));
    });
}
}  // namespace

extern "C" {

hm_status hm_projection_create(hm_ctx* ctx, const hm_geom* geom, int64_t n_nodes, const int64_t* row_ptr,
                               const int32_t* col, const double* val, hm_proj** out) {
    if (!ctx || !geom || !row_ptr || !col || !val || !out || n_nodes < 1) return HM_ERR_INVALID_ARG;
    *out = nullptr;
    Ctx* c = &ctx->c;
    return guarded(c, [&] {
        if (c->host_only) throw Error(HM_ERR_NOT_READY, "host-only context");
        const int64_t n = geom->g.n;
        if (row_ptr[0] != 0) throw Error(HM_ERR_INVALID_ARG, "projection: row_ptr[0] must be 0");
        for (int64_t i = 0; i < n; ++i)
            if (row_ptr[i + 1] < row_ptr[i]) throw Error(HM_ERR_INVALID_ARG, "projection: row_ptr not monotone");
        const int64_t nnz = row_ptr[n];
        for (int64_t q = 0; q < nnz; ++q) {
            if (col[q] < 0 || col[q] >= n_nodes)
                throw Error(HM_ERR_INVALID_ARG, "projection: node id out of range at entry " + std::to_string(q));
            if (!std::isfinite(val[q])) throw Error(HM_ERR_INVALID_ARG, "projection: non-finite value");
        }
        auto* H = new hm_proj;
        std::unique_ptr<hm_proj> guard(H);
        Proj& P = H->p;
        P.ctx = c;
        P.geom = &geom->g;
        P.n_facets = n;
        P.n_nodes = n_nodes;
        const cudaStream_t s = c->stream;
        P.rp.upload(c, std::vector<int64_t>(row_ptr, row_ptr + n + 1), "P row_ptr", s);
        P.ci.upload(c, std::vector<int32_t>(col, col + nnz), "P col", s);
        P.cv.upload(c, std::vector<double>(val, val + nnz), "P val", s);
        // transpose (node -> facets), entries in increasing facet order: fixed summation order
        std::vector<int64_t> tp(n_nodes + 1, 0);
        for (int64_t q = 0; q < nnz; ++q) ++tp[col[q] + 1];
        for (int64_t m = 0; m < n_nodes; ++m) tp[m + 1] += tp[m];
        std::vector<int32_t> ti(nnz);
        std::vector<double> tv(nnz);
        std::vector<int64_t> fill(tp.begin(), tp.end() - 1);
        for (int64_t i = 0; i < n; ++i)
            for (int64_t q = row_ptr[i]; q < row_ptr[i + 1]; ++q) {
                const int64_t d = fill[col[q]]++;
                ti[d] = (int32_t)i;
                tv[d] = val[q];
            }
        P.tp.upload(c, tp, "P^T row_ptr", s);
        P.ti.upload(c, ti, "P^T facets", s);
        P.tv.upload(c, tv, "P^T val", s);
        P.eta.alloc(c, (size_t)n, "cavity eta");
        P.rbar.alloc(c, (size_t)n, "cavity Rbar eta");
        const Shard& S = geom->g.shard;
        if (S.sharded()) {   // this rank's facets in local internal order (the sharded flux's slice)
            const int64_t lb = S.lb(), nl = S.le() - S.lb();
            std::vector<int64_t> rl(nl + 1, 0);
            std::vector<int32_t> cl;
            std::vector<double> vl;
            for (int64_t r = 0; r < nl; ++r) {
                const int64_t i = geom->g.perm[lb + r];
                for (int64_t q = row_ptr[i]; q < row_ptr[i + 1]; ++q) {
                    cl.push_back(col[q]);
                    vl.push_back(val[q]);
                }
                rl[r + 1] = (int64_t)cl.size();
            }
            std::vector<int64_t> tl(n_nodes + 1, 0);
            for (int32_t m : cl) ++tl[m + 1];
            for (int64_t m = 0; m < n_nodes; ++m) tl[m + 1] += tl[m];
            std::vector<int32_t> til(cl.size());
            std::vector<double> tvl(cl.size());
            std::vector<int64_t> fl(tl.begin(), tl.end() - 1);
            for (int64_t r = 0; r < nl; ++r)
                for (int64_t q = rl[r]; q < rl[r + 1]; ++q) {
                    const int64_t d = fl[cl[q]]++;
                    til[d] = (int32_t)r;
                    tvl[d] = vl[q];
                }
            P.n_loc = nl;
            P.qcount = (n_nodes + 1) & ~int64_t(1);
            P.rp_loc.upload(c, rl, "P row_ptr (local)", s);
            P.ci_loc.upload(c, cl.empty() ? std::vector<int32_t>{0} : cl, "P col (local)", s);
            P.cv_loc.upload(c, vl.empty() ? std::vector<double>{0.0} : vl, "P val (local)", s);
            P.tp_loc.upload(c, tl, "P^T row_ptr (local)", s);
            P.ti_loc.upload(c, til.empty() ? std::vector<int32_t>{0} : til, "P^T facets (local)", s);
            P.tv_loc.upload(c, tvl.empty() ? std::vector<double>{0.0} : tvl, "P^T val (local)", s);
            P.eta_loc.alloc(c, (size_t)std::max<int64_t>(nl, 1), "cavity eta (local)");
            P.rbar_loc.alloc(c, (size_t)std::max<int64_t>(nl, 1), "cavity Rbar eta (local)");
            P.qpart.alloc(c, (size_t)(S.world * P.qcount), "cavity node partials");
        }
        HM_CUDA(cudaStreamSynchronize(s));
        *out = guard.release();
    });
}

void hm_destroy_projection(hm_proj* P) { delete P; }

hm_status hm_cavity_flux(hm_ctx* ctx, const hm_hmat* F, const hm_hlu* LU, hm_proj* P, int32_t nrhs, const double* T_nodes,
                         double* Q_nodes, void* stream) {
    return cavity_call(ctx, F, LU, P, nrhs, T_nodes, nullptr, Q_nodes, stream, 0);
}

hm_status hm_cavity_jacobian(hm_ctx* ctx, const hm_hmat* F, const hm_hlu* LU, hm_proj* P, int32_t nrhs,
                             const double* T_nodes, const double* x_nodes, double* y_nodes, void* stream) {
    return cavity_call(ctx, F, LU, P, nrhs, T_nodes, x_nodes, y_nodes, stream, 1);
}

}  // extern "C"
