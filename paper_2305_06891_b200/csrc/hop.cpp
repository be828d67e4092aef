// Operator builder: flattens a set of blocks (dense + low-rank U V^T) into the two-pass
// column-stream layout of the hot path:
//
//   arena = [ phase-1 panels: per column cluster tau, the V^T of every low-rank block (., tau)
//             stacked: column-major, ld = K_tau (even), n_tau columns                        ]
//           [ phase-2 panels: per leaf row r, the leaf-row slices of every dense block and U
//             factor covering r: column-major, ld = m_r (even), in block order              ]
//   colsrc[c] = index into XT = [x (n) | t (sum k)] of the input multiplying column c.
// Panels are cut into ~48 KB work units (row tile <= 128 rows x column chunk).
#include <algorithm>
#include <map>

#include "hm_internal.h"

namespace hm {

static inline int64_t align2(int64_t x) { return (x + 1) & ~int64_t(1); }

static void make_units(Ctx* ctx, StreamPass& P, cudaStream_t s) {
    std::vector<Unit> units;
    int64_t part = 0;
    int32_t grp = 0;
    constexpr int kThreads = 256, kQ = 12;  // must match kernels_apply.cu: <= kQ columns per thread
    for (const Panel& pn : P.panels) {
        if (pn.ncols == 0) continue;
        for (int32_t tr0 = 0; tr0 < pn.nrows; tr0 += 128) {
            const int32_t tn = std::min<int32_t>(128, pn.nrows - tr0);
            const int32_t tn_pad = (tn + 1) & ~1;
            const int64_t G = kThreads / (tn_pad / 2);
            int64_t C = kQ * G;  // ~ 12 * 256 * 2 doubles = 48 KB of payload per work unit
            const int32_t nseg = (int32_t)((pn.ncols + C - 1) / C);
            C = (pn.ncols + nseg - 1) / nseg;
            const int32_t g = nseg > 1 ? grp++ : -1;
            for (int32_t sg = 0; sg < nseg; ++sg) {
                Unit u{};
                u.a_off = pn.a_off + tr0;
                u.out0 = pn.out0 + tr0;
                u.part_off = nseg > 1 ? part : 0;
                u.ld = pn.ld;
                u.nrows = tn;
                u.c0 = (int32_t)(sg * C);
                u.ncols = (int32_t)std::min<int64_t>(C, pn.ncols - sg * C);
                u.cs_off = pn.cs_off;
                u.grp = g;
                u.nseg = nseg;
                u.seg = sg;
                units.push_back(u);
                if (nseg > 1) part += tn_pad;
            }
        }
    }
    P.n_units = (int64_t)units.size();
    P.units.upload(ctx, units, "work units", s);
    P.part.alloc(ctx, (size_t)std::max<int64_t>(part, 2), "split-K partials");
    P.counters.alloc(ctx, (size_t)std::max<int32_t>(grp, 1), "split-K counters");
    HM_CUDA(cudaMemsetAsync(P.counters.p, 0, sizeof(int32_t) * std::max<int32_t>(grp, 1), s));
}

void build_hop(Ctx* ctx, const Geom& g, std::vector<SrcBlock>& blocks, HOp& op, cudaStream_t s) {
    const int64_t n = g.n;
    const int nleaves = (int)g.leaves.size();
    op.n_rows_total = n;
    op.items.clear();
    op.p1.panels.clear();
    op.p2.panels.clear();
    op.p1.doubles = op.p2.doubles = 0;
    op.n_lr = op.n_dense = op.rank_sum = 0;
    op.rank_max = 0;
    std::vector<int32_t> colsrc;
    std::vector<int64_t> pack;   // dst, src, rows, cols, rs, cs, dld
    std::vector<int64_t> fill;   // dst, r0, rows, c0, cols, dld
    int64_t off = 0, tcount = 0;

    // ---- phase-1 panels: low-rank blocks grouped by column cluster (first-appearance order)
    std::vector<int64_t> tbase(blocks.size(), -1), voff(blocks.size(), -1), vld(blocks.size(), 0);
    std::map<std::pair<int64_t, int64_t>, int> tau_index;
    std::vector<std::vector<int>> taus;
    for (size_t b = 0; b < blocks.size(); ++b) {
        const SrcBlock& B = blocks[b];
        if (B.kind != KIND_LR) { ++op.n_dense; continue; }
        ++op.n_lr;
        op.rank_sum += B.k;
        op.rank_max = std::max(op.rank_max, B.k);
        if (B.k == 0) continue;
        auto key = std::make_pair(B.c0, B.n);
        auto it = tau_index.find(key);
        if (it == tau_index.end()) {
            tau_index[key] = (int)taus.size();
            taus.push_back({(int)b});
        } else {
            taus[it->second].push_back((int)b);
        }
    }
    for (const auto& members : taus) {
        const SrcBlock& B0 = blocks[members[0]];
        int64_t K = 0;
        for (int b : members) K += blocks[b].k;
        const int64_t ld = align2(K);
        Panel pn{off, n + tcount, (int32_t)ld, (int32_t)K, (int32_t)B0.n, (int32_t)colsrc.size()};
        for (int64_t j = 0; j < B0.n; ++j) colsrc.push_back((int32_t)(B0.c0 + j));
        int64_t local = 0;
        for (int b : members) {
            const SrcBlock& B = blocks[b];
            tbase[b] = tcount + local;
            voff[b] = off + local;
            vld[b] = ld;
            // V_b[j, l] -> panel row local+l, column j
            pack.insert(pack.end(), {off + local, (int64_t)(uintptr_t)B.V, (int64_t)B.k, B.n, B.v_ld, 1, ld});
            local += B.k;
        }
        op.p1.panels.push_back(pn);
        op.p1.doubles += K * B0.n;
        off += ld * B0.n;
        tcount += K;
    }
    op.n_t = tcount;

    // ---- phase-2 panels: per leaf row, the slices of every block covering it (block order)
    std::vector<std::vector<int>> items(nleaves);
    for (size_t b = 0; b < blocks.size(); ++b) {
        const SrcBlock& B = blocks[b];
        if (B.kind == KIND_LR && B.k == 0) continue;
        const int l0 = g.leaf_of(B.r0), l1 = g.leaf_of(B.r0 + B.m - 1);
        for (int l = l0; l <= l1; ++l) items[l].push_back((int)b);
    }
    for (int l = 0; l < nleaves; ++l) {
        if (items[l].empty()) continue;
        const Node& L = g.nodes[g.leaves[l]];
        const int64_t lr0 = L.begin, lm = L.size(), ld = align2(lm);
        Panel pn{off, lr0, (int32_t)ld, (int32_t)lm, 0, (int32_t)colsrc.size()};
        for (int b : items[l]) {
            const SrcBlock& B = blocks[b];
            const int64_t ro = lr0 - B.r0;
            if (B.kind != KIND_LR) {
                if (B.fill_entries)
                    fill.insert(fill.end(), {off, lr0, lm, B.c0, B.n, ld});
                else
                    pack.insert(pack.end(), {off, (int64_t)(uintptr_t)(B.dense + ro * B.d_rs), lm, B.n, B.d_rs, B.d_cs, ld});
                for (int64_t j = 0; j < B.n; ++j) colsrc.push_back((int32_t)(B.c0 + j));
                op.items.push_back(HOp::ItemRec{off, ld, -1, 0, lr0, lm, B.c0, B.n, 0});
                off += ld * B.n;
                pn.ncols += (int32_t)B.n;
                op.p2.doubles += lm * B.n;
            } else {
                pack.insert(pack.end(), {off, (int64_t)(uintptr_t)(B.U + ro), lm, (int64_t)B.k, 1, B.u_ld, ld});
                for (int q = 0; q < B.k; ++q) colsrc.push_back((int32_t)(n + tbase[b] + q));
                op.items.push_back(HOp::ItemRec{off, ld, voff[b], vld[b], lr0, lm, B.c0, B.n, B.k});
                off += ld * B.k;
                pn.ncols += B.k;
                op.p2.doubles += lm * B.k;
            }
        }
        op.p2.panels.push_back(pn);
    }
    if ((int64_t)n + tcount >= INT32_MAX || (int64_t)colsrc.size() >= INT32_MAX)
        throw Error(HM_ERR_UNSUPPORTED, "index space exceeds int32");

    op.arena.alloc(ctx, (size_t)std::max<int64_t>(off, 2), "operator arena");
    HM_CUDA(cudaMemsetAsync(op.arena.p, 0, sizeof(double) * (size_t)std::max<int64_t>(off, 2), s));
    op.colsrc.upload(ctx, colsrc, "colsrc", s);
    make_units(ctx, op.p1, s);
    make_units(ctx, op.p2, s);
    DBuf<int64_t> d_pack, d_fill;
    d_pack.upload(ctx, pack, "pack tasks", s);
    d_fill.upload(ctx, fill, "fill tasks", s);
    k::pack(d_pack.p, (int)(pack.size() / 7), op.arena.p, s);
    static_assert(sizeof(int64_t) == sizeof(void*), "pointer size");
    if (!fill.empty()) {
        DBuf<int32_t> err;
        err.alloc(ctx, 4, "err");
        HM_CUDA(cudaMemsetAsync(err.p, 0, 4 * sizeof(int32_t), s));
        k::fill_entries(g.d_geo.p, n, d_fill.p, (int)(fill.size() / 6), op.arena.p, err.p, s);
        int32_t h[4];
        HM_CUDA(cudaMemcpyAsync(h, err.p, sizeof(h), cudaMemcpyDeviceToHost, s));
        HM_CUDA(cudaStreamSynchronize(s));
        if (h[0])
            throw Error(HM_ERR_DEGENERATE_GEOMETRY, "coincident collocation points for facets " +
                                                        std::to_string(g.perm[h[1]]) + "," + std::to_string(g.perm[h[2]]));
    }
    HM_CUDA(cudaStreamSynchronize(s));
}

}  // namespace hm
