// Operator builder: flattens a set of blocks (dense + low-rank U V^T) into the two-phase stream
// layout of the hot path:
//
//   arena = [ V^T of every low-rank block (k x n, row-major) ]  -> phase 1, one task per row
//           [ per leaf row r: one contiguous column stream ]     -> phase 2, one CTA per leaf row
//                 each column = m_r contiguous doubles: the leaf-row slice of a dense block
//                 (column-major) or of a U factor (column-major), in block order
//   colsrc[c] = index into XT = [x (n) | t (sum k)] of the input that multiplies column c.
#include <algorithm>

#include "hm_internal.h"

namespace hm {

static inline int64_t align2(int64_t x) { return (x + 1) & ~int64_t(1); }

void build_hop(Ctx* ctx, const Geom& g, std::vector<SrcBlock>& blocks, HOp& op, cudaStream_t s) {
    const int64_t n = g.n;
    const int nleaves = (int)g.leaves.size();
    op.n_rows_total = n;
    op.items.clear();
    op.h_p2.clear();
    op.h_colsrc.clear();
    op.n_lr = op.n_dense = op.rank_sum = 0;
    op.rank_max = 0;
    op.p1_doubles = op.p2_doubles = 0;

    // V^T region first, t bases in block order
    std::vector<int64_t> tbase(blocks.size(), -1), vtoff(blocks.size(), -1);
    std::vector<P1Task> p1;
    std::vector<int64_t> pack;   // dst, src, rows, cols, rs, cs
    std::vector<int64_t> fill;   // dst, r0, rows, c0, cols
    int64_t off = 0, tcount = 0;
    for (size_t b = 0; b < blocks.size(); ++b) {
        const SrcBlock& B = blocks[b];
        if (B.kind != KIND_LR) { ++op.n_dense; continue; }
        ++op.n_lr;
        op.rank_sum += B.k;
        op.rank_max = std::max(op.rank_max, B.k);
        if (B.k == 0) continue;
        tbase[b] = tcount;
        vtoff[b] = off;
        for (int l = 0; l < B.k; ++l) p1.push_back(P1Task{off + (int64_t)l * B.n, (int32_t)B.n, (int32_t)B.c0});
        pack.insert(pack.end(), {off, (int64_t)(uintptr_t)B.V, B.n, (int64_t)B.k, 1, B.v_ld});
        off = align2(off + B.n * B.k);
        op.p1_doubles += B.n * B.k;
        tcount += B.k;
    }
    // items per leaf row
    std::vector<std::vector<int>> items(nleaves);
    for (size_t b = 0; b < blocks.size(); ++b) {
        const SrcBlock& B = blocks[b];
        if (B.kind == KIND_LR && B.k == 0) continue;
        const int l0 = g.leaf_of(B.r0), l1 = g.leaf_of(B.r0 + B.m - 1);
        for (int l = l0; l <= l1; ++l) items[l].push_back((int)b);
    }
    int max_m = 0;
    for (int l = 0; l < nleaves; ++l) {
        if (items[l].empty()) continue;
        const Node& L = g.nodes[g.leaves[l]];
        const int64_t lr0 = L.begin, lm = L.size();
        max_m = std::max<int>(max_m, (int)lm);
        P2Row row{off, (int32_t)lr0, (int32_t)lm, (int32_t)op.h_colsrc.size(), 0};
        for (int b : items[l]) {
            const SrcBlock& B = blocks[b];
            const int64_t ro = lr0 - B.r0;
            if (B.kind != KIND_LR) {
                if (B.fill_entries) {
                    fill.insert(fill.end(), {off, lr0, lm, B.c0, B.n});
                } else {
                    pack.insert(pack.end(), {off, (int64_t)(uintptr_t)(B.dense + ro * B.d_rs), lm, B.n, B.d_rs, B.d_cs});
                }
                for (int64_t j = 0; j < B.n; ++j) op.h_colsrc.push_back((int32_t)(B.c0 + j));
                op.items.push_back(HOp::ItemRec{off, -1, lr0, lm, B.c0, B.n, 0});
                off += lm * B.n;
                row.ncols += (int32_t)B.n;
                op.p2_doubles += lm * B.n;
            } else {
                pack.insert(pack.end(), {off, (int64_t)(uintptr_t)(B.U + ro), lm, (int64_t)B.k, 1, B.u_ld});
                for (int q = 0; q < B.k; ++q) op.h_colsrc.push_back((int32_t)(n + tbase[b] + q));
                op.items.push_back(HOp::ItemRec{off, vtoff[b], lr0, lm, B.c0, B.n, B.k});
                off += lm * B.k;
                row.ncols += B.k;
                op.p2_doubles += lm * B.k;
            }
        }
        op.h_p2.push_back(row);
        off = align2(off);
    }
    if ((int64_t)n + tcount >= INT32_MAX) throw Error(HM_ERR_UNSUPPORTED, "n + total rank exceeds int32 index space");
    op.max_m = max_m;
    op.n_p1 = (int64_t)p1.size();
    op.n_p2 = (int64_t)op.h_p2.size();
    op.n_cols = (int64_t)op.h_colsrc.size();
    op.arena.alloc(ctx, (size_t)std::max<int64_t>(off, 2), "operator arena");
    op.p1.upload(ctx, p1, "phase-1 tasks", s);
    op.p2.upload(ctx, op.h_p2, "phase-2 rows", s);
    op.colsrc.upload(ctx, op.h_colsrc, "colsrc", s);
    DBuf<int64_t> d_pack, d_fill;
    d_pack.upload(ctx, pack, "pack tasks", s);
    d_fill.upload(ctx, fill, "fill tasks", s);
    k::pack(d_pack.p, (int)(pack.size() / 6), op.arena.p, nullptr, s);
    static_assert(sizeof(int64_t) == sizeof(void*), "pointer size");
    if (!fill.empty()) {
        DBuf<int32_t> err;
        err.alloc(ctx, 4, "err");
        HM_CUDA(cudaMemsetAsync(err.p, 0, 4 * sizeof(int32_t), s));
        k::fill_entries(g.d_geo.p, n, d_fill.p, (int)(fill.size() / 5), op.arena.p, err.p, s);
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
