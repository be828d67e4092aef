// Operator builder: flattens a set of blocks (dense + low-rank U V^T) into the two-pass
// column-stream layout of the hot path:
//
//   arena = [ phase-1 panels: per column cluster tau, the V^T of every low-rank block (., tau)
//             stacked: column-major, ld = K_tau (even), n_tau columns                        ]
//           [ phase-2 panels: per leaf row r, the leaf-row slices of every dense block and U
//             factor covering r: column-major, ld = m_r (even), in block order              ]
//   colsrc[c] = index into XT = [x (n) | t (sum k)] of the input multiplying column c.
// Panels have <= 128 rows and are cut into work units of <= kStageDoubles (single vector, 56.6 KB)
// or kUnitPayloadDoubles (multi-RHS, 32 KB) of contiguous payload.
#include <algorithm>
#include <cstdlib>
#include <map>

#include "hm_internal.h"

namespace hm {

static inline int64_t align2(int64_t x) { return (x + 1) & ~int64_t(1); }

// experiment knobs (piece sizing): positive integers only, else the default
static int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    if (!e) return dflt;
    const int v = atoi(e);
    return v >= 1 && v <= 1 << 20 ? v : dflt;
}

static bool force_colsrc() {
    const char* e = getenv("HM_FORCE_COLSRC");
    return e && e[0] == '1';
}

// Cut panels into pieces (only panels above 512 KB are split, for load balance) and pieces into
// chunks of <= one engine stage of contiguous payload (<= 256 columns), each chunk with its own 16-byte
// aligned column-source segment (so the engine can TMA both).
// max_cols: columns per chunk (single vector: kUnitMaxCols; multi-RHS: kMrhsMaxCols); part_scale:
// partial-sum doubles per panel row (1, or kMrhsMax for the multi-RHS units)
static void make_units(Ctx* ctx, StreamPass& P, const std::vector<int32_t>& pcs, std::vector<int32_t>& ucs,
                       cudaStream_t s, int max_cols = kUnitMaxCols, int part_scale = 1, bool split_xonly = true,
                       int order = 0 /* 0: largest first; 1: all pieces by key; 2: t-reading pieces by key */,
                       int64_t max_doubles = kUnitPayloadDoubles /* payload doubles per chunk */) {
    std::vector<Unit>& units = P.h_units;
    units.clear();
    P.unit_panel.clear();
    P.unit_xonly.clear();
    int64_t part = 0;
    int32_t grp = 0;
    // piece size adapted to the pass: ~2 tasks per SM (small passes still spread over the chip),
    // between four chunks and kPieceDoubles (measured on C2: 2 per SM 193 us, 4 per SM 197 us,
    // 8 per SM 209 us -- fewer split-K partials beat a shorter pass tail); HM_PIECE_DIV /
    // HM_PIECE_MIN override for experiments
    int64_t pass_doubles = 0;
    for (const Panel& pn : P.panels) pass_doubles += (int64_t)pn.ncols * pn.ld;
    static const int piece_div = env_int("HM_PIECE_DIV", 2);
    static const int piece_min = env_int("HM_PIECE_MIN", 4);
    static const int mrhs_min = env_int("HM_MRHS_PIECE_MIN", 64);   // measured C2 64-RHS flux: 4 -> 1.46, 64 -> 1.35 ms
    // multi-RHS units (part_scale > 1): compute-bound, and every split piece costs a rows x 64 partial
    // write + combine, so only panels above mrhs_min chunks (HM_MRHS_PIECE_MIN) are split
    const int64_t piece = part_scale > 1
        ? std::max<int64_t>((int64_t)mrhs_min * kUnitPayloadDoubles,
                            std::min<int64_t>(kPieceDoubles, pass_doubles / (piece_div * 148)))
        : std::max<int64_t>(piece_min * kUnitPayloadDoubles,
                            std::min<int64_t>(kPieceDoubles, pass_doubles / (piece_div * 148)));
    struct Piece { std::vector<Unit> u; std::vector<int32_t> cs; int32_t panel; int64_t doubles; uint8_t xonly; int64_t key; };
    std::vector<Piece> pieces;
    for (size_t pi = 0; pi < P.panels.size(); ++pi) {
        const Panel& pn = P.panels[pi];
        if (pn.ncols == 0) continue;
        // two column segments: [0, ndense) reads only x (may run before the t values exist),
        // [ndense, ncols) reads t; each is cut into pieces, all pieces of the panel combine
        struct Seg { int64_t c0, c1; int32_t np; };
        // (multi-RHS: no split -- the kernel is compute-bound, and every extra piece costs a
        // rows x 64 partial write + combine)
        const int64_t nd = split_xonly ? pn.ndense : 0;
        Seg segs[2] = {{0, nd, 0}, {nd, pn.ncols, 0}};
        int32_t npieces = 0;
        for (Seg& sg : segs) {
            const int64_t w = sg.c1 - sg.c0;
            if (w <= 0) continue;
            // t-reading segments of split passes (phase 2) end the pass: optionally finer pieces there
            static const int tdiv = env_int("HM_PIECE_TDIV", 2);   // measured: 1 -> 184.7, 2 -> 183.4 us
            const int64_t pc_sz = (&sg == &segs[1] && nd > 0) ? std::max<int64_t>(2 * kUnitPayloadDoubles, piece / tdiv) : piece;
            sg.np = (int32_t)std::min<int64_t>(w, (w * pn.ld + pc_sz - 1) / pc_sz);
            npieces += sg.np;
        }
        const int32_t g = npieces > 1 ? grp++ : -1;
        int32_t pc = 0;
        for (int sgi = 0; sgi < 2; ++sgi) {
            const Seg& sg = segs[sgi];
            if (sg.np == 0) continue;
            const int64_t Cp = (sg.c1 - sg.c0 + sg.np - 1) / sg.np;
            for (int32_t q = 0; q < sg.np; ++q, ++pc) {
                const int64_t p0 = sg.c0 + q * Cp, p1 = std::min<int64_t>(sg.c1, p0 + Cp);
                if (p1 <= p0) { --pc; continue; }
                int64_t C = std::min<int64_t>(max_cols, max_doubles / pn.ld);
                const int32_t nch = (int32_t)((p1 - p0 + C - 1) / C);
                C = (p1 - p0 + nch - 1) / nch;
                Piece PC;
                PC.panel = (int32_t)pi;
                PC.key = pn.key;
                PC.doubles = (p1 - p0) * pn.ld;
                PC.xonly = p1 <= pn.ndense ? 1 : 0;   // reads only x (no t)
                for (int32_t ch = 0; ch < nch; ++ch) {
                    Unit u{};
                    const int64_t c0 = p0 + ch * C;
                    u.ncols = (int32_t)std::min<int64_t>(C, p1 - c0);
                    u.a_off = pn.a_off + c0 * pn.ld;
                    u.out0 = pn.out0;
                    u.part_off = (part + (npieces > 1 ? (int64_t)pc * pn.ld : 0)) * part_scale;
                    u.cs_off = (int64_t)PC.cs.size();   // relative; rebased below
                    for (int32_t c = 0; c < u.ncols; ++c) PC.cs.push_back(pcs[pn.cs_off + c0 + c]);
                    {   // run-length form of the column sources
                        const int32_t* src = &pcs[pn.cs_off + c0];
                        int nr = 0;
                        bool ok = true;
                        for (int32_t c = 0; c < u.ncols && ok; ++c) {
                            if (c > 0 && src[c] == src[c - 1] + 1 && u.run_len[nr - 1] < 65535) {
                                ++u.run_len[nr - 1];
                            } else if (nr < kMaxRuns) {
                                u.run_src[nr] = src[c];
                                u.run_len[nr] = 1;
                                ++nr;
                            } else {
                                ok = false;
                            }
                        }
                        // HM_FORCE_COLSRC=1 (tests): every chunk takes the per-column colsrc path
                        u.nruns = ok && !force_colsrc() ? nr : 0;
                    }
                    while (PC.cs.size() % 4) PC.cs.push_back(0);
                    u.ld = pn.ld;
                    u.nrows = pn.nrows;
                    u.grp = g;
                    u.seg = pc;
                    u.pass = 0;
                    u.type = UNIT_STREAM;
                    u.chunk = ch;
                    u.nchunks = nch;
                    PC.u.push_back(u);
                }
                pieces.push_back(std::move(PC));
            }
        }
        for (size_t q = pieces.size() - pc; q < pieces.size(); ++q)
            for (Unit& u : pieces[q].u) u.nseg = pc;
        if (pc > 1) part += (int64_t)pc * pn.ld;
        else for (size_t q = pieces.size() - pc; q < pieces.size(); ++q) for (Unit& u : pieces[q].u) { u.grp = -1; u.part_off = 0; }
    }
    // x-only pieces first, then largest first (tasks are taken in order: a pass starts with work that
    // needs no t values and ends on small tasks)
    // (order 1 / 2: all pieces / the t-reading pieces in panel-key order instead, so the row groups of
    // Program::link_rows become ready, or complete, one after another)
    std::stable_sort(pieces.begin(), pieces.end(), [order](const Piece& a, const Piece& b) {
        if (a.xonly != b.xonly) return a.xonly > b.xonly;
        if ((order == 1 || (order == 2 && !a.xonly)) && a.key != b.key) return a.key < b.key;
        return a.doubles > b.doubles;
    });
    for (Piece& PC : pieces) {
        const int64_t first = (int64_t)units.size();
        const int64_t cs0 = (int64_t)ucs.size();
        ucs.insert(ucs.end(), PC.cs.begin(), PC.cs.end());
        for (Unit& u : PC.u) {
            u.cs_off += cs0;
            u.first_chunk = first;
            units.push_back(u);
            P.unit_panel.push_back(PC.panel);
            P.unit_xonly.push_back(PC.xonly);
        }
    }
    P.n_units = (int64_t)units.size();
    P.part.alloc(ctx, (size_t)std::max<int64_t>(part * part_scale, 2), "split-K partials");
    P.counters.alloc(ctx, (size_t)std::max<int32_t>(grp, 1), "split-K counters");
    HM_CUDA(cudaMemsetAsync(P.counters.p, 0, sizeof(int32_t) * std::max<int32_t>(grp, 1), s));
}

void build_hop(Ctx* ctx, const Geom& g, std::vector<SrcBlock>& blocks, HOp& op, cudaStream_t s, const Shard* sh,
               int64_t t_off, const double* quad) {
    const int64_t n = g.n;
    // sharded: only blocks with rows on this rank; x indices and outputs in the
    // padded layout (x region of XT = n_pad), t after it
    const bool shd = sh && sh->sharded();
    const int64_t nx = shd ? sh->n_pad() : n;
    auto xi = [&](int64_t i) -> int32_t { return (int32_t)(shd ? sh->pad(i) : i); };
    auto mine = [&](const SrcBlock& B) { return !shd || (B.r0 < sh->le() && B.r0 + B.m > sh->lb()); };
    op.n_x = nx;
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
        if (!mine(B)) continue;
        if (B.kind != KIND_LR) { ++op.n_dense; continue; }
        if (B.k > 128)   // a phase-1 panel stacks whole blocks of <= 128 rows (callers split larger ranks)
            throw Error(HM_ERR_UNSUPPORTED, "low-rank block of rank " + std::to_string(B.k) + " > 128 in the operator builder");
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
        size_t q0 = 0;
        while (q0 < members.size()) {           // sub-panels of <= 128 rows, whole blocks each
            size_t q1 = q0;
            int64_t K = 0;
            while (q1 < members.size() && K + blocks[members[q1]].k <= 128) K += blocks[members[q1++]].k;
            const SrcBlock& B0 = blocks[members[q0]];
            const int64_t ld = align2(K);
            Panel pn{off, nx + t_off + tcount, (int32_t)ld, (int32_t)K, (int32_t)B0.n, (int32_t)colsrc.size(), B0.c0,
                     (int32_t)B0.n};
            for (int64_t j = 0; j < B0.n; ++j) colsrc.push_back(xi(B0.c0 + j));
            int64_t local = 0;
            for (size_t q = q0; q < q1; ++q) {
                const int b = members[q];
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
            q0 = q1;
        }
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
        if (shd && !(L.begin >= sh->lb() && L.end <= sh->le())) continue;   // another rank's leaf row
        for (int64_t rc = L.begin; rc < L.end; rc += 128) {   // row chunks of <= 128
            const int64_t lr0 = rc, lm = std::min<int64_t>(128, L.end - rc), ld = align2(lm);
            Panel pn{off, xi(lr0), (int32_t)ld, (int32_t)lm, 0, (int32_t)colsrc.size(), lr0, 0};
            // dense blocks first (they read only x), then the U factors (they read t)
            std::vector<int> order;
            for (int b : items[l]) if (blocks[b].kind != KIND_LR) order.push_back(b);
            pn.ndense = 0;
            for (int b : order) pn.ndense += (int32_t)blocks[b].n;
            for (int b : items[l]) if (blocks[b].kind == KIND_LR) order.push_back(b);
            for (int b : order) {
                const SrcBlock& B = blocks[b];
                const int64_t ro = lr0 - B.r0;
                if (B.kind != KIND_LR) {
                    if (B.fill_entries)
                        fill.insert(fill.end(), {off, lr0, lm, B.c0, B.n, ld});
                    else
                        pack.insert(pack.end(), {off, (int64_t)(uintptr_t)(B.dense + ro * B.d_rs), lm, B.n, B.d_rs, B.d_cs, ld});
                    for (int64_t j = 0; j < B.n; ++j) colsrc.push_back(xi(B.c0 + j));
                    op.items.push_back(HOp::ItemRec{off, ld, -1, 0, lr0, lm, B.c0, B.n, 0});
                    off += ld * B.n;
                    pn.ncols += (int32_t)B.n;
                    op.p2.doubles += lm * B.n;
                } else {
                    pack.insert(pack.end(), {off, (int64_t)(uintptr_t)(B.U + ro), lm, (int64_t)B.k, 1, B.u_ld, ld});
                    for (int q = 0; q < B.k; ++q) colsrc.push_back((int32_t)(nx + t_off + tbase[b] + q));
                    op.items.push_back(HOp::ItemRec{off, ld, voff[b], vld[b], lr0, lm, B.c0, B.n, B.k});
                    off += ld * B.k;
                    pn.ncols += B.k;
                    op.p2.doubles += lm * B.k;
                }
            }
            op.p2.panels.push_back(pn);
        }
    }
    if (nx + t_off + tcount >= INT32_MAX || (int64_t)colsrc.size() >= INT32_MAX)
        throw Error(HM_ERR_UNSUPPORTED, "index space exceeds int32");

    op.xt_len = nx + t_off + tcount;
    op.arena.alloc(ctx, (size_t)std::max<int64_t>(off, 2), "operator arena");
    HM_CUDA(cudaMemsetAsync(op.arena.p, 0, sizeof(double) * (size_t)std::max<int64_t>(off, 2), s));
    std::vector<int32_t> ucs;
    const int64_t chunk_doubles = kStageDoubles;   // chunk payload cap: one engine stage (56.6 KB)
    make_units(ctx, op.p1, colsrc, ucs, s, kUnitMaxCols, 1, true, op.p1_by_key ? 1 : 0, chunk_doubles);
    make_units(ctx, op.p2, colsrc, ucs, s, kUnitMaxCols, 1, true, op.p2_by_row ? 2 : 0, chunk_doubles);
    {   // multi-RHS chunking of the same panels (<= kMrhsMaxCols columns: X tile in smem)
        op.p1m.panels = op.p1.panels;
        op.p2m.panels = op.p2.panels;
        op.p1m.doubles = op.p1.doubles;
        op.p2m.doubles = op.p2.doubles;
        // largest pieces first (load balance; measured on the C2 64-RHS flux: cluster / row order with
        // row-group links 0.927 ms, without links 1.005 ms, largest first 0.913 ms); HM_MRHS_KEY_ORDER=1
        // selects the keyed order
        static const bool keyed = getenv("HM_MRHS_KEY_ORDER") != nullptr;
        make_units(ctx, op.p1m, colsrc, ucs, s, kMrhsMaxCols, kMrhsMax, false, keyed && op.p1_by_key ? 1 : 0,
                   kMrhsPayloadDoubles);
        make_units(ctx, op.p2m, colsrc, ucs, s, kMrhsMaxCols, kMrhsMax, false, keyed && op.p2_by_row ? 2 : 0,
                   kMrhsPayloadDoubles);
    }
    op.colsrc.upload(ctx, ucs, "colsrc", s);
    // the same column sources for passes that gather straight from the caller's external-order
    // vector (fused prologue): x-region index j becomes -(perm[j] + 1)
    if (!shd) {
        for (int32_t& j : ucs)
            if (j < n) j = -(g.perm[j] + 1);
        op.colsrc_ext.upload(ctx, ucs, "colsrc (external)", s);
    }
    DBuf<int64_t> d_pack, d_fill;
    d_pack.upload(ctx, pack, "pack tasks", s);
    d_fill.upload(ctx, fill, "fill tasks", s);
    k::pack(d_pack.p, (int)(pack.size() / 7), op.arena.p, s);
    static_assert(sizeof(int64_t) == sizeof(void*), "pointer size");
    if (!fill.empty()) {
        DBuf<int32_t> err;
        err.alloc(ctx, 4, "err");
        HM_CUDA(cudaMemsetAsync(err.p, 0, 4 * sizeof(int32_t), s));
        k::fill_entries(g.d_geo.p, n, d_fill.p, (int)(fill.size() / 6), op.arena.p, err.p, s, quad);
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
