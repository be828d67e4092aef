// One-time factorisation of C = I - Lambda F and the level-scheduled
// substitution that applies C^-1, DESIGN.md §"Solve in level form".
//
// Two factorisations produce the same factor set (the forms of reading R27):
//  * stage B (default, hla.cpp, reading R33): hierarchical arithmetic on C's blocks in F's
//    partition -- the paper's 4-step recursion with recursive substitutions and block products,
//    every low-rank sum truncated at eps_LU; any n.  C's blocks are read back
//    from F's arena (C = I - Lambda F block by block), factored on the host (OpenMP
//    tasks over independent blocks) and the solve-form blocks uploaded for the packer.
//  * stage A (method 1, n up to ~1e5): C expanded dense on the GPU, the same recursion on dense
//    tiles with FP64 DMMA carrying the triangular inverses, then truncation block by block in F's
//    partition by cross approximation with full pivoting.
// Both give, per internal node t above the cut level,
//     W^L_t = L21 L11^-1      W^U_t = U12 U22^-1
// and below it the inverse factors of the cut-level diagonal blocks (cut 0: L^-1 and U^-1).
//
// Solve: for levels top-down  b_t2 -= W^L_t b_t1   (one two-phase launch pair per level),
//        leaves              y_r  = L_rr^-1 b_r,
//        for levels top-down  y_t1 -= W^U_t y_t2,
//        leaves              z_r  = U_rr^-1 y_r.
// This re-associates the forward/backward substitution (same C^-1 in exact arithmetic) so that
// all nodes of a level are independent.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <malloc.h>
#include <memory>

#include <unordered_map>

#include "hla.h"
#include "hm_internal.h"

namespace hm {

namespace {

struct Factorizer {
    HLU& L;
    const HMat& F;
    const Geom& g;
    Ctx* c;
    cudaStream_t s;
    int64_t n;
    double eps_lu;
    double* M = nullptr;
    double* Minv = nullptr;
    double* T = nullptr;
    int32_t* err = nullptr;
    std::vector<std::vector<int>> lower, upper;          // F-block ids per tree node
    std::vector<std::vector<SrcBlock>> fwd_src, bwd_src;  // per level
    std::vector<DBuf<double>> staging;

    static constexpr int KMAX_LU = 64;
    int cut = 0;  // W blocks are formed only for tree nodes above the cut level

    void collect() {
        lower.assign(g.nodes.size(), {});
        upper.assign(g.nodes.size(), {});
        for (size_t b = 0; b < g.blocks.size(); ++b) {
            const Blk& B = g.blocks[b];
            int r = B.rnode, q = B.cnode;
            if (r == q) continue;  // leaf diagonal block: part of the leaf factors
            while (g.nodes[r].parent != g.nodes[q].parent) {
                r = g.nodes[r].parent;
                q = g.nodes[q].parent;
            }
            const int t = g.nodes[r].parent;
            const Node& Tn = g.nodes[t];
            if (B.r0 >= g.nodes[Tn.child[1]].begin) lower[t].push_back((int)b);
            else upper[t].push_back((int)b);
        }
    }

    // Stage the blocks of W (in T, rows b_rows.., cols b_cols.., ld) into staging buffers.
    // Phase A (before T is destroyed): dense copies.  Phase B: compress admissible blocks in place.
    void stage_dense(const std::vector<int>& ids, int64_t row0, int64_t col0, int64_t ld, std::vector<SrcBlock>& out) {
        std::vector<int64_t> tasks;
        int64_t tot = 0;
        std::vector<std::pair<int, int64_t>> place;
        for (int b : ids) {
            const Blk& B = g.blocks[b];
            if (B.adm) continue;
            const int64_t m = B.r1 - B.r0, nn = B.c1 - B.c0;
            place.push_back({b, tot});
            tot += m * nn;
        }
        if (place.empty()) return;
        DBuf<double> buf;
        buf.alloc(c, (size_t)tot, "W dense staging");
        for (auto& pr : place) {
            const Blk& B = g.blocks[pr.first];
            const int64_t m = B.r1 - B.r0, nn = B.c1 - B.c0;
            const double* src = T + (B.r0 - row0) * ld + (B.c0 - col0);
            tasks.insert(tasks.end(), {pr.second, (int64_t)(uintptr_t)src, m, nn, ld, 1, m});
            SrcBlock S;
            S.r0 = B.r0; S.m = m; S.c0 = B.c0; S.n = nn;
            S.kind = KIND_DENSE;
            S.dense = buf.p + pr.second;
            S.d_rs = 1;
            S.d_cs = m;  // staged column-major
            out.push_back(S);
        }
        DBuf<int64_t> d;
        d.upload(c, tasks, "stage tasks", s);
        k::pack(d.p, (int)(tasks.size() / 7), buf.p, s);
        HM_CUDA(cudaStreamSynchronize(s));
        staging.push_back(std::move(buf));
    }

    void compress(const std::vector<int>& ids, int64_t row0, int64_t col0, int64_t ld, std::vector<SrcBlock>& out) {
        std::vector<int64_t> blk;
        std::vector<int32_t> kcap;
        std::vector<int> which;
        int64_t tot = 0;
        for (int b : ids) {
            const Blk& B = g.blocks[b];
            if (!B.adm) continue;
            const int64_t m = B.r1 - B.r0, nn = B.c1 - B.c0;
            const int64_t klim = (m * nn + m + nn - 1) / (m + nn);
            const int kc = (int)std::min<int64_t>(KMAX_LU, klim);
            const int64_t uo = tot;
            tot += (m * kc + 1) & ~1LL;
            const int64_t vo = tot;
            tot += (nn * kc + 1) & ~1LL;
            blk.insert(blk.end(), {B.r0 - row0, m, B.c0 - col0, nn, uo, vo, 0});
            kcap.push_back(kc);
            which.push_back(b);
        }
        if (which.empty()) return;
        DBuf<double> fac;
        fac.alloc(c, (size_t)std::max<int64_t>(tot, 2), "W factor staging");
        DBuf<int64_t> dblk;
        DBuf<int32_t> dk, dr;
        dblk.upload(c, blk, "cpaca blocks", s);
        dk.upload(c, kcap, "cpaca kcap", s);
        dr.alloc(c, which.size(), "cpaca ranks");
        k::cpaca_batch(T, ld, dblk.p, dk.p, (int)which.size(), eps_lu, fac.p, dr.p, s);
        std::vector<int32_t> rk(which.size());
        HM_CUDA(cudaMemcpyAsync(rk.data(), dr.p, rk.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        HM_CUDA(cudaStreamSynchronize(s));
        std::vector<int> failed;
        for (size_t q = 0; q < which.size(); ++q) {
            const Blk& B = g.blocks[which[q]];
            const int64_t m = B.r1 - B.r0, nn = B.c1 - B.c0;
            if (rk[q] < 0) { failed.push_back(which[q]); continue; }
            SrcBlock S;
            S.r0 = B.r0; S.m = m; S.c0 = B.c0; S.n = nn;
            S.kind = KIND_LR;
            S.k = rk[q];
            S.U = fac.p + blk[7 * q + 4];
            S.u_ld = m;
            S.V = fac.p + blk[7 * q + 5];
            S.v_ld = nn;
            out.push_back(S);
        }
        staging.push_back(std::move(fac));
        if (!failed.empty()) {  // restored dense in T: stage them as dense
            std::vector<int> tmp;
            for (int b : failed) tmp.push_back(b);
            // temporarily mark as dense for staging
            std::vector<SrcBlock> dense_out;
            std::vector<int64_t> tasks;
            int64_t t2 = 0;
            for (int b : tmp) {
                const Blk& B = g.blocks[b];
                t2 += (B.r1 - B.r0) * (B.c1 - B.c0);
            }
            DBuf<double> buf;
            buf.alloc(c, (size_t)t2, "W dense staging (failed compression)");
            int64_t off = 0;
            for (int b : tmp) {
                const Blk& B = g.blocks[b];
                const int64_t m = B.r1 - B.r0, nn = B.c1 - B.c0;
                tasks.insert(tasks.end(), {off, (int64_t)(uintptr_t)(T + (B.r0 - row0) * ld + (B.c0 - col0)), m, nn, ld, 1, m});
                SrcBlock S;
                S.r0 = B.r0; S.m = m; S.c0 = B.c0; S.n = nn;
                S.kind = KIND_DENSE;
                S.dense = buf.p + off;
                S.d_rs = 1;
                S.d_cs = m;
                out.push_back(S);
                off += m * nn;
            }
            DBuf<int64_t> d;
            d.upload(c, tasks, "stage tasks", s);
            k::pack(d.p, (int)(tasks.size() / 7), buf.p, s);
            HM_CUDA(cudaStreamSynchronize(s));
            staging.push_back(std::move(buf));
        }
    }

    double* Mp(int64_t r, int64_t col) { return M + r * n + col; }
    double* Ip(int64_t r, int64_t col) { return Minv + r * n + col; }

    void rec(int node, int64_t b1, int64_t size) {
        const bool tree_internal = node >= 0 && !g.nodes[node].is_leaf();
        if (!tree_internal && size <= 64) {
            k::leaf_lu_inv(Mp(b1, b1), Ip(b1, b1), n, (int)size, err, s);
            return;
        }
        const int64_t n1 = tree_internal ? g.nodes[g.nodes[node].child[0]].size() : (size + 1) / 2;
        const int64_t n2 = size - n1, b2 = b1 + n1;
        const int ch0 = tree_internal ? g.nodes[node].child[0] : -1;
        const int ch1 = tree_internal ? g.nodes[node].child[1] : -1;
        rec(ch0, b1, n1);
        // step 2: U12 = L11^-1 C12 ; step 3: L21 = C21 U11^-1 ; step 4: C22 -= L21 U12
        k::dgemm(n1, n2, n1, 1.0, Ip(b1, b1), n, 1, Mp(b1, b2), n, 0, 0.0, T, n2, s);
        k::copy2d(T, n2, Mp(b1, b2), n, n1, n2, s);
        k::dgemm(n2, n1, n1, 1.0, Mp(b2, b1), n, 0, Ip(b1, b1), n, 2, 0.0, T, n1, s);
        k::copy2d(T, n1, Mp(b2, b1), n, n2, n1, s);
        k::dgemm(n2, n2, n1, -1.0, Mp(b2, b1), n, 0, Mp(b1, b2), n, 0, 1.0, Mp(b2, b2), n, s);
        rec(ch1, b2, n2);
        // W^L = L21 L11^-1 ; (L^-1)21 = -L22^-1 W^L
        k::dgemm(n2, n1, n1, 1.0, Mp(b2, b1), n, 0, Ip(b1, b1), n, 1, 0.0, T, n1, s);
        const int lvl = tree_internal ? g.nodes[node].level : -1;
        const bool wform = tree_internal && lvl < cut;
        if (wform) stage_dense(lower[node], b2, b1, n1, fwd_src[lvl]);
        k::dgemm(n2, n1, n2, -1.0, Ip(b2, b2), n, 1, T, n1, 0, 0.0, Ip(b2, b1), n, s);
        if (wform) compress(lower[node], b2, b1, n1, fwd_src[lvl]);
        // W^U = U12 U22^-1 ; (U^-1)12 = -U11^-1 W^U
        k::dgemm(n1, n2, n2, 1.0, Mp(b1, b2), n, 0, Ip(b2, b2), n, 2, 0.0, T, n2, s);
        if (wform) stage_dense(upper[node], b1, b2, n2, bwd_src[lvl]);
        k::dgemm(n1, n2, n1, -1.0, Ip(b1, b1), n, 2, T, n2, 0, 0.0, Ip(b1, b2), n, s);
        if (wform) compress(upper[node], b1, b2, n2, bwd_src[lvl]);
    }
};

// The blocks of the solve forms (reading R27), as sources for the operator builder.
struct FactorSet {
    std::vector<std::vector<SrcBlock>> fwd, bwd;   // W^L_t / W^U_t blocks per tree level < cut
    std::vector<SrcBlock> srcL, srcU;              // inverse factors of the cut-level diagonal blocks
    std::vector<DBuf<double>> staging;             // device payload the sources point into
};

// ---- stage A: dense tiles on the GPU (reading R28)
void stage_a(HLU& L, const HMat& F, const Geom& g, const std::vector<double>& lam, int Lc, FactorSet& out) {
    Ctx* c = L.ctx;
    const cudaStream_t s = c->stream;
    const int64_t n = g.n;
    const int64_t half = (n + 1) / 2;
    const int64_t maxT = std::max<int64_t>(half * (n - half), 1);
    const double need = 8.0 * (2.0 * n * n + maxT) * 1.25;
    size_t freeb = 0, totb = 0;
    HM_CUDA(cudaMemGetInfo(&freeb, &totb));
    if (need > (double)freeb)
        throw Error(HM_ERR_UNSUPPORTED, "dense-stage H-LU needs ~" + std::to_string((int64_t)(need / 1e9)) +
                                            " GB of device memory (" + std::to_string((int64_t)(freeb / 1e9)) + " GB free)");
    DBuf<double> dlam, dM, dMinv, dT;
    DBuf<int32_t> derr;
    dlam.upload(c, lam, "lambda", s);
    dM.alloc(c, (size_t)(n * n), "dense C / LU");
    dMinv.alloc(c, (size_t)(n * n), "dense L^-1 / U^-1");
    dT.alloc(c, (size_t)maxT, "W workspace");
    derr.alloc(c, 4, "err");
    HM_CUDA(cudaMemsetAsync(derr.p, 0, 4 * sizeof(int32_t), s));

    // ---- C = I - Lambda F_H expanded from the stored H-format
    double t0 = now_seconds();
    HM_CUDA(cudaMemsetAsync(dM.p, 0, sizeof(double) * (size_t)(n * n), s));
    {
        std::vector<int64_t> tasks;
        tasks.reserve(10 * F.op.items.size());
        for (const auto& it : F.op.items)
            tasks.insert(tasks.end(), {it.a_off, it.a_ld, it.v_off, it.v_ld, it.r0, it.m, it.c0, it.ncols, it.k, 0});
        DBuf<int64_t> d;
        d.upload(c, tasks, "expand tasks", s);
        k::expand_C(d.p, (int)F.op.items.size(), F.op.arena.p, dlam.p, dM.p, n, s);
        k::add_identity(dM.p, n, n, s);
        HM_CUDA(cudaStreamSynchronize(s));
    }
    L.setup_seconds[0] = now_seconds() - t0;

    // ---- block LU over the cluster tree with level-form W extraction
    t0 = now_seconds();
    Factorizer fz{L, F, g, c, s, n, L.params.eps_lu};
    fz.M = dM.p;
    fz.Minv = dMinv.p;
    fz.T = dT.p;
    fz.err = derr.p;
    fz.collect();
    fz.cut = Lc;
    fz.fwd_src.assign(std::max(Lc, 0), {});
    fz.bwd_src.assign(std::max(Lc, 0), {});
    fz.rec(0, 0, n);
    int32_t herr[4];
    HM_CUDA(cudaMemcpyAsync(herr, derr.p, sizeof(herr), cudaMemcpyDeviceToHost, s));
    HM_CUDA(cudaStreamSynchronize(s));
    if (herr[0]) throw Error(HM_ERR_SINGULAR, "near-zero pivot (|pivot| <= 1e-14 ||block||) in a leaf LU of C");
    // cut nodes: level == Lc, or leaves shallower than Lc
    std::vector<int> cut_nodes;
    {
        std::vector<int> st{0};
        while (!st.empty()) {
            const int t = st.back();
            st.pop_back();
            const Node& N = g.nodes[t];
            if (N.level == Lc || N.is_leaf()) { cut_nodes.push_back(t); continue; }
            st.push_back(N.child[1]);
            st.push_back(N.child[0]);
        }
    }
    // leaf diagonal inverses (masked unit-lower / upper)
    int64_t leaf_tot = 0;
    for (int l : g.leaves) leaf_tot += g.nodes[l].size() * g.nodes[l].size();
    DBuf<double> dLi, dUi;
    dLi.alloc(c, (size_t)leaf_tot, "leaf L^-1");
    dUi.alloc(c, (size_t)leaf_tot, "leaf U^-1");
    int64_t off = 0;
    for (int l : g.leaves) {
        const Node& N = g.nodes[l];
        const int64_t m = N.size();
        k::extract_tri(dMinv.p, n, N.begin, m, 1, dLi.p + off, s);
        k::extract_tri(dMinv.p, n, N.begin, m, 2, dUi.p + off, s);
        SrcBlock S;
        S.r0 = N.begin; S.m = m; S.c0 = N.begin; S.n = m;
        S.kind = KIND_DENSE;
        S.d_rs = m;
        S.d_cs = 1;
        S.dense = dLi.p + off;
        out.srcL.push_back(S);
        S.dense = dUi.p + off;
        out.srcU.push_back(S);
        off += m * m;
    }
    HM_CUDA(cudaStreamSynchronize(s));
    // off-diagonal blocks of the cut diagonal blocks' inverse factors, compressed in F's partition
    // straight out of L^-1 / U^-1 (dense blocks staged first, admissible blocks truncated in place)
    fz.T = dMinv.p;
    for (int t0n : cut_nodes) {
        std::vector<int> st{t0n};
        while (!st.empty()) {
            const int t = st.back();
            st.pop_back();
            const Node& N = g.nodes[t];
            if (N.is_leaf()) continue;
            fz.stage_dense(fz.lower[t], 0, 0, n, out.srcL);
            fz.stage_dense(fz.upper[t], 0, 0, n, out.srcU);
            fz.compress(fz.lower[t], 0, 0, n, out.srcL);
            fz.compress(fz.upper[t], 0, 0, n, out.srcU);
            st.push_back(N.child[0]);
            st.push_back(N.child[1]);
        }
    }
    HM_CUDA(cudaStreamSynchronize(s));
    L.setup_seconds[1] = now_seconds() - t0;
    out.fwd = std::move(fz.fwd_src);
    out.bwd = std::move(fz.bwd_src);
    for (auto& b : fz.staging) out.staging.push_back(std::move(b));
    out.staging.push_back(std::move(dLi));
    out.staging.push_back(std::move(dUi));
}

}  // namespace

// ---- reading an operator's payload back from its arena (stage B input, hm_export_factors)
// For every phase-2 item (a leaf-row slice of a block): its payload (dense m x ncols, or the U slice
// m x k, column-major) and, when want_v(item) is true and the item is low rank, the block's V
// (ncols x k, column-major), staged through the device in batches of <= 64 Mi doubles.
void read_items(Ctx* c, const HOp& op, const std::function<bool(size_t)>& want_v,
                const std::function<void(size_t, const double*, const double*)>& fn) {
    const cudaStream_t s = c->stream;
    const int64_t budget = int64_t(1) << 26;
    const size_t ni = op.items.size();
    size_t i0 = 0;
    DBuf<double> stage;
    // pinned host staging (one buffer for the whole read-back: several times the pageable bandwidth)
    struct Pinned {
        double* p = nullptr;
        size_t n = 0;
        ~Pinned() { if (p) cudaFreeHost(p); }
        double* get(size_t want) {
            if (want > n) {
                if (p) cudaFreeHost(p);
                p = nullptr;
                if (cudaMallocHost(&p, want * sizeof(double)) != cudaSuccess) throw Error(HM_ERR_OOM, "pinned read-back staging");
                n = want;
            }
            return p;
        }
    } host;
    while (i0 < ni) {
        std::vector<int64_t> tasks;
        std::vector<int64_t> po, vo;
        int64_t tot = 0;
        size_t i1 = i0;
        for (; i1 < ni; ++i1) {
            const HOp::ItemRec& it = op.items[i1];
            const bool lr = it.v_off >= 0;
            const int64_t cols = lr ? it.k : it.ncols;
            const bool wv = lr && it.k > 0 && want_v(i1);
            const int64_t need = it.m * cols + (wv ? it.ncols * it.k : 0);
            if (i1 > i0 && tot + need > budget) break;
            po.push_back(tot);
            if (it.m * cols > 0)
                tasks.insert(tasks.end(), {tot, (int64_t)(uintptr_t)(op.arena.p + it.a_off), it.m, cols, 1, it.a_ld, it.m});
            tot += it.m * cols;
            vo.push_back(wv ? tot : -1);
            if (wv) {
                tasks.insert(tasks.end(), {tot, (int64_t)(uintptr_t)(op.arena.p + it.v_off), it.ncols, it.k, it.v_ld, 1, it.ncols});
                tot += it.ncols * it.k;
            }
        }
        if ((int64_t)stage.n < std::max<int64_t>(tot, 2)) stage.alloc(c, (size_t)std::max<int64_t>(tot, 2), "read-back staging");
        if (!tasks.empty()) {
            DBuf<int64_t> d;
            d.upload(c, tasks, "read-back tasks", s);
            k::pack(d.p, (int)(tasks.size() / 7), stage.p, s);
        }
        double* hp = host.get((size_t)std::max<int64_t>(tot, 1));
        if (tot > 0) HM_CUDA(cudaMemcpyAsync(hp, stage.p, (size_t)tot * sizeof(double), cudaMemcpyDeviceToHost, s));
        HM_CUDA(cudaStreamSynchronize(s));
        // items of a batch write disjoint destinations: scatter them on all host threads
        hla::parallel_for((int64_t)(i1 - i0), [&](int64_t d) {
            const size_t q = i0 + (size_t)d;
            fn(q, hp + po[d], vo[d] >= 0 ? hp + vo[d] : nullptr);
        });
        i0 = i1;
    }
}

// geom block of every phase-2 item of an operator built in F's partition (block = the one whose
// rows contain the item's rows and whose first column is the item's)
std::vector<int> item_blocks(const Geom& g, const HOp& op) {
    std::unordered_map<int64_t, int> key;
    key.reserve(op.items.size() * 2);
    for (size_t b = 0; b < g.blocks.size(); ++b) {
        const Blk& B = g.blocks[b];
        const int l0 = g.leaf_of(B.r0), l1 = g.leaf_of(B.r1 - 1);
        for (int l = l0; l <= l1; ++l) key[((int64_t)l << 32) | B.c0] = (int)b;
    }
    std::vector<int> out(op.items.size(), -1);
    for (size_t q = 0; q < op.items.size(); ++q) {
        const HOp::ItemRec& it = op.items[q];
        auto f = key.find(((int64_t)g.leaf_of(it.r0) << 32) | it.c0);
        if (f == key.end()) throw Error(HM_ERR_CUDA, "operator item outside F's partition");
        out[q] = f->second;
    }
    return out;
}

namespace {

// ---- stage B: hierarchical arithmetic (reading R33)
void stage_b_root(HLU& L, const HMat& F, const Geom& g, const std::vector<double>& lam, int Lc, FactorSet& out) {
    Ctx* c = L.ctx;
    const double eps = L.params.eps_lu;
    double t0 = now_seconds();
    std::vector<std::pair<int, int>> lb(g.blocks.size());
    for (size_t b = 0; b < g.blocks.size(); ++b) lb[b] = {g.blocks[b].rnode, g.blocks[b].cnode};
    auto hf = std::make_shared<hla::HFactor>(g.nodes, lb);
    // C = I - Lambda F block by block: rows scaled by -lambda_i, identity on the
    // diagonal leaves
    auto to_C = [&](int b) {
        const Blk& B = g.blocks[b];
        hla::Mat& M = hf->leaf(b);
        const int64_t m = M.m, nn = M.n;
        if (M.type == hla::T_LR) {
            for (int l = 0; l < M.k; ++l)
                for (int64_t i = 0; i < m; ++i) M.U[i + l * m] *= -lam[B.r0 + i];
        } else {
            for (int64_t j = 0; j < nn; ++j)
                for (int64_t i = 0; i < m; ++i) M.D[i + j * m] *= -lam[B.r0 + i];
            if (B.rnode == B.cnode)
                for (int64_t i = 0; i < m; ++i) M.D[i + i * m] += 1.0;
        }
    };
    if (c->host_only) {
        if (F.host_blocks.size() != g.blocks.size()) throw Error(HM_ERR_NOT_READY, "F holds no host blocks");
        hf->for_each_leaf([&](int b, hla::Mat& M) {
            const HostBlock& H = F.host_blocks[b];
            if (H.kind == KIND_LR) {
                M.type = hla::T_LR;
                M.k = H.k;
                M.U = H.U;
                M.V = H.V;
            } else {
                M.type = hla::T_DENSE;
                M.D = H.D;
            }
            to_C(b);
        });
    } else {
        const std::vector<int> ib = item_blocks(g, F.op);
        hf->for_each_leaf([&](int b, hla::Mat& M) {
            if (F.blk_kind[b] == KIND_LR) {
                M.type = hla::T_LR;
                M.k = F.blk_rank[b];
                M.U.assign((size_t)(M.m * M.k), 0.0);
                M.V.assign((size_t)(M.n * M.k), 0.0);
            } else {
                M.type = hla::T_DENSE;
                M.D.assign((size_t)(M.m * M.n), 0.0);
            }
        });
        read_items(
            c, F.op, [&](size_t q) { return F.op.items[q].r0 == g.blocks[ib[q]].r0; },
            [&](size_t q, const double* pay, const double* V) {
                const HOp::ItemRec& it = F.op.items[q];
                const Blk& B = g.blocks[ib[q]];
                hla::Mat& M = hf->leaf(ib[q]);
                const int64_t ro = it.r0 - B.r0;
                if (M.type == hla::T_LR) {
                    for (int l = 0; l < M.k; ++l)
                        std::copy(pay + l * it.m, pay + (l + 1) * it.m, M.U.begin() + l * M.m + ro);
                    if (V) std::copy(V, V + M.n * M.k, M.V.begin());
                } else {
                    for (int64_t j = 0; j < M.n; ++j)
                        std::copy(pay + j * it.m, pay + (j + 1) * it.m, M.D.begin() + j * M.m + ro);
                }
            });
        hf->for_each_leaf([&](int b, hla::Mat&) { to_C(b); });
    }
    L.setup_seconds[0] = now_seconds() - t0;

    t0 = now_seconds();
    hf->normalize(eps);
    hf->factor(eps);
    if (hf->singular())
        throw Error(HM_ERR_SINGULAR, "near-zero pivot (|pivot| <= 1e-14 max|block|) in the leaf LU of C at internal " +
                                         hf->singular_where());
    hf->solve_form(Lc, eps);
    if (getenv("HM_HLU_VERBOSE")) {
        const hla::Stats& st = hf->stats();
        fprintf(stderr, "[hm] stage-B H-LU n=%lld threads=%d: read %.3f s, lu %.3f s, form %.3f s, %lld truncations "
                        "(mean rank in %.2f, out %.2f)\n",
                (long long)g.n, hf->threads(), L.setup_seconds[0], st.seconds_lu, st.seconds_form,
                (long long)st.truncations, st.truncations ? (double)st.trunc_rank_in / st.truncations : 0.0,
                st.truncations ? (double)st.trunc_rank_out / st.truncations : 0.0);
        hla::prof_dump();
    }
    L.hlu_truncations = hf->stats().truncations;
    L.hlu_threads = hf->threads();
    L.setup_seconds[1] = now_seconds() - t0;
    if (c->host_only) {
        L.host_factor = hf;
        return;
    }

    // ---- upload the solve-form blocks (host chunks of <= 32 Mi doubles)
    t0 = now_seconds();
    out.fwd.assign(std::max(Lc, 0), {});
    out.bwd.assign(std::max(Lc, 0), {});
    int64_t total = 0;
    // A block is stored dense when that is no larger than its factors -- or, in the level form, when it
    // belongs to the W of a node of at most HM_DENSE_W_ROWS rows (default 640): those levels are
    // latency-bound (~16 us per level whatever their bytes, profiles/round2_trace_levelform_c2.txt), and
    // a dense W is one pass per level instead of a phase-1 / phase-2 pair
    static const int64_t dense_w_rows = [] {
        const char* e = getenv("HM_DENSE_W_ROWS");
        return e ? (int64_t)atoll(e) : (int64_t)640;
    }();
    auto dense_out = [&](const hla::LeafView& v) {
        const hla::Mat& M = *v.M;
        if (M.type != hla::T_LR || (int64_t)M.k * (M.m + M.n) >= M.m * M.n) return true;
        if (v.node >= 0 && g.nodes[v.node].level < Lc) {
            const Node& N = g.nodes[v.node];
            return N.end - N.begin <= dense_w_rows;
        }
        return false;
    };
    hf->visit([&](const hla::LeafView& v) {
        const hla::Mat& M = *v.M;
        if (v.side == 0) total += 2 * M.m * M.m;
        else if (dense_out(v)) total += M.m * M.n;
        else total += M.k * (M.m + M.n);
    });
    DBuf<double> dev;
    dev.alloc(c, (size_t)std::max<int64_t>(total, 2), "H-LU factor blocks");
    const cudaStream_t s = c->stream;
    // pinned double buffer of 32 Mi doubles: the copy of one half overlaps the filling of the other
    const int64_t chunk = int64_t(1) << 25;
    double* pin[2] = {nullptr, nullptr};
    cudaEvent_t evs[2] = {nullptr, nullptr};
    struct PinGuard {
        double** p;
        cudaEvent_t* e;
        ~PinGuard() {
            for (int i = 0; i < 2; ++i) {
                if (p[i]) cudaFreeHost(p[i]);
                if (e[i]) cudaEventDestroy(e[i]);
            }
        }
    } pg{pin, evs};
    const int64_t cap = std::min<int64_t>(chunk, std::max<int64_t>(total, 1));
    for (int i = 0; i < 2; ++i) {
        if (cudaMallocHost(&pin[i], (size_t)cap * sizeof(double)) != cudaSuccess) throw Error(HM_ERR_OOM, "pinned upload staging");
        HM_CUDA(cudaEventCreateWithFlags(&evs[i], cudaEventDisableTiming));
    }
    int cur = 0;
    int64_t fill = 0, flushed = 0;
    auto flush = [&]() {
        if (fill == 0) return;
        HM_CUDA(cudaMemcpyAsync(dev.p + flushed, pin[cur], (size_t)fill * sizeof(double), cudaMemcpyHostToDevice, s));
        HM_CUDA(cudaEventRecord(evs[cur], s));
        flushed += fill;
        fill = 0;
        cur ^= 1;
        HM_CUDA(cudaEventSynchronize(evs[cur]));   // the other half is free again
    };
    HM_CUDA(cudaEventRecord(evs[0], s));
    HM_CUDA(cudaEventRecord(evs[1], s));
    auto put = [&](const double* p, int64_t cnt) -> double* {   // device address of the copy
        if (fill + cnt > cap) flush();
        double* at = dev.p + flushed + fill;
        if (cnt > cap) {   // larger than a chunk: straight copy
            HM_CUDA(cudaStreamSynchronize(s));
            HM_CUDA(cudaMemcpy(dev.p + flushed, p, (size_t)cnt * sizeof(double), cudaMemcpyHostToDevice));
            flushed += cnt;
            return at;
        }
        std::memcpy(pin[cur] + fill, p, (size_t)cnt * sizeof(double));
        fill += cnt;
        return at;
    };
    hf->visit([&](const hla::LeafView& v) {
        const hla::Mat& M = *v.M;
        SrcBlock S;
        S.r0 = M.r0; S.m = M.m; S.c0 = M.c0; S.n = M.n;
        if (v.side == 0) {   // packed leaf inverses -> unit-lower L_rr^-1 and upper U_rr^-1, column-major
            const int64_t m = M.m;
            std::vector<double> Li((size_t)(m * m), 0.0), Ui((size_t)(m * m), 0.0);
            for (int64_t j = 0; j < m; ++j)
                for (int64_t i = 0; i < m; ++i) {
                    const double a = M.D[i + j * m];
                    if (i > j) Li[i + j * m] = a;
                    else Ui[i + j * m] = a;
                    if (i == j) Li[i + j * m] = 1.0;
                }
            S.kind = KIND_DENSE;
            S.d_rs = 1;
            S.d_cs = m;
            S.dense = put(Li.data(), m * m);
            out.srcL.push_back(S);
            S.dense = put(Ui.data(), m * m);
            out.srcU.push_back(S);
            return;
        }
        if (dense_out(v)) {
            S.kind = KIND_DENSE;
            S.d_rs = 1;
            S.d_cs = M.m;
            if (M.type == hla::T_LR) {
                std::vector<double> D((size_t)(M.m * M.n), 0.0);
                for (int l = 0; l < M.k; ++l)
                    for (int64_t j = 0; j < M.n; ++j) {
                        const double vj = M.V[j + l * M.n];
                        for (int64_t i = 0; i < M.m; ++i) D[i + j * M.m] += M.U[i + l * M.m] * vj;
                    }
                S.dense = put(D.data(), M.m * M.n);
            } else {
                S.dense = put(M.D.data(), M.m * M.n);
            }
        } else {
            // a low-rank block above the operator panels' rank limit (a phase-1 panel holds <= 128 stacked
            // ranks) is stored as several blocks of <= 64 columns of U and V on the same footprint
            // (U V^T = sum of the parts; multi-body geometries reach ranks in the hundreds at the top
            // levels of the inverse factors)
            const int lvl = g.nodes[v.node].level;
            auto& dst = lvl < Lc ? (v.side == 1 ? out.fwd[lvl] : out.bwd[lvl]) : (v.side == 1 ? out.srcL : out.srcU);
            for (int p0 = 0; p0 < M.k; p0 += 64) {
                const int kp = std::min(64, M.k - p0);
                S.kind = KIND_LR;
                S.k = kp;
                S.u_ld = M.m;
                S.v_ld = M.n;
                S.U = put(M.U.data() + (int64_t)p0 * M.m, M.m * kp);
                S.V = put(M.V.data() + (int64_t)p0 * M.n, M.n * kp);
                dst.push_back(S);
            }
            if (M.k == 0) {
                S.kind = KIND_LR;
                S.k = 0;
                dst.push_back(S);
            }
            return;
        }
        const int lvl = g.nodes[v.node].level;
        if (lvl < Lc) (v.side == 1 ? out.fwd[lvl] : out.bwd[lvl]).push_back(S);
        else (v.side == 1 ? out.srcL : out.srcU).push_back(S);
    });
    flush();
    HM_CUDA(cudaStreamSynchronize(s));
    out.staging.push_back(std::move(dev));
    L.setup_seconds[2] = now_seconds() - t0;
}

// Sharded runs (world > 1): rank 0 factors (all host cores) and broadcasts the solve-form blocks over
// the library's communicator (one header, the block records, the payload); every rank rebuilds the
// same block lists on its own copy, keeps its rows when it packs (build_hop with the shard).  A
// failure on rank 0 travels in the header, so no rank waits on a broadcast that never comes.
void stage_b_inner(HLU& L, const HMat& F, const Geom& g, const std::vector<double>& lam, int Lc, FactorSet& out);

// The factorisation's millions of small host blocks are freed when it ends; hand the arena memory back
// to the system (glibc keeps freed small chunks in its per-thread arenas otherwise, and a process that
// factors twice at C5 size would hold both peaks)
void stage_b(HLU& L, const HMat& F, const Geom& g, const std::vector<double>& lam, int Lc, FactorSet& out) {
    struct Trim { ~Trim() { malloc_trim(0); } } trim;
    stage_b_inner(L, F, g, lam, Lc, out);
}

void stage_b_inner(HLU& L, const HMat& F, const Geom& g, const std::vector<double>& lam, int Lc, FactorSet& out) {
    Ctx* c = L.ctx;
    if (c->host_only || !g.shard.sharded() || !c->ex) {
        stage_b_root(L, F, g, lam, Lc, out);
        return;
    }
    const cudaStream_t s = c->stream;
    const bool root = c->rank == 0;
    int64_t head[4] = {0, 0, 0, 0};   // status, records, payload doubles, message length
    std::string msg;
    hm_status code = HM_OK;
    std::vector<int64_t> rec;
    const double* base = nullptr;
    if (root) {
        try {
            stage_b_root(L, F, g, lam, Lc, out);
        } catch (const Error& e) {
            code = e.code;
            msg = e.what();
        }
        if (code == HM_OK) {
            base = out.staging.empty() ? nullptr : out.staging.back().p;
            auto add = [&](int64_t list, const SrcBlock& S) {
                const int64_t od = S.dense ? S.dense - base : -1, ou = S.U ? S.U - base : -1, ov = S.V ? S.V - base : -1;
                rec.insert(rec.end(), {list, S.r0, S.m, S.c0, S.n, S.kind, S.k, S.d_rs, S.d_cs, od, S.u_ld, ou, S.v_ld, ov});
            };
            for (int lv = 0; lv < Lc; ++lv) {
                for (const SrcBlock& S : out.fwd[lv]) add(2 * lv, S);
                for (const SrcBlock& S : out.bwd[lv]) add(2 * lv + 1, S);
            }
            for (const SrcBlock& S : out.srcL) add(-1, S);
            for (const SrcBlock& S : out.srcU) add(-2, S);
            head[2] = out.staging.empty() ? 0 : (int64_t)out.staging.back().n;
        }
        head[0] = code;
        head[1] = (int64_t)rec.size() / 14;
        head[3] = (int64_t)msg.size();
    }
    DBuf<int64_t> dh;
    dh.upload(c, std::vector<int64_t>(head, head + 4), "factor broadcast header", s);
    c->ex->broadcast(dh.p, sizeof(head), 0, s);
    HM_CUDA(cudaMemcpyAsync(head, dh.p, sizeof(head), cudaMemcpyDeviceToHost, s));
    HM_CUDA(cudaStreamSynchronize(s));
    if (head[0] != HM_OK) {
        std::vector<int64_t> m((size_t)(head[3] + 7) / 8 + 1, 0);
        if (root) std::memcpy(m.data(), msg.data(), msg.size());
        DBuf<int64_t> dm;
        dm.upload(c, m, "factor broadcast message", s);
        c->ex->broadcast(dm.p, m.size() * 8, 0, s);
        HM_CUDA(cudaMemcpyAsync(m.data(), dm.p, m.size() * 8, cudaMemcpyDeviceToHost, s));
        HM_CUDA(cudaStreamSynchronize(s));
        throw Error((hm_status)head[0], std::string((const char*)m.data(), (size_t)head[3]) + " (on rank 0)");
    }
    rec.resize((size_t)head[1] * 14);
    DBuf<int64_t> dr;
    dr.upload(c, rec, "factor broadcast records", s);
    if (!root) {
        out.staging.clear();
        DBuf<double> pay;
        pay.alloc(c, (size_t)std::max<int64_t>(head[2], 2), "H-LU factor blocks");
        out.staging.push_back(std::move(pay));
    }
    if (!rec.empty()) c->ex->broadcast(dr.p, rec.size() * 8, 0, s);
    if (head[2] > 0) c->ex->broadcast(out.staging.back().p, (size_t)head[2] * 8, 0, s);
    if (!root && !rec.empty()) HM_CUDA(cudaMemcpyAsync(rec.data(), dr.p, rec.size() * 8, cudaMemcpyDeviceToHost, s));
    HM_CUDA(cudaStreamSynchronize(s));
    if (!root) {
        const double* b = out.staging.back().p;
        out.fwd.assign(std::max(Lc, 0), {});
        out.bwd.assign(std::max(Lc, 0), {});
        for (size_t q = 0; q < rec.size(); q += 14) {
            const int64_t* r = &rec[q];
            SrcBlock S;
            S.r0 = r[1]; S.m = r[2]; S.c0 = r[3]; S.n = r[4];
            S.kind = (int)r[5]; S.k = (int)r[6];
            S.d_rs = r[7]; S.d_cs = r[8];
            S.dense = r[9] >= 0 ? b + r[9] : nullptr;
            S.u_ld = r[10];
            S.U = r[11] >= 0 ? b + r[11] : nullptr;
            S.v_ld = r[12];
            S.V = r[13] >= 0 ? b + r[13] : nullptr;
            const int64_t list = r[0];
            if (list == -1) out.srcL.push_back(S);
            else if (list == -2) out.srcU.push_back(S);
            else (list % 2 == 0 ? out.fwd : out.bwd)[list / 2].push_back(S);
        }
    }
}

void account(HLU& L, const HOp& op) {
    L.bytes += op.p1_doubles() + op.p2_doubles();
    L.n_blocks += op.n_lr + op.n_dense;
    L.n_lr += op.n_lr;
    L.rank_sum += op.rank_sum;
    L.rank_max = std::max(L.rank_max, op.rank_max);
}

}  // namespace

void factor_hlu(HLU& L, const double* emissivity) {
    const HMat& F = *L.F;
    const Geom& g = *F.geom;
    Ctx* c = L.ctx;
    const cudaStream_t s = c->stream;
    const int64_t n = g.n;
    std::vector<double> eps_int(n), lam(n);
    for (int64_t i = 0; i < n; ++i) {
        const double e = emissivity[g.perm[i]];
        if (!(e > 0.0 && e <= 1.0)) throw Error(HM_ERR_INVALID_ARG, "emissivity of facet " + std::to_string(g.perm[i]) + " not in (0, 1]");
        eps_int[i] = e;
        lam[i] = (1.0 - e) / g.area[i];  // Lambda_ii = (1 - eps_i) / A_i (eq:reflection_matrix)
    }
    if (!(L.params.eps_lu > 0.0 && L.params.eps_lu < 1.0)) throw Error(HM_ERR_INVALID_ARG, "eps_lu must be in (0, 1)");
    const int D = g.depth;
    // cut level (reading R27): W-form updates for levels < Lc, then block-diagonal solves with
    // the inverse factors of the level-Lc diagonal blocks.  < 0 -> 0 (the default: U^-1 (L^-1 b) with
    // the inverse factors in F's partition, fewest dependent passes, measured fastest on C2);
    // >= depth -> pure level form (leaf inverses only)
    const int Lc = L.params.cut_level < 0 ? 0 : std::min(L.params.cut_level, D);
    L.cut_level = Lc;
    FactorSet fs;
    if (L.params.method == 1) {
        if (c->host_only) throw Error(HM_ERR_UNSUPPORTED, "the dense stage-A factorisation needs a device");
        stage_a(L, F, g, lam, Lc, fs);
    } else {
        stage_b(L, F, g, lam, Lc, fs);
    }
    if (c->host_only) return;   // factors kept on the host for hm_export_factors
    L.eps_int.upload(c, eps_int, "eps", s);
    L.eps_ext.upload(c, std::vector<double>(emissivity, emissivity + n), "eps (external)", s);

    // ---- pack the level-form operators
    double t0 = now_seconds();
    L.fwd.resize(std::max(Lc, 0));
    L.bwd.resize(std::max(Lc, 0));
    L.bytes = L.bytes_leaf = L.n_blocks = L.n_lr = L.rank_sum = 0;
    L.rank_max = 0;
    // t slots: disjoint per operator within a sweep's buffer (xtA: forward levels then leafL; xtB:
    // backward levels then leafU)
    int64_t tA = 0, tB = 0;
    for (int lv = 0; lv < Lc; ++lv) {
        build_hop(c, g, fs.fwd[lv], L.fwd[lv], s, nullptr, tA);
        build_hop(c, g, fs.bwd[lv], L.bwd[lv], s, nullptr, tB);
        account(L, L.fwd[lv]);
        account(L, L.bwd[lv]);
        tA += L.fwd[lv].n_t;
        tB += L.bwd[lv].n_t;
    }
    if (Lc == 0) {   // inverse-factor form: L^-1 -> U^-1 -> F chained group by group (Program::link_rows)
        L.leafL.p2_by_row = true;
        L.leafU.p1_by_key = L.leafU.p2_by_row = true;
    }
    build_hop(c, g, fs.srcL, L.leafL, s, nullptr, tA);
    build_hop(c, g, fs.srcU, L.leafU, s, nullptr, tB);
    tA += L.leafL.n_t;
    tB += L.leafU.n_t;
    int64_t tA_loc = 0, tB_loc = 0;
    if (g.shard.sharded()) {   // this rank's rows of the level-form W operators and the cut inverse factors
        L.fwd_loc.resize(std::max(Lc, 0));
        L.bwd_loc.resize(std::max(Lc, 0));
        for (int lv = 0; lv < Lc; ++lv) {
            build_hop(c, g, fs.fwd[lv], L.fwd_loc[lv], s, &g.shard, tA_loc);
            build_hop(c, g, fs.bwd[lv], L.bwd_loc[lv], s, &g.shard, tB_loc);
            tA_loc += L.fwd_loc[lv].n_t;
            tB_loc += L.bwd_loc[lv].n_t;
        }
        build_hop(c, g, fs.srcL, L.leafL_loc, s, &g.shard, tA_loc);
        build_hop(c, g, fs.srcU, L.leafU_loc, s, &g.shard, tB_loc);
        tA_loc += L.leafL_loc.n_t;
        tB_loc += L.leafU_loc.n_t;
    }
    account(L, L.leafL);
    account(L, L.leafU);
    L.bytes_leaf = L.leafL.p1_doubles() + L.leafL.p2_doubles() + L.leafU.p1_doubles() + L.leafU.p2_doubles();
    fs.staging.clear();
    L.xtA.alloc(c, (size_t)(n + tA), "solve xtA");
    L.xtB.alloc(c, (size_t)(n + tB), "solve xtB");
    L.z.alloc(c, (size_t)n, "solve z");
    L.setup_seconds[2] += now_seconds() - t0;

    // ---- hot-path programs for the persistent engine (tree dependencies within each sweep)
    HMat& Fm = const_cast<HMat&>(F);
    auto node_at_level = [&](int64_t row, int level) {   // deepest node on the row's path with level <= level
        int node = 0;
        while (g.nodes[node].level < level && !g.nodes[node].is_leaf()) {
            const Node& N = g.nodes[node];
            node = row < g.nodes[N.child[1]].begin ? N.child[0] : N.child[1];
        }
        return node;
    };
    auto node_map = [&](const StreamPass& sp, int level) {
        std::vector<int32_t> m;
        for (const Panel& pn : sp.panels) m.push_back(node_at_level(pn.key, level));
        return m;
    };
    const auto mL1 = node_map(L.leafL.p1, Lc), mL2 = node_map(L.leafL.p2, Lc);
    const auto mU1 = node_map(L.leafU.p1, Lc), mU2 = node_map(L.leafU.p2, Lc);
    // forward sweep, block-diagonal L^-1 at the cut, backward sweep (U^-1 at the cut left to the caller).
    // With Lc == 0 nothing updates b in place, so the prologue (permute-in, or eta = T^4 and
    // w = eps eta for the flux) is fused into the gathers of the first operator's passes (in_mode);
    // otherwise an element-wise pass materialises b first.
    auto solve_passes = [&](Program& P, int in_mode, double* copy_in = nullptr) {
        P.n_x = n;
        // pinned host input: an element-wise pass copies it into copy_in first (the payload stream
        // starts meanwhile; every reader of the input waits for the pass)
        if (copy_in) P.add_elementwise(UNIT_COPYIN, n, copy_in, copyin_rows(n));
        if (Lc > 0) {
            P.add_elementwise(in_mode == IN_FLUX ? UNIT_PROLOGUE : UNIT_PERMUTE, n, L.xtA.p);
            in_mode = IN_PLAIN;
        }
        P.sweep_dep[0] = (int32_t)P.h_passes.size() - 1;  // the copy-in / prologue / permute pass (-1: none)
        for (int lv = 0; lv < Lc; ++lv) {
            HOp& op = L.fwd[lv];
            const auto m1 = node_map(op.p1, lv), m2 = node_map(op.p2, lv);
            P.add_stream(op.p1, op, L.xtA.p, L.xtA.p, OUT_ASSIGN, DEP_FWD_P1, &m1);
            P.add_stream(op.p2, op, L.xtA.p, L.xtA.p, OUT_SUB, DEP_FWD_P2, &m2);
        }
        P.add_stream(L.leafL.p1, L.leafL, L.xtA.p, L.xtA.p, OUT_ASSIGN, DEP_FWD_P1, &mL1, in_mode);
        P.sweep_dep[1] = (int32_t)P.h_passes.size();  // the cut L^-1 phase-2 pass
        P.add_stream(L.leafL.p2, L.leafL, L.xtA.p, L.xtB.p, OUT_ASSIGN, DEP_FWD_P2, &mL2, in_mode);
        for (int lv = 0; lv < Lc; ++lv) {
            HOp& op = L.bwd[lv];
            const auto m1 = node_map(op.p1, lv), m2 = node_map(op.p2, lv);
            P.add_stream(op.p1, op, L.xtB.p, L.xtB.p, OUT_ASSIGN, DEP_BWD_P1, &m1);
            P.add_stream(op.p2, op, L.xtB.p, L.xtB.p, OUT_SUB, DEP_BWD_P2, &m2);
        }
        const size_t np_before = P.h_passes.size();
        P.add_stream(L.leafU.p1, L.leafU, L.xtB.p, L.xtB.p, OUT_ASSIGN, DEP_BWD_P1, &mU1);
        if (Lc == 0 && P.h_passes.size() > np_before && P.sweep_dep[1] < (int32_t)np_before && !L.leafL.p2.empty())
            P.link_rows(P.sweep_dep[1], (int32_t)np_before);
    };
    solve_passes(L.prog_solve, IN_PERM);
    L.prog_solve.add_stream(L.leafU.p2, L.leafU, L.xtB.p, nullptr, OUT_PERM, DEP_BWD_P2, &mU2);
    L.prog_solve.finalize(c, s, &g);
    L.T_dev.alloc(c, (size_t)n, "pinned host copy-in (solve b / flux T)");
    solve_passes(L.prog_solve_h, IN_PERM, L.T_dev.p);
    L.prog_solve_h.add_stream(L.leafU.p2, L.leafU, L.xtB.p, nullptr, OUT_PERM, DEP_BWD_P2, &mU2);
    L.prog_solve_h.finalize(c, s, &g);
    solve_passes(L.prog_flux, IN_FLUX);
    // U^-1 phase 2 -> F phase 1, linked group by group (cut level 0); returns the pass that writes z
    // (the F input), which F's x-only (near-field) phase-2 tasks wait for -- F may have no phase 1 at all
    // (no low-rank block: small n, or every admissible block capped), so it is not "two passes back"
    auto add_U2_F1 = [&](Program& P) {
        const size_t a = P.h_passes.size();
        P.add_stream(L.leafU.p2, L.leafU, L.xtB.p, Fm.xt.p, OUT_ASSIGN, DEP_BWD_P2, &mU2);
        const int zpass = (int)P.h_passes.size() - 1;
        const size_t b = P.h_passes.size();
        P.add_stream(F.op.p1, F.op, Fm.xt.p, Fm.xt.p, OUT_ASSIGN);
        if (Lc == 0 && b == a + 1 && P.h_passes.size() == b + 1) P.link_rows((int32_t)a, (int32_t)b);
        return zpass;
    };
    const int zf = add_U2_F1(L.prog_flux);
    // x-only (near-field) tasks of phase 2 wait for z, not for phase 1
    L.prog_flux.add_stream(F.op.p2, F.op, Fm.xt.p, nullptr, OUT_FLUX, DEP_BARRIER, nullptr, IN_PLAIN, zf);
    L.prog_flux.finalize(c, s, &g);
    // the same flux program behind a copy-in pass, for a pinned host T (single vector, world == 1)
    solve_passes(L.prog_flux_h, IN_FLUX, L.T_dev.p);
    const int zh = add_U2_F1(L.prog_flux_h);
    L.prog_flux_h.add_stream(F.op.p2, F.op, Fm.xt.p, nullptr, OUT_FLUX, DEP_BARRIER, nullptr, IN_PLAIN, zh);
    L.prog_flux_h.finalize(c, s, &g);

    // ---- flux constant g = F C^-1 eps, with a setup program
    t0 = now_seconds();
    L.g_int.alloc(c, (size_t)n, "g");
    {
        Program pg;
        solve_passes(pg, IN_PERM);
        const int zg = add_U2_F1(pg);
        pg.add_stream(F.op.p2, F.op, Fm.xt.p, L.g_int.p, OUT_ASSIGN, DEP_BARRIER, nullptr, IN_PLAIN, zg);
        pg.finalize(c, s, &g);
        DBuf<double> eps_ext;
        eps_ext.upload(c, std::vector<double>(emissivity, emissivity + n), "eps (external)", s);
        ProgArgs a{};
        a.perm = g.d_perm.p;
        a.user_in = eps_ext.p;
        pg.launch(a, s);
        HM_CUDA(cudaStreamSynchronize(s));
    }
    L.setup_seconds[3] = now_seconds() - t0;

    // ---- multi-RHS programs (world == 1, inverse-factor form): blocks of kMrhsMax columns
    if (!g.shard.sharded() && Lc == 0) {
        L.xtA_m.alloc(c, (size_t)(n + L.leafL.n_t) * kMrhsMax, "solve xtA (multi-RHS)");
        L.xtB_m.alloc(c, (size_t)(n + L.leafU.n_t) * kMrhsMax, "solve xtB (multi-RHS)");
        auto mprog = [&](Program& P, int in_mode, double* out_u, int mode_u) {
            P.mrhs = true;
            P.n_x = n;
            // prologue: b (or w = eps T^4) into the internal n x 64 layout, then every gather is a
            // 512-byte TMA row copy
            P.add_elementwise(in_mode == IN_FLUX ? UNIT_PROLOGUE : UNIT_PERMUTE, n, L.xtA_m.p, elementwise_rows(n));
            // x-only phase-2 tasks wait for the pass that wrote their x input (an operator may have no
            // phase 1: no low-rank block)
            const int x0 = (int)P.h_passes.size() - 1;
            P.add_stream(L.leafL.p1m, L.leafL, L.xtA_m.p, L.xtA_m.p, OUT_ASSIGN);
            P.add_stream(L.leafL.p2m, L.leafL, L.xtA_m.p, L.xtB_m.p, OUT_ASSIGN, DEP_BARRIER, nullptr, IN_PLAIN, x0);
            const int32_t l2 = (int32_t)P.h_passes.size() - 1;
            const size_t nb = P.h_passes.size();
            P.add_stream(L.leafU.p1m, L.leafU, L.xtB_m.p, L.xtB_m.p, OUT_ASSIGN);
            // U^-1 phase 1 of a cluster waits for L^-1 phase 2 on its row group only (as in the
            // single-vector programs): the next operator starts group by group, no full pass drain
            if (!getenv("HM_MRHS_NO_LINKS") && P.h_passes.size() == nb + 1) P.link_rows(l2, (int32_t)nb);
            P.add_stream(L.leafU.p2m, L.leafU, L.xtB_m.p, out_u, mode_u, DEP_BARRIER, nullptr, IN_PLAIN, l2);
        };
        // final results go to an internal n x 64 buffer, then an element-wise epilogue pass emits them
        // (permute-out / flux epilogue) coalesced and fully parallel
        // (HM_MRHS_FUSED_EPI=1: the last stream pass emits through the output mode itself, no epilogue pass)
        const bool fused = mrhs_fused_epilogue();
        mprog(L.prog_solve_m, IN_PERM, Fm.y_m.p, fused ? OUT_PERM : OUT_ASSIGN);
        if (!fused) L.prog_solve_m.add_elementwise(UNIT_EPILOGUE, n, nullptr, elementwise_rows(n), Fm.y_m.p, OUT_PERM);
        L.prog_solve_m.finalize(c, s, &g);
        mprog(L.prog_flux_m, IN_FLUX, Fm.xt_m.p, OUT_ASSIGN);
        {
            Program& P = L.prog_flux_m;
            const int z = (int)P.h_passes.size() - 1;   // U^-1 phase 2 writes z, the F input
            P.add_stream(F.op.p1m, F.op, Fm.xt_m.p, Fm.xt_m.p, OUT_ASSIGN);
            if (!getenv("HM_MRHS_NO_LINKS") && (int)P.h_passes.size() == z + 2) P.link_rows(z, z + 1);
            P.add_stream(F.op.p2m, F.op, Fm.xt_m.p, Fm.y_m.p, fused ? OUT_FLUX : OUT_ASSIGN, DEP_BARRIER, nullptr, IN_PLAIN, z);
        }
        if (!fused) L.prog_flux_m.add_elementwise(UNIT_EPILOGUE, n, nullptr, elementwise_rows(n), Fm.y_m.p, OUT_FLUX);
        L.prog_flux_m.finalize(c, s, &g);
    } else if (!g.shard.sharded()) {
        // level form (cut level > 0) with 64 columns: the same tree-scheduled sweeps as the single-vector
        // solve, on the multi-RHS units (W updates b_t2 -= W b_t1 in place, OUT_SUB), prologue and
        // epilogue as element-wise passes
        L.xtA_m.alloc(c, (size_t)(n + tA) * kMrhsMax, "solve xtA (multi-RHS, level form)");
        L.xtB_m.alloc(c, (size_t)(n + tB) * kMrhsMax, "solve xtB (multi-RHS, level form)");
        auto mprog_lf = [&](Program& P, int in_mode, double* out_u) {
            P.mrhs = true;
            P.n_x = n;
            P.add_elementwise(in_mode == IN_FLUX ? UNIT_PROLOGUE : UNIT_PERMUTE, n, L.xtA_m.p, elementwise_rows(n));
            P.sweep_dep[0] = (int32_t)P.h_passes.size() - 1;
            for (int lv = 0; lv < Lc; ++lv) {
                HOp& op = L.fwd[lv];
                const auto m1 = node_map(op.p1m, lv), m2 = node_map(op.p2m, lv);
                P.add_stream(op.p1m, op, L.xtA_m.p, L.xtA_m.p, OUT_ASSIGN, DEP_FWD_P1, &m1);
                P.add_stream(op.p2m, op, L.xtA_m.p, L.xtA_m.p, OUT_SUB, DEP_FWD_P2, &m2);
            }
            const auto l1 = node_map(L.leafL.p1m, Lc), l2 = node_map(L.leafL.p2m, Lc);
            P.add_stream(L.leafL.p1m, L.leafL, L.xtA_m.p, L.xtA_m.p, OUT_ASSIGN, DEP_FWD_P1, &l1);
            P.sweep_dep[1] = (int32_t)P.h_passes.size();
            P.add_stream(L.leafL.p2m, L.leafL, L.xtA_m.p, L.xtB_m.p, OUT_ASSIGN, DEP_FWD_P2, &l2);
            for (int lv = 0; lv < Lc; ++lv) {
                HOp& op = L.bwd[lv];
                const auto m1 = node_map(op.p1m, lv), m2 = node_map(op.p2m, lv);
                P.add_stream(op.p1m, op, L.xtB_m.p, L.xtB_m.p, OUT_ASSIGN, DEP_BWD_P1, &m1);
                P.add_stream(op.p2m, op, L.xtB_m.p, L.xtB_m.p, OUT_SUB, DEP_BWD_P2, &m2);
            }
            const auto u1 = node_map(L.leafU.p1m, Lc), u2 = node_map(L.leafU.p2m, Lc);
            P.add_stream(L.leafU.p1m, L.leafU, L.xtB_m.p, L.xtB_m.p, OUT_ASSIGN, DEP_BWD_P1, &u1);
            P.add_stream(L.leafU.p2m, L.leafU, L.xtB_m.p, out_u, OUT_ASSIGN, DEP_BWD_P2, &u2);
        };
        mprog_lf(L.prog_solve_m, IN_PERM, Fm.y_m.p);
        L.prog_solve_m.add_elementwise(UNIT_EPILOGUE, n, nullptr, elementwise_rows(n), Fm.y_m.p, OUT_PERM);
        L.prog_solve_m.finalize(c, s, &g);
        mprog_lf(L.prog_flux_m, IN_FLUX, Fm.xt_m.p);
        const int z = (int)L.prog_flux_m.h_passes.size() - 1;   // the pass that writes z (F's input)
        L.prog_flux_m.add_stream(F.op.p1m, F.op, Fm.xt_m.p, Fm.xt_m.p, OUT_ASSIGN);
        L.prog_flux_m.add_stream(F.op.p2m, F.op, Fm.xt_m.p, Fm.y_m.p, OUT_ASSIGN, DEP_BARRIER, nullptr, IN_PLAIN, z);
        L.prog_flux_m.add_elementwise(UNIT_EPILOGUE, n, nullptr, elementwise_rows(n), Fm.y_m.p, OUT_FLUX);
        L.prog_flux_m.finalize(c, s, &g);
    }

    // ---- sharded hot path (world > 1): exchange steps between the engine programs
    if (g.shard.sharded()) {
        const Shard& S = g.shard;
        const int64_t np = S.n_pad();
        std::vector<double> gh(n), ep(np, 0.0), ap(np, 1.0), gp(np, 0.0);
        HM_CUDA(cudaMemcpyAsync(gh.data(), L.g_int.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
        HM_CUDA(cudaStreamSynchronize(s));
        for (int64_t i = 0; i < n; ++i) {   // every segment: the gathers read all ranks' eps
            const int64_t j = S.pad(i);
            ep[j] = eps_int[i];
            ap[j] = g.area[i];
            gp[j] = gh[i];
        }
        L.eps_pad.upload(c, ep, "eps (padded)", s);
        L.area_pad.upload(c, ap, "area (padded)", s);
        L.g_pad.upload(c, gp, "g (padded)", s);
        L.xtA_loc.alloc(c, (size_t)(np + tA_loc), "solve xtA (local)");
        L.xtB_loc.alloc(c, (size_t)(np + tB_loc), "solve xtB (local)");
        // Exchange points: the input is allgathered first; a level-form update at a
        // tree level lv < log2(world) reads rows updated on other ranks, so it is preceded by an
        // allgather of the vector it reads (levels >= log2(world) are rank-local); so are the cut-level
        // inverse factors when the cut is above log2(world), and the first backward level (L^-1 produced
        // only this rank's rows).
        int gl = 0;
        while ((1 << gl) < S.world) ++gl;
        // flux: T is gathered into xtA's x region (cut 0: the first operator's gathers form w = eps T^4
        // on the fly) or, in the level form whose updates overwrite b in place, into T_loc, from which
        // a prologue pass materialises w; the epilogue reads T from there
        if (Lc > 0) L.T_loc.alloc(c, (size_t)np, "T (padded)");
        L.T_pad = Lc > 0 ? L.T_loc.p : L.xtA_loc.p;
        auto sweeps = [&](SegProgram& SP, int in_mode) -> Program* {
            const bool pro = Lc > 0 && in_mode == IN_FLUXI;
            Program* P = &SP.add(pro ? L.T_loc.p : L.xtA_loc.p, true);
            P->n_x = np;
            int im = in_mode;
            if (pro) {
                P->add_elementwise(UNIT_PROLOGUE_INT, np, L.xtA_loc.p, 1024, L.T_loc.p);
                P->sweep_dep[0] = (int32_t)P->h_passes.size() - 1;   // the sweep's root waits for it
                im = IN_PLAIN;
            }
            for (int lv = 0; lv < Lc; ++lv) {
                if (lv > 0 && lv < gl) { P = &SP.add(L.xtA_loc.p, false); P->n_x = np; }
                HOp& op = L.fwd_loc[lv];
                const auto m1 = node_map(op.p1, lv), m2 = node_map(op.p2, lv);
                P->add_stream(op.p1, op, L.xtA_loc.p, L.xtA_loc.p, OUT_ASSIGN, DEP_FWD_P1, &m1);
                P->add_stream(op.p2, op, L.xtA_loc.p, L.xtA_loc.p, OUT_SUB, DEP_FWD_P2, &m2);
            }
            if (Lc > 0 && Lc < gl) { P = &SP.add(L.xtA_loc.p, false); P->n_x = np; }
            const auto l1 = node_map(L.leafL_loc.p1, Lc), l2 = node_map(L.leafL_loc.p2, Lc);
            P->add_stream(L.leafL_loc.p1, L.leafL_loc, L.xtA_loc.p, L.xtA_loc.p, OUT_ASSIGN, DEP_FWD_P1, &l1, im);
            P->add_stream(L.leafL_loc.p2, L.leafL_loc, L.xtA_loc.p, L.xtB_loc.p, OUT_ASSIGN, DEP_FWD_P2, &l2, im);
            for (int lv = 0; lv < Lc; ++lv) {
                if (lv < gl) { P = &SP.add(L.xtB_loc.p, false); P->n_x = np; }
                HOp& op = L.bwd_loc[lv];
                const auto m1 = node_map(op.p1, lv), m2 = node_map(op.p2, lv);
                P->add_stream(op.p1, op, L.xtB_loc.p, L.xtB_loc.p, OUT_ASSIGN, DEP_BWD_P1, &m1);
                P->add_stream(op.p2, op, L.xtB_loc.p, L.xtB_loc.p, OUT_SUB, DEP_BWD_P2, &m2);
            }
            if (Lc < gl) { P = &SP.add(L.xtB_loc.p, false); P->n_x = np; }
            return P;
        };
        {
            Program* P = sweeps(L.sp_solve, IN_PLAIN);
            const auto u1 = node_map(L.leafU_loc.p1, Lc), u2 = node_map(L.leafU_loc.p2, Lc);
            P->add_stream(L.leafU_loc.p1, L.leafU_loc, L.xtB_loc.p, L.xtB_loc.p, OUT_ASSIGN, DEP_BWD_P1, &u1);
            P->add_stream(L.leafU_loc.p2, L.leafU_loc, L.xtB_loc.p, nullptr, OUT_LOCAL, DEP_BWD_P2, &u2);
        }
        L.sp_solve.finalize(c, s, &g);
        {
            Program* P = sweeps(L.sp_flux, IN_FLUXI);
            const auto u1 = node_map(L.leafU_loc.p1, Lc), u2 = node_map(L.leafU_loc.p2, Lc);
            P->add_stream(L.leafU_loc.p1, L.leafU_loc, L.xtB_loc.p, L.xtB_loc.p, OUT_ASSIGN, DEP_BWD_P1, &u1);
            P->add_stream(L.leafU_loc.p2, L.leafU_loc, L.xtB_loc.p, Fm.xt_loc.p, OUT_ASSIGN, DEP_BWD_P2, &u2);
        }
        {
            Program& P = L.sp_flux.add(Fm.xt_loc.p, false);    // allgather z -> F -> q (local slice)
            P.n_x = np;
            P.add_stream(F.op_loc.p1, F.op_loc, Fm.xt_loc.p, Fm.xt_loc.p, OUT_ASSIGN);
            P.add_stream(F.op_loc.p2, F.op_loc, Fm.xt_loc.p, nullptr, OUT_FLUX_LOCAL, DEP_BARRIER, nullptr, IN_PLAIN, -1);
        }
        L.sp_flux.finalize(c, s, &g);
        if (Lc == 0) {   // sharded multi-RHS solve / flux (kMrhsMax columns per launch, DMMA engine)
            const int64_t nl = S.le() - S.lb();
            L.xtA_loc_m.alloc(c, (size_t)(np + tA_loc) * kMrhsMax, "solve xtA (local, multi-RHS)");
            L.xtB_loc_m.alloc(c, (size_t)(np + tB_loc) * kMrhsMax, "solve xtB (local, multi-RHS)");
            L.T_loc_m.alloc(c, (size_t)np * kMrhsMax, "T (padded, multi-RHS)");
            L.y_loc_m.alloc(c, (size_t)np * kMrhsMax, "F y (local, multi-RHS)");
            auto sweeps_m = [&](SegProgram& SP, bool flux, double* out_u, int mode_u) {
                SP.mrhs = true;
                Program* P = &SP.add(flux ? L.T_loc_m.p : L.xtA_loc_m.p, true);
                P->mrhs = true;
                P->n_x = np;
                if (flux) P->add_elementwise(UNIT_PROLOGUE_INT, np, L.xtA_loc_m.p, 128, L.T_loc_m.p);
                P->add_stream(L.leafL_loc.p1m, L.leafL_loc, L.xtA_loc_m.p, L.xtA_loc_m.p, OUT_ASSIGN);
                P->add_stream(L.leafL_loc.p2m, L.leafL_loc, L.xtA_loc_m.p, L.xtB_loc_m.p, OUT_ASSIGN, DEP_BARRIER,
                              nullptr, IN_PLAIN, -1);
                P = &SP.add(L.xtB_loc_m.p, false);   // allgather y -> U^-1
                P->mrhs = true;
                P->n_x = np;
                P->add_stream(L.leafU_loc.p1m, L.leafU_loc, L.xtB_loc_m.p, L.xtB_loc_m.p, OUT_ASSIGN);
                P->add_stream(L.leafU_loc.p2m, L.leafU_loc, L.xtB_loc_m.p, out_u, mode_u, DEP_BARRIER, nullptr,
                              IN_PLAIN, -1);
            };
            sweeps_m(L.sp_solve_m, false, nullptr, OUT_LOCAL);
            L.sp_solve_m.finalize(c, s, &g);
            sweeps_m(L.sp_flux_m, true, Fm.xt_loc_m.p, OUT_ASSIGN);
            {
                Program& P = L.sp_flux_m.add(Fm.xt_loc_m.p, false);   // allgather z -> F -> flux epilogue
                P.mrhs = true;
                P.n_x = np;
                P.add_stream(F.op_loc.p1m, F.op_loc, Fm.xt_loc_m.p, Fm.xt_loc_m.p, OUT_ASSIGN);
                P.add_stream(F.op_loc.p2m, F.op_loc, Fm.xt_loc_m.p, L.y_loc_m.p, OUT_ASSIGN, DEP_BARRIER, nullptr,
                             IN_PLAIN, -1);
                P.add_elementwise(UNIT_EPILOGUE, nl, nullptr, 128, L.y_loc_m.p, OUT_FLUX_LOCAL, S.base());
            }
            L.sp_flux_m.finalize(c, s, &g);
        }
        HM_CUDA(cudaStreamSynchronize(s));
    }
}

}  // namespace hm

using namespace hm;

extern "C" {

hm_status hm_factor_hlu(hm_ctx* ctx, const hm_hmat* F, const double* emissivity, const hm_lu_params* params,
                        hm_hlu** out) {
    if (!ctx || !F || !emissivity || !out) return HM_ERR_INVALID_ARG;
    *out = nullptr;
    Ctx* c = &ctx->c;
    try {
        auto* H = new hm_hlu;
        std::unique_ptr<hm_hlu> guard(H);
        H->h.ctx = c;
        H->h.F = &F->h;
        H->h.params.eps_lu = (params && params->eps_lu > 0.0) ? params->eps_lu : F->h.params.eps_aca;
        H->h.params.cut_level = params ? params->cut_level : -1;
        H->h.params.method = params ? params->method : 0;
        if (H->h.params.method != 0 && H->h.params.method != 1) throw Error(HM_ERR_INVALID_ARG, "method must be 0 or 1");
        factor_hlu(H->h, emissivity);
        *out = guard.release();
        return HM_OK;
    } catch (const Error& e) {
        c->last_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        c->last_error = e.what();
        return HM_ERR_CUDA;
    }
}

void hm_destroy_hlu(hm_hlu* LU) { delete LU; }

}  // extern "C"
