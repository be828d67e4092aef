// Cluster tree (Alg. 1) and block tree (Alg. 2) on the host.
// Compiled with -ffp-contract=off: the box arithmetic is the exact IEEE sequence of
// DESIGN.md readings R6/R7 so the partition is bit-identical to an independent evaluation.
#include <algorithm>
#include <cmath>
#include <numeric>

#include "hm_internal.h"

namespace hm {

namespace {

struct Builder {
    Geom& g;
    const double* xyz;
    const double* aabb;
    std::vector<int32_t>& perm;  // perm[internal] = external

    // Alg. 1 BuildIndexTree(tau) for tau = perm[begin:end)
    int rec(int64_t begin, int64_t end, int level, int parent) {
        const int id = (int)g.nodes.size();
        g.nodes.emplace_back();
        Node nd;
        nd.begin = begin;
        nd.end = end;
        nd.level = level;
        nd.parent = parent;
        double clo[3] = {INFINITY, INFINITY, INFINITY}, chi[3] = {-INFINITY, -INFINITY, -INFINITY};
        double flo[3] = {INFINITY, INFINITY, INFINITY}, fhi[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (int64_t q = begin; q < end; ++q) {
            const int64_t e = perm[q];
            for (int k = 0; k < 3; ++k) {
                clo[k] = std::min(clo[k], xyz[3 * e + k]);
                chi[k] = std::max(chi[k], xyz[3 * e + k]);
                if (g.params.adm_mode == 1) {
                    flo[k] = std::min(flo[k], aabb[6 * e + k]);
                    fhi[k] = std::max(fhi[k], aabb[6 * e + 3 + k]);
                }
            }
        }
        for (int k = 0; k < 3; ++k) {
            nd.lo[k] = g.params.adm_mode == 1 ? flo[k] : clo[k];
            nd.hi[k] = g.params.adm_mode == 1 ? fhi[k] : chi[k];
        }
        const int64_t m = end - begin;
        if (m <= g.params.n_min) {  // PAPER.md:311 "#tau <= n_min" -> leaf index set
            nd.leaf_index = (int)g.leaves.size();
            g.leaves.push_back(id);
            g.depth = std::max(g.depth, level);
            g.nodes[id] = nd;
            return id;
        }
        // hyperplane split: longest centroid-box axis, lowest axis on ties
        double ext[3] = {chi[0] - clo[0], chi[1] - clo[1], chi[2] - clo[2]};
        int axis = 0;
        for (int k = 1; k < 3; ++k)
            if (ext[k] > ext[axis]) axis = k;
        std::sort(perm.begin() + begin, perm.begin() + end, [&](int32_t a, int32_t b) {
            const double xa = xyz[3 * (int64_t)a + axis], xb = xyz[3 * (int64_t)b + axis];
            if (xa != xb) return xa < xb;
            return a < b;
        });
        const int64_t half = (m + 1) / 2;  // left child gets ceil(m/2)
        g.nodes[id] = nd;
        const int c0 = rec(begin, begin + half, level + 1, id);
        const int c1 = rec(begin + half, end, level + 1, id);
        g.nodes[id].child[0] = c0;
        g.nodes[id].child[1] = c1;
        return id;
    }
};

double diam2(const Node& c) {
    const double e0 = c.hi[0] - c.lo[0], e1 = c.hi[1] - c.lo[1], e2 = c.hi[2] - c.lo[2];
    return (e0 * e0 + e1 * e1) + e2 * e2;
}

double dist2(const Node& s, const Node& t) {
    double gsum[3];
    for (int k = 0; k < 3; ++k) gsum[k] = std::max(0.0, std::max(t.lo[k] - s.hi[k], s.lo[k] - t.hi[k]));
    return (gsum[0] * gsum[0] + gsum[1] * gsum[1]) + gsum[2] * gsum[2];
}

// min(diam A_s, diam A_t) <= c dist(A_s, A_t), squared, dist^2 > 0 (R6)
bool admissible(const Node& s, const Node& t, double eta) {
    const double d2 = dist2(s, t);
    return d2 > 0.0 && std::min(diam2(s), diam2(t)) <= (eta * eta) * d2;
}

void block_rec(Geom& g, int s, int t) {  // Alg. 2 BuildBlockTree(s, t)
    const Node& S = g.nodes[s];
    const Node& T = g.nodes[t];
    if (admissible(S, T, g.params.eta)) {
        g.blocks.push_back(Blk{S.level, S.begin, S.end, T.begin, T.end, 1, s, t, KIND_LR, 0});
        return;
    }
    if (S.is_leaf() || T.is_leaf()) {  // DESIGN.md reading R9
        g.blocks.push_back(Blk{S.level, S.begin, S.end, T.begin, T.end, 0, s, t, KIND_DENSE, 0});
        return;
    }
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) block_rec(g, S.child[a], T.child[b]);
}

}  // namespace

int Geom::leaf_of(int64_t row) const {
    auto it = std::upper_bound(leaf_begin.begin(), leaf_begin.end(), row);
    return (int)(it - leaf_begin.begin()) - 1;
}

void build_trees(Geom& g, const double* xyz, const double* nrm, const double* area, const double* aabb) {
    const int64_t n = g.n;
    g.perm.resize(n);
    std::iota(g.perm.begin(), g.perm.end(), 0);
    g.nodes.clear();
    g.leaves.clear();
    g.nodes.reserve(4 * (n / std::max(1, g.params.n_min) + 1));
    Builder b{g, xyz, aabb, g.perm};
    b.rec(0, n, 0, -1);
    g.leaf_begin.resize(g.leaves.size());
    for (size_t i = 0; i < g.leaves.size(); ++i) g.leaf_begin[i] = g.nodes[g.leaves[i]].begin;
    g.blocks.clear();
    block_rec(g, 0, 0);
    std::sort(g.blocks.begin(), g.blocks.end(), [](const Blk& a, const Blk& b) {
        return a.r0 != b.r0 ? a.r0 < b.r0 : a.c0 < b.c0;
    });
    // internal-order facet data
    g.cx.resize(n); g.cy.resize(n); g.cz.resize(n);
    g.nx.resize(n); g.ny.resize(n); g.nz.resize(n); g.area.resize(n);
    for (int64_t i = 0; i < n; ++i) {
        const int64_t e = g.perm[i];
        g.cx[i] = xyz[3 * e]; g.cy[i] = xyz[3 * e + 1]; g.cz[i] = xyz[3 * e + 2];
        g.nx[i] = nrm[3 * e]; g.ny[i] = nrm[3 * e + 1]; g.nz[i] = nrm[3 * e + 2];
        g.area[i] = area[e];
    }
}

}  // namespace hm
