// H-arithmetic on the host: the block H-LU of the reflection matrix C = I - Lambda F
// ("stage B", reading R33) and the conversion of its factors into
// the solve forms of the hot path (level-form W blocks above the cut, inverse factors below,
// DESIGN.md reading R27).  Pure C++ (no CUDA): hlu.cpp feeds it C's blocks read back from F's
// arena and uploads what it produces; the host-only test path feeds it the caller's blocks.
//
// Every matrix lives in F's block partition (the block tree of Alg. 2): a node
// (sigma, tau) is a dense leaf, a low-rank leaf U V^T, or subdivided into the four child pairs.
// The arithmetic is the paper's: the 4-step recursion of PAPER.md:770-775 with recursive forward
// / backward substitutions and block matrix products ("cf. Hackbusch2015"), and a
// rank truncation after every low-rank addition: ranks from the singular-value decay, keeping the
// smallest rank whose Frobenius tail is <= eps * the block's Frobenius norm (PAPER.md:779,
// reading R5).
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <string>
#include <vector>

namespace hm {
struct Node;
namespace hla {

enum Type : int { T_DENSE = 0, T_LR = 1, T_SUB = 2 };

struct Mat {
    int64_t m = 0, n = 0;   // rows, columns
    int64_t r0 = 0, c0 = 0; // first row / column (internal order)
    int rn = -1, cn = -1;   // row / column cluster (tree node ids)
    int type = T_DENSE;
    std::vector<double> D;  // dense: column-major m x n
    int k = 0;              // low rank: M = U V^T, U column-major m x k, V column-major n x k
    std::vector<double> U, V;
    std::unique_ptr<Mat> c[4];   // T_SUB: c[2 i + j] = (row child i, column child j)
    bool acc = false;       // an admissible leaf-x-leaf block held dense while the factorisation runs
                            // (its updates are GEMMs, not truncations); truncated once at the end
    Mat* ch(int i, int j) const { return c[2 * i + j].get(); }
};

struct Stats {
    int64_t truncations = 0;     // low-rank truncations (QR + SVD)
    int64_t trunc_rank_in = 0;   // sum of ranks entering a truncation
    int64_t trunc_rank_out = 0;
    double seconds_lu = 0, seconds_form = 0;
};

// One leaf of the final factor set (visit()).
struct LeafView {
    const Mat* M;
    int side;    // 0: diagonal leaf (packed L^-1 strictly below, U^-1 on and above the diagonal);
                 // 1: strictly lower (W^L or L^-1 block); 2: strictly upper (W^U or U^-1 block)
    int node;    // tree node t whose off-diagonal part (t2 x t1 / t1 x t2) holds the block
                 // (-1 for diagonal leaves)
};

class HFactor {
public:
    // Structure of F's block tree over the cluster tree `nodes` (preorder, nodes[0] = root);
    // blocks given as (row node, column node) pairs, one per leaf of the partition.
    HFactor(const std::vector<Node>& nodes, const std::vector<std::pair<int, int>>& leaf_blocks);
    ~HFactor();
    // Leaf b's payload (b indexes leaf_blocks).  Dense: column-major m x n.  Low rank: U m x k,
    // V n x k column-major.  Admissible blocks stored dense in F ("adm-dense") may be given dense:
    // they are converted to the low-rank form by truncation (exact up to eps).
    Mat& leaf(int b) { return *by_block_[b]; }
    // f(b, leaf(b)) for every partition block, OpenMP-parallel over blocks
    void for_each_leaf(const std::function<void(int, Mat&)>& f);
    // Converts dense payloads of admissible-structure leaves (both clusters inner nodes) to low rank.
    void normalize(double eps);
    // In place H-LU without pivoting (reading R12): unit-lower L strictly below the
    // diagonal, U on and above it.  Throws (via the callback-free error flag) on a near-zero pivot.
    void factor(double eps);
    // In place: for tree nodes t with level < cut: A[t2,t1] <- W^L_t = L21 L11^-1 and
    // A[t1,t2] <- W^U_t = U12 U22^-1; diagonal blocks of the cut level (and leaves above it) are
    // replaced by their inverse factors L_tt^-1 (strictly lower part) and U_tt^-1 (upper part).
    void solve_form(int cut, double eps);
    void visit(const std::function<void(const LeafView&)>& f) const;
    const Stats& stats() const { return stats_; }
    bool singular() const { return singular_; }
    std::string singular_where() const { return singular_where_; }
    const Mat& root() const { return *root_; }
    int threads() const;

private:
    const std::vector<Node>& nodes_;
    std::unique_ptr<Mat> root_;
    std::vector<Mat*> by_block_;
    Stats stats_;
    bool singular_ = false;
    std::string singular_where_;
    friend struct Impl;
};

// Dense helpers exposed for tests of the host arithmetic (column-major).
// Truncate U V^T (U m x K, V n x K) in place to the smallest rank whose Frobenius tail is
// <= eps ||U V^T||_F; returns the new rank (U, V resized to m x k', n x k').
void prof_dump();
// f(i) for i in [0, n), OpenMP-parallel (host helper for callers compiled without OpenMP)
void parallel_for(int64_t n, const std::function<void(int64_t)>& f);
int truncate(int64_t m, int64_t n, int K, std::vector<double>& U, std::vector<double>& V, double eps);

}  // namespace hla
}  // namespace hm
