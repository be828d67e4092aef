// Internal declarations of the hm library (host orchestration + kernel launchers).
// Nothing here is part of the C ABI (include/hm.h is).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/hm.h"

namespace hm {

// ------------------------------------------------------------------ errors
struct Error : std::runtime_error {
    hm_status code;
    Error(hm_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void cuda_check(cudaError_t e, const char* what, const char* file, int line);
#define HM_CUDA(x) ::hm::cuda_check((x), #x, __FILE__, __LINE__)
void debug_sync(cudaStream_t s, const char* what);

// ------------------------------------------------------------------ device memory
struct Ctx;
void* dmalloc(Ctx* ctx, size_t bytes, const char* what);
void dfree(Ctx* ctx, void* p);

template <class T>
struct DBuf {  // owning device buffer
    Ctx* ctx = nullptr;
    T* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept { *this = std::move(o); }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) { reset(); ctx = o.ctx; p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DBuf() { reset(); }
    void alloc(Ctx* c, size_t count, const char* what) {
        reset();
        ctx = c;
        n = count;
        p = count ? static_cast<T*>(dmalloc(c, count * sizeof(T), what)) : nullptr;
    }
    void upload(Ctx* c, const std::vector<T>& h, const char* what, cudaStream_t s) {
        alloc(c, h.size(), what);
        if (!h.empty()) HM_CUDA(cudaMemcpyAsync(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    void reset();
};

// The exchange step of the sharded hot path: in-place allgather of a padded vector (rank q's
// segment at buf[q*count, (q+1)*count)), stream-ordered.  shard.cpp.
struct Exchanger {
    virtual ~Exchanger() = default;
    virtual void allgather(double* buf, int64_t count, cudaStream_t s) = 0;
    // buf (bytes, device) of `root` to every rank, stream-ordered (setup: the H-LU factors)
    virtual void broadcast(void* buf, size_t bytes, int root, cudaStream_t s) = 0;
    virtual const char* kind() const = 0;
};

struct Ctx {
    int device = 0, rank = 0, world = 1;
    bool host_only = false;            // device < 0: trees / shard plan only (no CUDA)
    Exchanger* ex = nullptr;           // world > 1 (owned)
    bool skip_exchange = false;        // measurement only (hm_profile_flux): sharded programs skip their allgathers
    uint32_t flags = 0;
    cudaStream_t stream = nullptr;  // setup stream
    std::string last_error;
    void* (*alloc_fn)(size_t, void*, void*) = nullptr;
    void (*free_fn)(void*, void*, void*) = nullptr;
    void* alloc_user = nullptr;
    bool debug = false;
};

template <class T>
void DBuf<T>::reset() {
    if (p) dfree(ctx, p);
    p = nullptr;
    n = 0;
}

// ------------------------------------------------------------------ geometry / trees
struct Node {
    int64_t begin = 0, end = 0;
    int level = 0;
    int child[2] = {-1, -1};
    int parent = -1;
    int leaf_index = -1;  // index into Geom::leaves if leaf
    double lo[3], hi[3];  // admissibility box
    int64_t size() const { return end - begin; }
    bool is_leaf() const { return child[0] < 0; }
};

enum Kind : int { KIND_DENSE = 0, KIND_LR = 1, KIND_ADM_DENSE = 2 };

struct Blk {
    int level;
    int64_t r0, r1, c0, c1;
    int adm;
    int rnode, cnode;
    int kind = KIND_DENSE;
    int rank = 0;
};

// Row-cluster shard of this rank: padded layout of G segments of maxc entries.
struct Shard {
    int rank = 0, world = 1;
    int64_t maxc = 0;
    std::vector<int64_t> rb, re;   // per-rank internal-order row ranges
    bool sharded() const { return world > 1; }
    int64_t lb() const { return rb[rank]; }
    int64_t le() const { return re[rank]; }
    int64_t n_pad() const { return (int64_t)world * maxc; }
    int64_t base() const { return (int64_t)rank * maxc; }
    int rank_of(int64_t i) const;
    int64_t pad(int64_t i) const {
        if (world == 1) return i;
        const int q = rank_of(i);
        return (int64_t)q * maxc + (i - rb[q]);
    }
    bool owns_row(int64_t i) const { return world == 1 || (i >= lb() && i < le()); }
};

struct Geom {
    Ctx* ctx;
    Shard shard;
    int64_t n;
    hm_tree_params params;
    std::vector<int32_t> perm;  // perm[internal] = external
    std::vector<Node> nodes;    // preorder; nodes[0] = root
    std::vector<int> leaves;    // node ids in internal order
    std::vector<int64_t> leaf_begin;  // sorted begins of leaves
    int depth = 0;
    std::vector<Blk> blocks;    // sorted by (r0, c0)
    // internal-order facet data (host copies)
    std::vector<double> cx, cy, cz, nx, ny, nz, area;
    // device copies (SoA, internal order)
    DBuf<double> d_geo;         // 7*n: cx cy cz nx ny nz A
    DBuf<int32_t> d_perm;
    double setup_seconds = 0;
    int leaf_of(int64_t row) const;  // leaf index containing internal row
};

void build_trees(Geom& g, const double* xyz, const double* nrm, const double* area,
                 const double* aabb);
void local_range(const Geom& g, int rank, int world, int64_t* begin, int64_t* end);
void make_shard(Geom& g, int rank, int world);
std::unique_ptr<Exchanger> make_exchanger(int device, int rank, int world, const void* comm_id, uint32_t flags);

// ------------------------------------------------------------------ the two-phase stream operator
// Both phases are "column-stream panels": a column-major matrix (column stride ld, even) whose
// column c multiplies the gathered input XT[colsrc[cs_off + c]].
//   phase 1: one panel per column cluster tau: the V^T of every low-rank block (sigma, tau)
//            stacked (K_tau = sum k rows); output rows are t entries (XT[n + ...]).
//   phase 2: one panel per leaf row r: the leaf-row slices of the dense blocks and U factors
//            covering r; output rows are the leaf's facets.
// A panel is cut into work units (row tile <= 128 rows x column chunk of ~48 KB).  Units of the
// same row tile ("group") write partial sums; the last-arriving unit adds them in segment order
// (deterministic, no floating-point atomics).
// A chunk: <= one engine stage (kStageDoubles, 56.6 KB; 32 KB in the multi-RHS engine) of contiguous
// payload (ncols * ld doubles) + its column-source list; the unit
// of TMA transfer.  A task = consecutive chunks of one panel piece, processed by one CTA that
// accumulates in registers and emits once.  Pieces of the same panel (only panels > 512 KB are
// split) combine deterministically: the last-finishing piece adds the partials in piece order.
constexpr int kMaxRuns = 16;
struct alignas(16) Unit {
    int64_t a_off;     // arena offset of the chunk payload
    int64_t out0;      // output index of row 0 of the panel
    int64_t part_off;  // partial-sum scratch offset of this piece (nseg > 1)
    int64_t cs_off;    // colsrc offset of the chunk's first column (multiple of 4: 16-byte aligned)
    int32_t ld;        // column stride (even, <= 128)
    int32_t nrows;     // rows (<= 128)
    int32_t ncols;     // columns of this chunk (<= 512)
    int32_t grp;       // combine group of the panel (-1: single piece writes directly)
    int32_t nseg;      // pieces in the group
    int32_t seg;       // piece index
    int32_t pass;      // program pass index (engine)
    int32_t type;      // UNIT_STREAM / UNIT_PROLOGUE / UNIT_PERMUTE
    int32_t chunk;     // chunk index within the piece
    int32_t nchunks;   // chunks in the piece
    int64_t first_chunk;  // index (in the unit list) of the piece's first chunk
    // column sources as runs of consecutive input indices (nruns = 0: too many runs, use colsrc):
    // the gather can start as soon as the descriptor is known, without a round trip for colsrc
    int32_t nruns;
    int32_t run_src[kMaxRuns];
    uint16_t run_len[kMaxRuns];
    // the task this chunk belongs to and its dependency record (copied from the Task at program
    // finalisation, so the engine's chunk header is self-contained)
    int64_t task;
    int32_t wait_id[2], wait_cnt[2], inc_id[2];
};
static_assert(sizeof(Unit) % 16 == 0, "Unit is TMA-copied");
// UNIT_EPILOGUE (multi-RHS): rows of an internal n x kMrhsMax result emitted through the pass's output
// mode (permute-out / flux epilogue) by element-wise units, coalesced and fully parallel
// UNIT_PROLOGUE_INT (sharded level form): out[row] = eps[row] * in[row]^4 on padded internal rows
// UNIT_COPYIN (pinned host input): out[row * ld + col] = host_in[row * ld + col], rows in external order
enum UnitType : int32_t { UNIT_STREAM = 0, UNIT_PROLOGUE = 1, UNIT_PERMUTE = 2, UNIT_EPILOGUE = 3, UNIT_PROLOGUE_INT = 4,
                          UNIT_COPYIN = 5 };
constexpr int kUnitPayloadDoubles = 4096;   // 32 KB TMA stage (multi-RHS engine)
#ifndef HM_STAGE_DOUBLES
#define HM_STAGE_DOUBLES 7240
#endif
constexpr int kStageDoubles = HM_STAGE_DOUBLES;   // single-vector engine payload stage (doubles): 56.6 KB
constexpr int kMrhsMax = 64;                // multi-RHS block width (columns of X per program launch)
// multi-RHS chunk geometry (experiment overrides through HM_BUILD_DEFINES): <= HM_MRHS_MAXCOLS panel
// columns (X tile HM_MRHS_MAXCOLS x 64) and <= HM_MRHS_PAYLOAD doubles of payload per chunk
#ifndef HM_MRHS_MAXCOLS
#define HM_MRHS_MAXCOLS 64
#endif
#ifndef HM_MRHS_PAYLOAD
#define HM_MRHS_PAYLOAD 4096
#endif
constexpr int kMrhsMaxCols = HM_MRHS_MAXCOLS;
constexpr int kMrhsPayloadDoubles = HM_MRHS_PAYLOAD;
constexpr int kUnitMaxCols = 256;
constexpr int64_t kPieceDoubles = 65536;    // panels above 512 KB are split into pieces

// A task waits until counter[wait_id[i]] >= epoch * wait_cnt[i] (i < 2, id -1 = none) before its
// first input gather, and on retirement increments counter[pass] and counter[inc_id[i]].
struct Task {
    int64_t first_unit;
    int32_t n_units;
    int32_t pass;
    int32_t wait_id[2];
    int32_t wait_cnt[2];
    int32_t inc_id[2];
};
// dependency kinds of a pass (engine programs)
enum DepKind : int { DEP_BARRIER = 0, DEP_FWD_P1, DEP_FWD_P2, DEP_FWD_LEAF, DEP_BWD_P1, DEP_BWD_P2, DEP_BWD_LEAF };

struct Panel {         // host description of a panel
    int64_t a_off;     // arena offset of row 0, column 0
    int64_t out0;      // output index of row 0
    int32_t ld, nrows, ncols, cs_off;
    int64_t key;       // phase 1: first column of the cluster tau; phase 2: first row of the leaf
    int32_t ndense;    // leading columns that read only the x region (phase 2: dense blocks first)
};

struct StreamPass {    // one pass worth of chunks (host copy; programs upload them)
    std::vector<Unit> h_units;
    std::vector<int32_t> unit_panel;   // panel index of each chunk
    std::vector<uint8_t> unit_xonly;   // 1: the chunk's piece reads only the x region (no t)
    int64_t n_units = 0;
    DBuf<double> part;
    DBuf<int32_t> counters;
    std::vector<Panel> panels;
    int64_t doubles = 0;   // algorithmic payload read by this pass
    bool empty() const { return n_units == 0; }
};

// A block as a source for the operator builder.
struct SrcBlock {
    int64_t r0, m, c0, n;
    int kind;        // KIND_LR -> U/V; otherwise dense
    int k = 0;
    bool fill_entries = false;       // dense: evaluate view-factor entries (F near field)
    const double* dense = nullptr;   // dense element (i,j) at dense[i*d_rs + j*d_cs]
    int64_t d_rs = 0, d_cs = 0;
    const double* U = nullptr;       // U element (i,l) at U[l*u_ld + i]
    int64_t u_ld = 0;
    const double* V = nullptr;       // V element (j,l) at V[l*v_ld + j]
    int64_t v_ld = 0;
};

struct HOp {
    int64_t n_rows_total = 0;     // n
    int64_t n_x = 0;              // size of the x region of XT
    DBuf<double> arena;
    StreamPass p1, p2;
    StreamPass p1m, p2m;           // the same panels chunked for the multi-RHS kernel (world == 1)
    DBuf<int32_t> colsrc;          // per-unit, 16-byte aligned column-source segments
    DBuf<int32_t> colsrc_ext;      // same, x-region entries as -(external index + 1) (fused prologue)
    int64_t n_t = 0;              // total rank (size of t)
    int64_t xt_len = 0;           // column sources index [0, xt_len) of the XT buffer (x region + t_off + n_t)
    struct ItemRec {              // one phase-2 item (a leaf-row slice of one block)
        int64_t a_off;            // U slice / dense slice, column-major with stride a_ld
        int64_t a_ld;
        int64_t v_off;            // LR: V_b[j,l] at v_off + j*v_ld + l ; dense: -1
        int64_t v_ld;
        int64_t r0, m, c0, ncols; // rows of the slice, columns of the block
        int64_t k;
    };
    std::vector<ItemRec> items;
    int64_t n_lr = 0, n_dense = 0;
    int64_t rank_sum = 0;
    int rank_max = 0;
    // task order (set before build_hop): phase-1 pieces by cluster start (they wait on row groups of
    // the previous operator, Program::link_rows), phase-2 t-reading pieces by row (they feed the next
    // operator's phase 1 group by group); default: largest first
    bool p1_by_key = false, p2_by_row = false;
    int64_t p1_doubles() const { return p1.doubles; }
    int64_t p2_doubles() const { return p2.doubles; }
    bool empty() const { return p1.empty() && p2.empty(); }
};

// Build the operator; XT layout is [x (n_x) | t (n_t)].  With a shard (world > 1) only the block
// rows of this rank are stored, x indices and phase-2 outputs use the padded layout (n_x = n_pad).
// t_off: first t slot of this operator in its XT buffer (operators of different levels that share a
// buffer get disjoint t regions, so a level's phase 1 never overwrites t still to be read by another
// subtree's phase 2 of an earlier level)
void build_hop(Ctx* ctx, const Geom& g, std::vector<SrcBlock>& blocks, HOp& op, cudaStream_t s,
               const Shard* sh = nullptr, int64_t t_off = 0, const double* quad = nullptr);
// adaptive Gauss quadrature of the view-factor entries (reading R35): per facet
// (internal order) kQStride doubles: 3 + 6 + 24 quadrature points (x, y, z) of the three tiers, then
// the squared longest edge
constexpr int kQStride = 100, kQOff1 = 0, kQOff2 = 9, kQOff3 = 27, kQH2 = 99;
std::vector<double> quad_table(const Geom& g, const double* vertices_ext);

// ------------------------------------------------------------------ persistent stream engine
struct Pass {
    int32_t type;        // UnitType of its units
    int32_t dep;         // pass whose completion this pass waits for (-1: none)
    int32_t mode;        // OutMode
    int32_t in_mode;     // InMode: how x-region inputs (index < n_x) are gathered
    int64_t first_unit, n_units;
    int64_t n_tasks;
    const double* arena;
    const int32_t* colsrc;
    const double* in;    // input vector (nullptr: the call's user_in)
    double* out;         // output vector (OUT_ASSIGN / OUT_SUB; element-wise units)
    double* part;        // split-K partials
    int32_t* counters;   // split-K group counters
};

struct ProgArgs {
    const Pass* passes;
    int32_t n_passes;
    int32_t pad0;
    const Unit* units;
    const Task* tasks;
    int64_t n_tasks;
    unsigned long long* queue;  // monotone task counter: advances by n_tasks + grid per launch
    int64_t n_units;
    unsigned long long* done;   // dependency counters (passes, then per-node), monotone over launches
    unsigned long long* trace;  // optional: per pass [first gather, last retire] (%globaltimer ns)
    unsigned long long* stats;  // optional: per-role SM cycle counters (diagnostics, HM_ENGINE_STATS=1)
    // [0] launch number of this program (1-based), [1] CTA starts so far.  Read by every CTA at its
    // start; the last CTA to start advances [0] -- so the epoch lives on the device and a launch
    // captured in a CUDA graph is replayable (no host-side launch counter baked into the arguments)
    unsigned long long* epoch_dev;
    const int32_t* perm;
    const double* user_in;      // x / b / T (external order, ld x ncol)
    const double* host_in;      // UNIT_COPYIN: device alias of the caller's pinned host input
    int64_t n_x;                // size of the x region of XT (IN_PERM / IN_FLUX apply below it)
    double* user_out;           // y / z / q (external order)
    int ld, col;
    const double* eps_int;
    const double* eps_ext;      // emissivity in external order (IN_FLUX gathers)
    const double* area_int;
    const double* g_int;
    const double* amb;          // open-cavity ambient term (eqn:flux_to_ambient): A_i (1 - c_i) per row, or nullptr
    double t_inf4;              // T_inf^4 (0 in the Jacobian mode: the derivative drops the constant)
    double sigma;
    int32_t eta_in;             // 1: the flux input is the facet power eta itself (not T: no T^4)
    int32_t rbar_out;           // 1: emit A o q = (Rbar eta) (eq:Rbardef) instead of q
    int64_t local0;             // sharded: padded index of this rank's first row
    int32_t nrhs;               // multi-RHS: columns of this launch (<= kMrhsMax; user arrays have ld >= nrhs)
    const double* T_pad;        // sharded flux: gathered temperatures (padded internal order)
    // HM_DEVICE_CHECKS builds only: per pass {arena doubles, column-source entries, input index bound}
    // (the engines check every chunk descriptor and gathered index against them, then trap)
    const int64_t* chk;
};

// input modes of a stream pass: the prologue / permute-in fused into the gather
// IN_FLUXI (sharded flux): x-region input j is T_j (padded internal order), gathered as eps_j T_j^4
enum InMode : int { IN_PLAIN = 0, IN_PERM = 1, IN_FLUX = 2, IN_FLUXI = 3 };

// A program = passes in topological order; executes in one cooperative launch.
struct Program {
    std::vector<Pass> h_passes;
    std::vector<Unit> h_units;
    std::vector<Task> h_tasks;
    DBuf<Pass> passes;
    DBuf<Unit> units;
    DBuf<Task> tasks;
    DBuf<unsigned long long> queue;   // monotone task counter (epoch * n_tasks at the end of a launch)
    DBuf<unsigned long long> done;
    DBuf<unsigned long long> epoch_dev;   // see ProgArgs::epoch_dev
    int grid = 0;
    bool ready = false;
    bool mrhs = false;   // multi-RHS program (engine_mrhs_kernel, kMrhsMax columns per launch)
    int64_t n_x = 0;     // x-region size of the programs' XT buffers (fused-prologue gathers)
    std::vector<int32_t> task_kind, task_node;   // dependency kind / tree node of each task
    std::vector<int64_t> task_key;               // panel key (phase 1: cluster start, phase 2: row start)
    std::vector<int32_t> task_span;              // phase 1: cluster size
    std::vector<std::pair<int32_t, int32_t>> row_links;   // (phase-2 pass, next operator's phase-1 pass)
    std::vector<uint8_t> task_xonly;             // task reads only the x region of its input
    std::vector<int32_t> pass_xdep;              // per pass: see add_stream
    int32_t sweep_dep[2] = {-1, -1};             // pass the root of the fwd / bwd sweep waits for
    int64_t n_counters = 0;
    DBuf<unsigned long long> trace;
    DBuf<unsigned long long> stats;
    std::vector<int64_t> h_chk;   // per pass: arena doubles, column-source entries, input index bound
    DBuf<int64_t> chk;            // (uploaded in HM_DEVICE_CHECKS builds)
    // builder: panel_node (optional) maps each panel of `sp` to its tree node (tree kinds)
    // xdep (DEP_BARRIER passes): the pass whose completion x-only tasks wait for instead of the
    // previous pass (-2: no distinction, -1: no wait)
    void add_stream(const StreamPass& sp, const HOp& op, const double* in, double* out, int mode,
                    int kind = DEP_BARRIER, const std::vector<int32_t>* panel_node = nullptr, int in_mode = IN_PLAIN,
                    int xdep = -2);
    void add_elementwise(int type, int64_t n, double* out, int rows_per_unit = 1024, const double* in = nullptr,
                         int mode = 0 /* OUT_ASSIGN */, int64_t row0 = 0 /* rows [row0, row0 + n) */);
    // the phase-1 tasks of pass p1 whose cluster lies inside one row group (a tree node of level
    // depth - 4) wait for the phase-2 tasks of pass p2 on that group's rows instead of for all of p2
    void link_rows(int32_t p2, int32_t p1) { row_links.emplace_back(p2, p1); }
    void finalize(Ctx* ctx, cudaStream_t s, const Geom* g = nullptr);
    void launch(ProgArgs a, cudaStream_t s);
};

// Sharded hot path (world > 1): engine programs separated by exchange steps.  Before segment i,
// if pre[i] != nullptr: (pre_user[i]: copy the caller's local slice, column `col`, into this rank's
// segment of pre[i]) then allgather pre[i] in place (count = maxc per rank).
struct SegProgram {
    std::vector<std::unique_ptr<Program>> segs;
    std::vector<double*> pre;
    std::vector<uint8_t> pre_user;
    bool mrhs = false;   // vectors row-major n_pad x kMrhsMax: the user slice is a.nrhs columns from
                         // column a.col, the allgather moves maxc x kMrhsMax doubles per rank
    Program& add(double* exch_buf, bool user_slice) {
        segs.emplace_back(new Program());
        pre.push_back(exch_buf);
        pre_user.push_back(user_slice ? 1 : 0);
        return *segs.back();
    }
    bool empty() const { return segs.empty(); }
    void finalize(Ctx* ctx, cudaStream_t s, const Geom* g) {
        for (auto& p : segs) p->finalize(ctx, s, g);
    }
    void launch(Ctx* ctx, const Geom& g, ProgArgs a, cudaStream_t s);
};

// rows per element-wise unit of the multi-RHS programs (prologue / permute / epilogue): one unit per
// SM (measured C2 64-RHS flux: 32-row units took 15 + 30 us for the prologue and epilogue, every
// unit paying the pipeline's per-chunk latency), at least 32 rows
inline int elementwise_rows(int64_t n) {
    const int64_t r = (n + 147) / 148;
    return (int)std::max<int64_t>(32, (r + 7) & ~int64_t(7));
}

// multi-RHS programs: the last stream pass emits the caller's result itself (OUT_PERM / OUT_FLUX from the
// task's accumulators) instead of writing the internal n x 64 buffer for an element-wise epilogue pass
// (HM_MRHS_FUSED_EPI=1; read when a program is built)
inline bool mrhs_fused_epilogue() {
    const char* e = getenv("HM_MRHS_FUSED_EPI");
    return e && e[0] == '1';
}

// rows per copy-in unit (pinned host input read through its device alias over PCIe): about one unit per
// SM, so the pass is one or two latency-bound round trips per CTA instead of a few long units (1,024-row
// units left 20 units on C2, each a chain of four round trips); multiple of 4 (unrolled loads)
inline int copyin_rows(int64_t n) {
    const int64_t r = (n + 147) / 148;
    return (int)std::max<int64_t>(64, (r + 3) & ~int64_t(3));
}

size_t engine_smem_bytes();
int engine_mrhs_grid();
int engine_mrhs_max_passes();
void engine_mrhs_launch(const ProgArgs& A, int grid, cudaStream_t s);
int engine_max_passes();
int engine_grid();
void engine_launch(const ProgArgs& A, int grid, cudaStream_t s);

// output modes of phase 2
// OUT_LOCAL / OUT_FLUX_LOCAL (sharded): the caller's vectors are this rank's slice in internal order
enum OutMode : int { OUT_ASSIGN = 0, OUT_SUB = 1, OUT_PERM = 2, OUT_FLUX = 3, OUT_LOCAL = 4, OUT_FLUX_LOCAL = 5 };
struct FluxEpi {  // OUT_FLUX: q_ext[perm[i]] = sigma * eps_i / A_i * (acc - eta_i g_i)
    const double* T_ext;
    const int32_t* perm;
    const double* eps_int;
    const double* eps_ext;      // emissivity in external order (IN_FLUX gathers)
    const double* area_int;
    const double* g_int;
    double sigma;
    int ld;    // leading dimension (nrhs) of the external arrays; also used by OUT_PERM
    int col;   // column of the external arrays
};

namespace hla { class HFactor; }

// A block payload held on the host (host-only contexts: hm_hmat_from_host).
struct HostBlock {
    int kind = KIND_DENSE;   // KIND_DENSE: D column-major m x n; KIND_LR: U (m x k), V (n x k) column-major
    int k = 0;
    std::vector<double> D, U, V;
};

struct HMat {
    Ctx* ctx;
    const Geom* geom;
    hm_aca_params params;
    std::vector<HostBlock> host_blocks;   // host-only contexts: the caller's F, per geom block
    HOp op;
    std::vector<double> s_ext, c_ext;  // row sums / clamped (external order)
    std::vector<int> blk_kind, blk_rank;  // per geom block
    double setup_seconds[4] = {0, 0, 0, 0};
    // apply workspace
    DBuf<double> xt;   // [x | t]
    DBuf<double> y;    // internal-order output
    DBuf<double> host_stage_in, host_stage_out;
    Program prog_apply;   // permute-in -> F phase 1 -> F phase 2 (+ permute-out)
    Program prog_apply_h; // the same behind a copy-in pass for a pinned host x (single vector)
    DBuf<double> x_dev;   // its device copy of x
    // sharded hot path (world > 1): this rank's block rows, padded vectors
    HOp op_loc;
    DBuf<double> xt_loc;  // [x_pad | t]
    SegProgram sp_apply;  // allgather x -> phase 1 -> phase 2
    SegProgram sp_apply_m;   // the same for up to kMrhsMax columns (DMMA engine)
    DBuf<double> xt_loc_m;
    // multi-RHS hot path (world == 1): blocks of kMrhsMax columns, row-major n x kMrhsMax vectors
    DBuf<double> xt_m;
    Program prog_apply_m;
    DBuf<double> y_m;     // internal n x kMrhsMax result (epilogue pass input)
};

struct HLU {
    Ctx* ctx;
    const HMat* F;
    hm_lu_params params;
    std::shared_ptr<hla::HFactor> host_factor;   // host-only contexts: the factors in solve form
    int64_t hlu_truncations = 0;                 // stage B statistics (hm_storage_report)
    double hlu_threads = 0;
    std::vector<HOp> fwd, bwd;   // per level above the cut (may be empty ops)
    HOp leafL, leafU;            // block-diagonal inverse factors of the cut-level diagonal blocks
    int cut_level = 0;
    DBuf<double> xtA;            // [b | t] forward pass (t sized for the largest level)
    DBuf<double> xtB;            // [y | t] backward pass
    DBuf<double> z;              // internal-order result
    DBuf<double> eps_int, eps_ext, g_int;
    DBuf<double> amb_int, amb_pad;   // hm_set_ambient: A_i (1 - c_i), internal / padded order
    bool ambient = false;
    double t_inf4 = 0.0;
    DBuf<double> host_stage_in, host_stage_out;
    double setup_seconds[4] = {0, 0, 0, 0};
    int64_t bytes = 0, bytes_leaf = 0, n_blocks = 0, n_lr = 0, rank_sum = 0;
    int rank_max = 0;
    Program prog_solve;   // permute-in -> forward levels -> leaf L^-1 -> backward levels -> leaf U^-1
    Program prog_solve_h; // the same behind a copy-in pass for a pinned host b (single vector)
    Program prog_flux;    // prologue -> solve passes -> F phase 1 -> F phase 2 + flux epilogue
    Program prog_flux_h;  // the same behind a copy-in pass for a pinned host T (single vector)
    DBuf<double> T_dev;   // its device copy of T
    // sharded hot path (world > 1, inverse-factor form): this rank's rows of L^-1, U^-1
    HOp leafL_loc, leafU_loc;
    std::vector<HOp> fwd_loc, bwd_loc;   // level-form W operators, this rank's rows
    DBuf<double> T_loc;                  // sharded level-form flux: gathered temperatures (padded)
    const double* T_pad = nullptr;       // where the sharded flux epilogue reads T
    DBuf<double> xtA_loc, xtB_loc;
    DBuf<double> eps_pad, area_pad, g_pad;
    SegProgram sp_solve;  // AG b -> L^-1 -> AG y -> U^-1
    SegProgram sp_flux;   // AG T -> L^-1 (w = eps T^4 fused) -> AG y -> U^-1 -> AG z -> F + flux epilogue
    // sharded multi-RHS (cut level 0): the same exchanges on n_pad x 64 blocks, DMMA engine
    SegProgram sp_solve_m, sp_flux_m;
    DBuf<double> xtA_loc_m, xtB_loc_m, T_loc_m, y_loc_m;
    // multi-RHS hot path (world == 1, inverse-factor form)
    DBuf<double> xtA_m, xtB_m;
    Program prog_solve_m, prog_flux_m;
};

// ------------------------------------------------------------------ kernel launchers (kernels_*.cu)
namespace k {
// assembly
void aca_batch(const double* geo, int64_t n, const int64_t* blk /*[nb][4] r0,m,c0,n*/,
               const int64_t* uoff, const int64_t* voff, int probes, const int32_t* kcap, int nb, double eps,
               double* scratch, int32_t* rank_out, double* margin_out, int32_t* err, cudaStream_t s,
               int64_t max_m, int64_t max_n, const double* quad = nullptr);
// quad: the adaptive-quadrature table of reading R35 (internal order, kQStride doubles per facet) or null
void fill_entries(const double* geo, int64_t n, const int64_t* tasks /*[nt][6] dst,r0,rows,c0,cols,dld*/,
                  int nt, double* arena, int32_t* err, cudaStream_t s, const double* quad = nullptr);
// dst element (i,j) at arena[dst + j*dld + i] = src[i*rs + j*cs] (src absolute address)
void pack(const int64_t* tasks /*[nt][7] dst,src,rows,cols,rs,cs,dld*/, int nt, double* arena, cudaStream_t s);
void scale_rows(const int64_t* tasks /*[nt][5] a_off,ld,m,ncols,r0*/, int nt, double* arena, const double* cdiv,
                cudaStream_t s);
void fill_value(double* p, int64_t n, double v, cudaStream_t s);
void proj_facets(const int64_t* rp, const int32_t* col_idx, const double* val, const double* T, const double* x,
                 int mode, int ld, int col, double* eta, int64_t n, cudaStream_t s);
// out[N * ld + col] = sum_{r < world} buf[r * count + N] in rank order (sharded node reduction)
void sum_segments(const double* buf, int world, int64_t count, int64_t n, int ld, int col, double* out, cudaStream_t s);
void proj_nodes(const int64_t* tp, const int32_t* tidx, const double* tval, const double* y, int ld, int col, double* Q,
                int64_t n_nodes, cudaStream_t s);
void row_sums_clamp(const double* y, const double* area, double* sv, double* c, double* cdiv,
                    int64_t n, cudaStream_t s);
// dense linear algebra (setup)
void expand_C(const int64_t* tasks /*[nt][10]*/, int nt, const double* arena, const double* lam,
              double* M, int64_t ld, cudaStream_t s);
void add_identity(double* M, int64_t ld, int64_t n, cudaStream_t s);
// C = beta*C + alpha*op(A)*op(B); tri: 0 none, 1 lower-unit, 2 upper (masking of the operand)
void dgemm(int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda, int triA,
           const double* B, int64_t ldb, int triB, double beta, double* C, int64_t ldc, cudaStream_t s);
void leaf_lu_inv(double* M, double* Minv, int64_t ld, int n, int32_t* err, cudaStream_t s);
void extract_tri(const double* Minv, int64_t ld, int64_t r0, int64_t m, int mode, double* dst, cudaStream_t s);
void copy2d(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows, int64_t cols,
            cudaStream_t s);
// ACA factor recompression (kernels_recompress.cu): blk[5 q + 0..4] = uoff, m, voff, n, k (k in [2, 64])
void recompress_batch(double* base, const int64_t* blk, int nb, double eps, int32_t* new_rank, cudaStream_t s);
void cpaca_batch(double* T, int64_t ldt, const int64_t* blk /*[nb][7] i0,m,j0,n,uoff,voff,ld (<=0: ldt)*/,
                 const int32_t* kcap, int nb, double eps, double* fac, int32_t* rank_out,
                 cudaStream_t s);
}  // namespace k

double now_seconds();

// Read an operator's phase-2 items back from its arena (hlu.cpp): fn(item, payload, V) with the
// item's payload (dense m x ncols or U slice m x k, column-major) and, for low-rank items with
// want_v(item), the block's V (ncols x k column-major; else nullptr).  Synchronous.
void read_items(Ctx* c, const HOp& op, const std::function<bool(size_t)>& want_v,
                const std::function<void(size_t, const double*, const double*)>& fn);
// geom block index of every phase-2 item of an operator built in F's partition
std::vector<int> item_blocks(const Geom& g, const HOp& op);

// hot-path launches for one column (api.cpp): world == 1 -> one engine program; sharded -> the
// segmented program with its exchange steps
int64_t vec_rows(const Geom& g);
ProgArgs base_args(const Geom& g, const double* in, double* out, int ld, int col);
void launch_flux_m(HLU& L, const double* Td, double* qd, int ld, int r, cudaStream_t s);
void launch_apply(Ctx* c, HMat& F, const double* xd, double* yd, int ld, int col, cudaStream_t s);
void launch_solve(Ctx* c, HLU& L, const double* bd, double* zd, int ld, int col, cudaStream_t s);
void launch_flux(Ctx* c, HLU& L, const double* Td, double* qd, int ld, int col, cudaStream_t s,
                 unsigned long long* trace = nullptr);

}  // namespace hm

struct hm_ctx { hm::Ctx c; };
struct hm_geom { hm::Geom g; };
struct hm_hmat { hm::HMat h; };
struct hm_hlu { hm::HLU h; };
namespace hm {
// Facet <- node projection P and its transpose, CSR on the device (NEXT-1).
struct Proj {
    Ctx* ctx;
    const Geom* geom;
    int64_t n_facets = 0, n_nodes = 0;
    DBuf<int64_t> rp, tp;       // rows: facets (external order) / nodes
    DBuf<int32_t> ci, ti;       // node ids / facet ids
    DBuf<double> cv, tv;
    DBuf<double> eta, rbar;     // facet workspaces (external order)
    DBuf<double> host_in, host_in2, host_out;
    // sharded (world > 1): this rank's facets (internal rows [lb, le)) as CSR rows in local order, the
    // transpose restricted to them, and the allgather buffer of per-rank node partials (qcount each)
    DBuf<int64_t> rp_loc, tp_loc;
    DBuf<int32_t> ci_loc, ti_loc;
    DBuf<double> cv_loc, tv_loc, eta_loc, rbar_loc, qpart;
    int64_t n_loc = 0, qcount = 0;
};
}  // namespace hm
struct hm_proj { hm::Proj p; };
