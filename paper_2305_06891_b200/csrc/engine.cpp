// Host side of the persistent stream engine: assemble passes, chunks and tasks into a program and
// derive each task's dependency waits.
//
// Level-form sweeps (DESIGN.md §"Solve in level form"): the update of node t reads b[t1] and
// writes b[t2]; every ancestor's update writes rows of t (RAW) or reads rows t writes (WAR), and
// every descendant's update touches rows t reads or writes.  So the sweep's dependency graph is
// the cluster tree itself: a node's tasks wait for its nearest ancestor with work to have retired
// (which transitively covers all ancestors), and a node's phase-2 tasks also wait for its own
// phase-1 tasks (the t = V^T b values).  Independent subtrees never wait for each other; only the
// sweep boundaries (forward -> backward -> F apply) are barriers.
#include "engine.h"

#include <cstdio>
#include <algorithm>
#include <cstdlib>

namespace hm {

int add_stream_impl(Program& P, const StreamPass& sp, const HOp& op, const double* in, double* out, int mode, int kind,
                    const std::vector<int32_t>* panel_node, int in_mode, int xdep) {
    if (sp.h_units.empty()) return -1;
    Pass p{};
    p.type = UNIT_STREAM;
    p.dep = (int32_t)P.h_passes.size() - 1;
    p.mode = mode;
    p.in_mode = in_mode;
    p.first_unit = (int64_t)P.h_units.size();
    p.n_units = (int64_t)sp.h_units.size();
    p.arena = op.arena.p;
    // IN_FLUXI (sharded flux) gathers by internal padded index like IN_PLAIN; colsrc_ext (external
    // indices, fused prologue) exists only for unsharded operators
    p.colsrc = (in_mode == IN_PLAIN || in_mode == IN_FLUXI) ? op.colsrc.p : op.colsrc_ext.p;
    if (!p.colsrc) throw Error(HM_ERR_NOT_READY, "stream pass without column sources for its input mode");
    p.in = in;
    p.out = out;
    p.part = sp.part.p;
    p.counters = sp.counters.p;
    const int32_t idx = (int32_t)P.h_passes.size();
    const int64_t base = (int64_t)P.h_units.size();
    for (size_t q = 0; q < sp.h_units.size(); ++q) {
        Unit u = sp.h_units[q];
        u.pass = idx;
        u.type = UNIT_STREAM;
        u.first_chunk += base;
        if (u.chunk == 0) {
            Task t{};
            t.first_unit = (int64_t)P.h_units.size();
            t.n_units = u.nchunks;
            t.pass = idx;
            t.wait_id[0] = t.wait_id[1] = t.inc_id[0] = t.inc_id[1] = -1;
            P.h_tasks.push_back(t);
            P.task_kind.push_back(kind);
            P.task_node.push_back(panel_node ? (*panel_node)[sp.unit_panel[q]] : -1);
            P.task_xonly.push_back(sp.unit_xonly[q]);
            P.task_key.push_back(sp.panels[sp.unit_panel[q]].key);
            P.task_span.push_back(sp.panels[sp.unit_panel[q]].ncols);
            ++p.n_tasks;
        }
        P.h_units.push_back(u);
    }
    P.h_passes.push_back(p);
    P.pass_xdep.push_back(xdep);
    const DBuf<int32_t>& cs = (in_mode == IN_PLAIN || in_mode == IN_FLUXI) ? op.colsrc : op.colsrc_ext;
    P.h_chk.insert(P.h_chk.end(), {(int64_t)op.arena.n, (int64_t)cs.n, op.xt_len});
    return idx;
}

void Program::add_stream(const StreamPass& sp, const HOp& op, const double* in, double* out, int mode, int kind,
                         const std::vector<int32_t>* panel_node, int in_mode, int xdep) {
    add_stream_impl(*this, sp, op, in, out, mode, kind, panel_node, in_mode, xdep);
}

void Program::add_elementwise(int type, int64_t n, double* out, int rows_per_unit, const double* in, int mode,
                              int64_t row0) {
    Pass p{};
    p.type = type;
    p.dep = (int32_t)h_passes.size() - 1;
    p.mode = mode;
    p.first_unit = (int64_t)h_units.size();
    p.out = out;
    p.in = in;
    const int32_t idx = (int32_t)h_passes.size();
    for (int64_t r = row0; r < row0 + n; r += rows_per_unit) {
        Unit u{};
        u.out0 = r;
        u.nrows = (int32_t)std::min<int64_t>(rows_per_unit, row0 + n - r);
        u.grp = -1;
        u.nseg = 1;
        u.pass = idx;
        u.type = type;
        u.chunk = 0;
        u.nchunks = 1;
        u.first_chunk = (int64_t)h_units.size();
        Task t{};
        t.first_unit = (int64_t)h_units.size();
        t.n_units = 1;
        t.pass = idx;
        t.wait_id[0] = t.wait_id[1] = t.inc_id[0] = t.inc_id[1] = -1;
        h_tasks.push_back(t);
        task_kind.push_back(DEP_BARRIER);
        task_node.push_back(-1);
        task_xonly.push_back(0);
        task_key.push_back(r);
        task_span.push_back(0);
        h_units.push_back(u);
    }
    p.n_units = (int64_t)h_units.size() - p.first_unit;
    p.n_tasks = p.n_units;
    h_passes.push_back(p);
    pass_xdep.push_back(-2);
    h_chk.insert(h_chk.end(), {0, 0, 0});
}

void Program::finalize(Ctx* ctx, cudaStream_t s, const Geom* g) {
    for (const Unit& u : h_units)
        if (u.type == UNIT_STREAM && (u.ncols > (mrhs ? kMrhsMaxCols : kUnitMaxCols) || u.ld > 128 ||
                                      (int64_t)u.ncols * u.ld > (mrhs ? kMrhsPayloadDoubles : kStageDoubles)))
            throw Error(HM_ERR_UNSUPPORTED, "work unit exceeds the engine stage size");
    const int64_t P = (int64_t)h_passes.size();
    if (P > (mrhs ? engine_mrhs_max_passes() : engine_max_passes()))
        throw Error(HM_ERR_UNSUPPORTED, "program has " + std::to_string(P) + " passes, more than the " +
                                            (mrhs ? "multi-RHS" : "single-vector") + " engine's pass table (" +
                                            std::to_string(mrhs ? engine_mrhs_max_passes() : engine_max_passes()) +
                                            "; pure level form needs 7 + 4 depth)");
    const int64_t nn = g ? (int64_t)g->nodes.size() : 0;
    // row groups for link_rows: the tree nodes of level depth - 4 (leaves above it are groups too)
    std::vector<int32_t> groups;           // node ids, in row order
    if (g && !row_links.empty()) {
        int depth = 0;
        for (const Node& N : g->nodes) depth = std::max(depth, (int)N.level);
        const int lg = std::max(0, depth - 4);
        std::vector<int32_t> st{0};
        while (!st.empty()) {
            const int id = st.back();
            st.pop_back();
            const Node& N = g->nodes[id];
            if (N.level == lg || N.is_leaf()) { groups.push_back(id); continue; }
            st.push_back(N.child[1]);
            st.push_back(N.child[0]);
        }
    }
    const int64_t ng = (int64_t)groups.size();
    auto group_of = [&](int64_t row) {   // index of the group containing row (groups are in row order)
        int64_t lo = 0, hi = ng - 1;
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) / 2;
            if (g->nodes[groups[mid]].begin <= row) lo = mid; else hi = mid - 1;
        }
        return lo;
    };
    const int64_t c_rows0 = P + 4 * nn;
    n_counters = c_rows0 + (int64_t)row_links.size() * ng;
    auto c_p1 = [&](int sw, int node) { return (int32_t)(P + sw * 2 * nn + node); };
    auto c_all = [&](int sw, int node) { return (int32_t)(P + sw * 2 * nn + nn + node); };
    std::vector<int64_t> cnt(n_counters, 0);  // tasks that increment each counter
    auto sweep_of = [](int kind) { return kind >= DEP_BWD_P1 ? 1 : 0; };
    for (size_t i = 0; i < h_tasks.size(); ++i) {
        Task& t = h_tasks[i];
        const int kind = task_kind[i], node = task_node[i];
        cnt[t.pass]++;
        if (kind == DEP_FWD_P1 || kind == DEP_BWD_P1) {
            t.inc_id[0] = c_p1(sweep_of(kind), node);
            t.inc_id[1] = c_all(sweep_of(kind), node);
        } else if (kind == DEP_FWD_P2 || kind == DEP_BWD_P2) {
            t.inc_id[0] = c_all(sweep_of(kind), node);
        }
        for (int li = 0; li < (int)row_links.size(); ++li) {   // phase-2 tasks feed their row group
            if (t.pass != row_links[li].first) continue;
            const int slot = t.inc_id[0] < 0 ? 0 : t.inc_id[1] < 0 ? 1 : -1;
            if (slot < 0) throw Error(HM_ERR_UNSUPPORTED, "no free counter slot for a row-group link");
            t.inc_id[slot] = (int32_t)(c_rows0 + li * ng + group_of(task_key[i]));
        }
        for (int q = 0; q < 2; ++q)
            if (t.inc_id[q] >= 0) cnt[t.inc_id[q]]++;
    }
    for (size_t i = 0; i < h_tasks.size(); ++i) {
        Task& t = h_tasks[i];
        const int kind = task_kind[i], node = task_node[i];
        int nw = 0;
        auto wait = [&](int32_t id) {
            if (id >= 0 && cnt[id] > 0 && nw < 2) {
                t.wait_id[nw] = id;
                t.wait_cnt[nw] = (int32_t)cnt[id];
                ++nw;
            }
        };
        const bool xonly = task_xonly[i] != 0;
        if (kind == DEP_BARRIER) {
            // HM_DIAG_DEPS (timing experiments only, results are wrong): "none" drops every wait,
            // "intra" the phase-1 -> phase-2 waits, "cross" the operator-to-operator waits
            static const char* diagb = [] {
                const char* e = getenv("HM_DIAG_DEPS");
                if (e) fprintf(stderr, "[hm] HM_DIAG_DEPS=%s: dependency waits dropped -- timing experiment, results are WRONG\n", e);
                return e;
            }();
            const char* diag = diagb;
            const int xd = pass_xdep[t.pass];
            if (diag && diag[0] == 'n') continue;
            if (diag && diag[0] == 'i' && xd != -2) { wait(xd); continue; }
            if (diag && diag[0] == 'c' && (xonly || xd == -2 || pass_xdep[t.pass] == t.pass - 1)) {
                if (!xonly && xd != -2) wait(t.pass - 1);
                continue;
            }
            wait(xonly && xd != -2 ? xd : t.pass - 1);
            continue;
        }
        if (!g || node < 0) throw Error(HM_ERR_INVALID_ARG, "tree-dependency pass without tree nodes");
        const int sw = sweep_of(kind);
        static const char* diag = getenv("HM_DIAG_DEPS");
        if (diag && diag[0] == 'n') continue;
        int par = g->nodes[node].parent;
        while (par >= 0 && cnt[c_all(sw, par)] == 0) par = g->nodes[par].parent;
        if (!(diag && diag[0] == 'c')) {
            if (par >= 0) wait(c_all(sw, par));
            else wait(sweep_dep[sw]);
        }
        if ((kind == DEP_FWD_P2 || kind == DEP_BWD_P2) && !xonly && !(diag && diag[0] == 'i')) wait(c_p1(sw, node));
    }
    // row-group links: a phase-1 task whose cluster [key, key + span) lies in one group waits for that
    // group's phase-2 tasks of the linked pass instead of for the whole pass (its only input)
    for (int li = 0; li < (int)row_links.size(); ++li) {
        const int32_t p2 = row_links[li].first, p1 = row_links[li].second;
        for (size_t i = 0; i < h_tasks.size(); ++i) {
            Task& t = h_tasks[i];
            if (t.pass != p1) continue;
            const int64_t gi = group_of(task_key[i]);
            const Node& G = g->nodes[groups[gi]];
            if (task_key[i] + task_span[i] > G.end) continue;   // spans several groups: whole pass
            const int32_t id = (int32_t)(c_rows0 + li * ng + gi);
            for (int q = 0; q < 2; ++q)
                if (t.wait_id[q] == p2) {
                    t.wait_id[q] = cnt[id] > 0 ? id : -1;
                    t.wait_cnt[q] = (int32_t)cnt[id];
                }
        }
    }
    for (size_t i = 0; i < h_tasks.size(); ++i) {   // per-chunk copies of the task's dependency record
        const Task& t = h_tasks[i];
        for (int64_t q = t.first_unit; q < t.first_unit + t.n_units; ++q) {
            Unit& u = h_units[q];
            u.task = (int64_t)i;
            for (int j = 0; j < 2; ++j) {
                u.wait_id[j] = t.wait_id[j];
                u.wait_cnt[j] = t.wait_cnt[j];
                u.inc_id[j] = t.inc_id[j];
            }
        }
    }
    {   // HM_ENGINE_STATS=2: per-pass shape of the program (diagnostics)
        const char* e = getenv("HM_ENGINE_STATS");
        if (e && e[0] == '2') {
            for (size_t p = 0; p < h_passes.size(); ++p) {
                const Pass& P = h_passes[p];
                int64_t bytes = 0, nu = P.n_units, small = 0;
                for (int64_t u = P.first_unit; u < P.first_unit + P.n_units; ++u) {
                    const int64_t b = 8LL * h_units[u].ncols * h_units[u].ld;
                    bytes += b;
                    small += b < 16384;
                }
                fprintf(stderr, "[program %s] pass %zu type %d mode %d in %d: units %lld tasks %lld bytes %.1f MB "
                        "avg %.1f KB (<16KB: %lld)\n", mrhs ? "mrhs" : "1rhs", p, P.type, P.mode, P.in_mode,
                        (long long)nu, (long long)P.n_tasks, bytes / 1e6, nu ? bytes / 1e3 / nu : 0.0, (long long)small);
            }
        }
    }
#if HM_DEVICE_CHECKS
    // HM_CHECK_SELFTEST=1 (tests of the checked build): move one chunk past the end of its arena -- the
    // engine must trap on it
    if (const char* e = getenv("HM_CHECK_SELFTEST"); e && e[0] == '1')
        for (Unit& u : h_units)
            if (u.type == UNIT_STREAM) {
                u.a_off = h_chk[3 * (size_t)u.pass];
                break;
            }
#endif
    passes.upload(ctx, h_passes, "engine passes", s);
#if HM_DEVICE_CHECKS
    chk.upload(ctx, h_chk, "engine check bounds", s);
#endif
    units.upload(ctx, h_units, "engine units", s);
    tasks.upload(ctx, h_tasks, "engine tasks", s);
    done.alloc(ctx, (size_t)std::max<int64_t>(n_counters, 1), "engine dependency counters");
    HM_CUDA(cudaMemsetAsync(done.p, 0, sizeof(unsigned long long) * std::max<int64_t>(n_counters, 1), s));
    queue.alloc(ctx, 1, "engine task queue");
    HM_CUDA(cudaMemsetAsync(queue.p, 0, sizeof(unsigned long long), s));
    grid = mrhs ? engine_mrhs_grid() : engine_grid();
    {
        const unsigned long long e0[2] = {1ull, 0ull};
        epoch_dev.alloc(ctx, 2, "engine epoch");
        HM_CUDA(cudaMemcpyAsync(epoch_dev.p, e0, sizeof(e0), cudaMemcpyHostToDevice, s));
        HM_CUDA(cudaStreamSynchronize(s));
    }
    ready = true;
}

void Program::launch(ProgArgs a, cudaStream_t s) {
    if (h_tasks.empty()) return;
    a.passes = passes.p;
    a.n_passes = (int32_t)h_passes.size();
    a.n_x = n_x;
    a.units = units.p;
    a.tasks = tasks.p;
    a.n_tasks = (int64_t)h_tasks.size();
    a.queue = queue.p;
    // every CTA's producer takes exactly one index past the end: the counter advances by
    // n_tasks + grid per launch (the kernel derives its base from the device epoch)
    a.n_units = (int64_t)h_units.size();
    a.done = done.p;
    a.epoch_dev = epoch_dev.p;
    a.chk = chk.p;   // null unless HM_DEVICE_CHECKS
    if (a.ld == 0) a.ld = 1;
    static const bool want_stats = [] { const char* e = getenv("HM_ENGINE_STATS"); return e && e[0] == '1'; }();
    if (want_stats) {
        if (!stats.p) stats.alloc(nullptr, 16 + 64, "engine stats");
        HM_CUDA(cudaMemsetAsync(stats.p, 0, (16 + 64) * sizeof(unsigned long long), s));
        a.stats = stats.p;
    }
    // HM_TRACE_MRHS=1 (diagnostics): per-pass [first gather, last publish] of multi-RHS launches
    static const bool want_trace_m = [] { const char* e = getenv("HM_TRACE_MRHS"); return e && e[0] == '1'; }();
    std::vector<unsigned long long> tr_init;
    if (mrhs && want_trace_m && !a.trace) {
        const size_t np = h_passes.size();
        if (trace.n < 2 * np) trace.alloc(nullptr, 2 * np, "engine trace");
        tr_init.assign(2 * np, 0ull);
        for (size_t i = 0; i < np; ++i) tr_init[2 * i] = ~0ull;
        HM_CUDA(cudaMemcpyAsync(trace.p, tr_init.data(), 2 * np * sizeof(unsigned long long), cudaMemcpyHostToDevice, s));
        a.trace = trace.p;
    }
    if (mrhs) engine_mrhs_launch(a, grid, s);
    else engine_launch(a, grid, s);
    if (!tr_init.empty()) {
        const size_t np = h_passes.size();
        std::vector<unsigned long long> tr(2 * np);
        HM_CUDA(cudaMemcpyAsync(tr.data(), trace.p, 2 * np * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
        HM_CUDA(cudaStreamSynchronize(s));
        unsigned long long t0 = ~0ull;
        for (size_t i = 0; i < np; ++i) t0 = std::min(t0, tr[2 * i]);
        for (size_t i = 0; i < np; ++i) {
            double mb = 0;
            for (int64_t u = h_passes[i].first_unit; u < h_passes[i].first_unit + h_passes[i].n_units; ++u)
                mb += h_units[u].type == UNIT_STREAM ? 8e-6 * h_units[u].ncols * h_units[u].ld : 0.0;
            fprintf(stderr, "[mrhs trace] pass %zu type %d: %.1f -> %.1f us (%.1f MB)\n", i, h_passes[i].type,
                    tr[2 * i] == ~0ull ? -1.0 : (tr[2 * i] - t0) * 1e-3, (tr[2 * i + 1] - t0) * 1e-3, mb);
        }
    }
    if (want_stats) {
        unsigned long long h[16 + 64];
        HM_CUDA(cudaMemcpyAsync(h, stats.p, sizeof(h), cudaMemcpyDeviceToHost, s));
        HM_CUDA(cudaStreamSynchronize(s));
        const double G = (double)grid;
        fprintf(stderr,
                "[engine stats] passes %zu units %zu grid %d | per CTA (kcycles): producer wait-empty %.1f meta %.1f "
                "chunks %.0f | gatherer(sum of warps) wait-full %.1f dep %.1f gather %.1f | consumer wait %.1f "
                "compute %.1f task-end %.1f | retire wait %.1f work %.1f | producer wait-pempty %.1f total %.1f | consumer wait-gathered %.1f | handoff %.1f split-tasks %.0f\n",
                h_passes.size(), h_units.size(), grid, h[0] / G / 1e3, h[1] / G / 1e3, h[2] / G, h[3] / G / 1e3,
                h[4] / G / 1e3, h[5] / G / 1e3, h[6] / G / 1e3, h[7] / G / 1e3, h[8] / G / 1e3, h[9] / G / 1e3, h[10] / G / 1e3, h[11] / G / 1e3, h[12] / G / 1e3, h[13] / G / 1e3,
                h[14] / G / 1e3, (double)h[15]);
    }
}

void SegProgram::launch(Ctx* ctx, const Geom& g, ProgArgs a, cudaStream_t s) {
    const Shard& S = g.shard;
    for (size_t i = 0; i < segs.size(); ++i) {
        if (pre[i]) {   // (ctx->skip_exchange: compute-only timing of the segments, results not valid)
            if (pre_user[i]) {   // this rank's slice (columns a.col.. of the caller's n_loc x ld array)
                const int64_t nl = S.le() - S.lb();
                const size_t w = mrhs ? (size_t)a.nrhs : 1, dst_pitch = mrhs ? kMrhsMax : 1;
                if (nl > 0)
                    HM_CUDA(cudaMemcpy2DAsync(pre[i] + S.base() * dst_pitch, sizeof(double) * dst_pitch, a.user_in + a.col,
                                              sizeof(double) * (size_t)(a.ld ? a.ld : 1), sizeof(double) * w, (size_t)nl,
                                              cudaMemcpyDeviceToDevice, s));
            }
            if (!ctx->ex) throw Error(HM_ERR_NOT_READY, "sharded program without an exchanger");
            if (!ctx->skip_exchange) ctx->ex->allgather(pre[i], S.maxc * (mrhs ? kMrhsMax : 1), s);
            debug_sync(s, "allgather");
        }
        segs[i]->launch(a, s);
    }
}

}  // namespace hm
