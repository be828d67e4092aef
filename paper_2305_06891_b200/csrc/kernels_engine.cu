// Persistent pipelined stream engine: one cooperative launch executes a whole hot-path program
// (SURVEY.md §8(a) rows a1-a7): flux prologue / permute, the level-scheduled forward and backward
// substitution sweeps, the leaf inverses, both phases of the F apply and the flux epilogue.
//
// One CTA per SM (co-resident by cooperative launch), warp-specialised, 19 warps:
//   warp 0 (producer, one thread): grabs tasks (a panel, or a piece of a big panel) from a monotone
//          queue counter in topological order; per chunk it TMA-copies the chunk descriptor into a
//          header/gather slot (12-slot ring) and, kLookahead = 9 chunks later, the chunk's payload into
//          a 56.6 KB payload stage (3-stage ring), both with 1-D bulk copies and mbarrier transaction counts;
//   warps 1-4 (gatherers; warp w owns the header slots k = w-1 mod 4): before gathering for a task,
//          wait for the task's dependencies (per-pass or per-tree-node counters), then load the
//          chunk's inputs from L2 (ld.cg: written by other SMs) into the slot;
//   warps 5-12 (consumers): multiply from shared memory and accumulate the task in registers;
//          release each stage as soon as it is read; at the task's last chunk hand the per-thread
//          partials to a retire slot;
//   warps 13-18 (retire; warp w takes task ends k = w mod 6): reduce the partials in fixed order,
//          emit once (pieces of a split panel combine deterministically), publish the task (release
//          atomics on the pass / node counters).
//
// Deadlock freedom: tasks are grabbed in increasing (topological) order and every wait refers to
// lower-numbered tasks, so the lowest unfinished task can always proceed.  Counters are monotone
// over launches (targets are epoch * count), so nothing is reset between launches.  Factor payload
// is constant, so the TMA ring keeps streaming while gatherers wait.
#include <cstdint>

#include "engine.h"
#include "engine_dev.cuh"
#include "hm_internal.h"

namespace hm {
namespace {
using namespace dev;

// warp roles
constexpr int kGatherers = 4;                       // warps 1..4 (gatherer w owns header slots k = w-1 mod 4)
constexpr int kConsumerWarps = 8;                   // warps 5..12
constexpr int kConsumers = 32 * kConsumerWarps;
constexpr int kConsumer0 = 32 * (1 + kGatherers);
constexpr int kRetireWarp = 1 + kGatherers + kConsumerWarps;   // warps 13..18
constexpr int kRetireWarps = 6;   // 2 -> 6: the retire (emit + release) was the C2 bottleneck
constexpr int kThreads = 32 * (kRetireWarp + kRetireWarps);  // 608

// Two rings: payload stages (TMA of the factor bytes) and header/gather slots (chunk descriptor +
// gathered inputs).  The producer posts a chunk's header kLookahead chunks before it issues its
// payload, so the input gather (an L2 round trip) is finished by the time the payload lands.
#ifndef HM_PSTAGES
#define HM_PSTAGES 3
#endif
#ifndef HM_GSLOTS
#define HM_GSLOTS 12
#endif
#ifndef HM_RSLOTS
#define HM_RSLOTS 6
#endif
// Stage geometry (160 -> 170 KB of payload stages): 5 x 32 KB -> 3 x 56.6 KB chunks
// (HM_STAGE_DOUBLES = 7240): each CTA's pipe is bound by a per-chunk cost, so fewer, larger chunks
// win -- C2 flux 182.4 -> 171.5 us, C3 flux 0.910 -> 0.822 ms, C4 apply 2.011 -> 1.954 ms
// (scripts/gpu_stage_sweep*.sh; 4 x 42 KB is within 1 % of this)
constexpr int kPStages = HM_PSTAGES;
constexpr int kGSlots = HM_GSLOTS;
constexpr int kLookahead = kGSlots - kPStages;
constexpr int kRetireSlots = HM_RSLOTS;    // task-end handoff buffers (consumers -> retire warps)
constexpr int kMaxCols = 256;      // per chunk; payload <= kStageDoubles
constexpr int kMaxPasses = 64;     // pass table held in shared memory
static_assert(kGSlots % kGatherers == 0, "slot ownership");

struct __align__(16) PStage {
    double payload[kStageDoubles];
};

// Header/gather slot: the chunk's descriptor (TMA-copied by the producer: everything the gatherers
// and consumers need, so that no role issues a dependent global-memory load per chunk) and the
// gathered inputs.  hdr.type < 0: end-of-work marker.
struct __align__(16) GSlot {
    Unit hdr;
    double xs[kMaxCols];
};

// Task-end handoff: the consumers deposit their per-thread partial sums and the task's descriptor,
// the retire warp reduces, emits, publishes (fence + counters) off the consumers' critical path.
struct TaskEnd {       // what the retire warps need of a task's last chunk
    int32_t type, pass, nrows, ld, grp, nseg, seg, pad;
    int64_t out0, part_off;
};
struct RetireSlot {
    double2 red[kConsumers];
    TaskEnd u;         // u.type < 0: end of work
    int32_t inc_id[2];
};

struct EngineSmem {
    PStage st[kPStages];
    GSlot gs[kGSlots];
    Pass passes[kMaxPasses];   // the program's pass table, copied once per launch
    RetireSlot rs[kRetireSlots];
    unsigned long long gready[kGSlots], gathered[kGSlots], gempty[kGSlots];
    unsigned long long full[kPStages], pempty[kPStages];
    unsigned long long rfull[kRetireSlots], rempty[kRetireSlots];
    unsigned long long epoch;   // this launch's epoch (read_epoch)
};
// the whole engine state must fit the 227 KB opt-in limit (HM_BUILD_DEFINES overrides of the stage
// geometry fail here, at compile time, instead of at the first launch)
static_assert(sizeof(EngineSmem) + 128 <= 232448, "engine shared memory exceeds 227 KB");
static_assert(kLookahead > 0 && (kStageDoubles * 8) % 16 == 0, "stage geometry");

__device__ __forceinline__ void emit(const ProgArgs& A, const Pass& P, int64_t row, double s) {
    switch (P.mode) {
        case OUT_ASSIGN: P.out[row] = s; break;
        case OUT_SUB: P.out[row] = __ldcg(P.out + row) - s; break;
        case OUT_PERM: A.user_out[(int64_t)A.perm[row] * A.ld + A.col] = s; break;
        case OUT_LOCAL: A.user_out[(row - A.local0) * A.ld + A.col] = s; break;
        case OUT_FLUX_LOCAL: {   // sharded; eta_in / rbar_out as in OUT_FLUX (sharded cavity operator)
            const double t = __ldcg(A.T_pad + row);
            const double eta = A.eta_in ? t : pow4(t);
            const double sc = A.rbar_out ? A.eps_int[row] : A.eps_int[row] / A.area_int[row];
            const double amb = A.amb ? A.amb[row] * (eta - A.t_inf4) : 0.0;   // eqn:flux_to_ambient (R34)
            A.user_out[(row - A.local0) * A.ld + A.col] = A.sigma * sc * (s - eta * A.g_int[row] + amb);
            break;
        }
        default: {  // OUT_FLUX: q = sigma (eps/A) (F z - eta g)  (eq:qi_new_location, operator form);
                    // rbar_out: A o q = (Rbar eta)_i (eq:Rbardef)
            const int64_t e = A.perm[row];
            const double in = A.user_in[e * A.ld + A.col];
            const double eta = A.eta_in ? in : pow4(in);
            const double sc = A.rbar_out ? A.eps_int[row] : A.eps_int[row] / A.area_int[row];
            const double amb = A.amb ? A.amb[row] * (eta - A.t_inf4) : 0.0;   // eqn:flux_to_ambient (R34)
            A.user_out[e * A.ld + A.col] = A.sigma * sc * (s - eta * A.g_int[row] + amb);
        }
    }
}

__global__ void __launch_bounds__(kThreads, 1) engine_kernel(const ProgArgs A) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    EngineSmem& S = *reinterpret_cast<EngineSmem*>(smem_raw);
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int g = 0; g < kGSlots; ++g) {
            mbar_init(&S.gready[g], 1);
            mbar_init(&S.gathered[g], 1);
            mbar_init(&S.gempty[g], kConsumerWarps);
        }
        for (int p = 0; p < kPStages; ++p) {
            mbar_init(&S.full[p], 1);
            mbar_init(&S.pempty[p], kConsumerWarps);
        }
        for (int r = 0; r < kRetireSlots; ++r) {
            mbar_init(&S.rfull[r], kConsumerWarps);
            mbar_init(&S.rempty[r], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        read_epoch(A, &S.epoch);
    }
    for (int i = tid; i < A.n_passes; i += kThreads) S.passes[i] = A.passes[i];
    __syncthreads();
    const unsigned long long epoch = S.epoch;
    const unsigned long long queue_base = (epoch - 1) * (unsigned long long)(A.n_tasks + gridDim.x);

    if (warp == 0) {
        // ------------------------------------------------ producer (one thread): grab tasks; per chunk,
        // TMA its descriptor into a header slot (the gather starts when it lands) and, kLookahead chunks
        // behind, TMA its payload.  The next task index (atomic) and its Task record are requested one
        // task ahead, so the issue loop never waits on a global load.
        if (lane != 0) return;
        unsigned long long st_empty = 0, st_meta = 0, st_chunks = 0, st_pempty = 0;
        const long long t_start = clock64();
        const uint64_t pol = l2_evict_first_policy();
        int64_t k = 0;     // headers posted
        int64_t kp = 0;    // payloads issued
        auto issue_payload = [&]() {
            const int p = (int)(kp % kPStages);
            const int g = (int)(kp % kGSlots);
            long long c0 = clock64();
            mbar_wait(&S.gready[g], (uint32_t)((kp / kGSlots) & 1));   // its descriptor has landed
            if (kp >= kPStages) mbar_wait(&S.pempty[p], (uint32_t)(((kp / kPStages) - 1) & 1));
            st_pempty += clock64() - c0;
            const Unit& u = S.gs[g].hdr;
            if (u.type == UNIT_STREAM) {
#if HM_DEVICE_CHECKS
                check_payload(A, u.pass, u.a_off, u.ncols, u.ld);
#endif
                const uint32_t pb = (uint32_t)u.ncols * (uint32_t)u.ld * 8u;
                mbar_expect_tx(&S.full[p], pb);
                if (HM_PAYLOAD_EVICT_FIRST)
                    tma_load_1d_hint(S.st[p].payload, S.passes[u.pass].arena + u.a_off, pb, &S.full[p], pol);
                else
                    tma_load_1d(S.st[p].payload, S.passes[u.pass].arena + u.a_off, pb, &S.full[p]);
            } else {
                mbar_arrive(&S.full[p]);
            }
            ++kp;
        };
        auto wait_slot = [&](int64_t kk) {
            const int g = (int)(kk % kGSlots);
            long long c0 = clock64();
            if (kk >= kGSlots) mbar_wait(&S.gempty[g], (uint32_t)(((kk / kGSlots) - 1) & 1));
            st_empty += clock64() - c0;
            return g;
        };
        unsigned long long t = atomicAdd(A.queue, 1ull) - queue_base;
        bool have_t = t < (unsigned long long)A.n_tasks;
        unsigned long long tn = ~0ull;   // pending grab of the next task index
        Task task{};
        if (have_t) {
            tn = atomicAdd(A.queue, 1ull) - queue_base;
            task = A.tasks[t];
        }
        while (have_t) {
            long long c0 = clock64();
            const bool have_n = tn < (unsigned long long)A.n_tasks;
            Task task_n{};
            unsigned long long tnn = ~0ull;
            if (have_n) {
                task_n = A.tasks[tn];
                tnn = atomicAdd(A.queue, 1ull) - queue_base;
            }
            st_meta += clock64() - c0;
            const int nch = task.n_units;
#if HM_DEVICE_CHECKS
            if (task.first_unit < 0 || nch < 1 || task.first_unit + nch > A.n_units) {
                printf("hm device check failed: task %llu units [%lld, +%d) of %lld\n", t, (long long)task.first_unit, nch,
                       (long long)A.n_units);
                __trap();
            }
#endif
            for (int c = 0; c < nch; ++c) {
                const int g = wait_slot(k);
                ++st_chunks;
                mbar_expect_tx(&S.gready[g], (uint32_t)sizeof(Unit));
                tma_load_1d(&S.gs[g].hdr, A.units + task.first_unit + c, (uint32_t)sizeof(Unit), &S.gready[g]);
                ++k;
                if (k - kp > kLookahead) issue_payload();
            }
            t = tn;
            tn = tnn;
            task = task_n;
            have_t = have_n;
        }
        while (kp < k) issue_payload();
        // end of work: one marker per gatherer warp (each owns its own slots); no payload
        for (int c = 0; c < kGatherers; ++c) {
            const int g = wait_slot(k);
            S.gs[g].hdr.type = -1;
            mbar_arrive(&S.gready[g]);
            ++k;
        }
        if (A.stats) {
            atomicAdd(A.stats + 0, st_empty);
            atomicAdd(A.stats + 1, st_meta);
            atomicAdd(A.stats + 2, st_chunks);
            atomicAdd(A.stats + 11, st_pempty);
            atomicAdd(A.stats + 12, (unsigned long long)(clock64() - t_start));
        }
        return;
    }
    if (warp >= 1 && warp <= kGatherers) {
        // ------------------------------------------------ gatherers: warp w owns header slots k = w-1 (mod kGatherers)
        int64_t verified = -1;  // last task whose waits this warp has checked
        int sat_id[2] = {-1, -1};                 // recently satisfied counters (lane 0)
        unsigned long long sat_tgt[2] = {0, 0};
        unsigned long long st_full = 0, st_dep = 0, st_gather = 0;
        for (int64_t k = warp - 1;; k += kGatherers) {
            const int s = (int)(k % kGSlots);
            long long c0 = clock64();
            mbar_wait(&S.gready[s], (uint32_t)((k / kGSlots) & 1));
            long long c1 = clock64();
            st_full += c1 - c0;
            const Unit& H = S.gs[s].hdr;
            const int type = H.type;
            if (type >= 0) {
                const int64_t ti = H.task;
                if (ti != verified) {
                    // dependency waits (acquire); counters only grow, so a (counter, target) pair
                    // already seen satisfied by this warp is not polled again
                    if (lane == 0) {
#pragma unroll
                        for (int q = 0; q < 2; ++q) {
                            const int id = H.wait_id[q];
                            if (id < 0) continue;
                            const unsigned long long tgt = epoch * (unsigned long long)H.wait_cnt[q];
                            if (id == sat_id[0] && tgt <= sat_tgt[0]) continue;
                            if (id == sat_id[1] && tgt <= sat_tgt[1]) continue;
                            wait_counter(A, epoch, id, H.wait_cnt[q]);
                            sat_id[1] = sat_id[0]; sat_tgt[1] = sat_tgt[0];
                            sat_id[0] = id; sat_tgt[0] = tgt;
                        }
                        if (A.trace && H.chunk == 0) atomicMin(A.trace + 2 * H.pass, gtimer());
                    }
                    __syncwarp();
                    verified = ti;
                }
                c0 = clock64();
                st_dep += c0 - c1;
#if HM_DEVICE_CHECKS
                if (type == UNIT_STREAM) check_chunk(A, H, S.passes[H.pass < A.n_passes ? H.pass : 0], kMaxCols, kStageDoubles, lane);
#endif
                if (type == UNIT_STREAM) {
                    const Pass& P = S.passes[H.pass];
                    const double* in = P.in ? P.in : A.user_in;
                    const int32_t* cs = P.colsrc + H.cs_off;   // global (static): chunks without runs
                    const int ncols = H.ncols;
                    const int im = P.in_mode;
                    constexpr int kPer = kMaxCols / 32;
                    double v[kPer];
                    if ((im == IN_PLAIN || im == IN_FLUXI) && H.nruns > 0) {
                        // run-encoded column sources: lane's columns c = lane + 32 q are increasing, so
                        // its run index only moves forward
                        const int nr = H.nruns;
                        int r = 0, rs = 0, rl = H.run_len[0];
                        int32_t rsrc = H.run_src[0];
                        int32_t idx[kPer];
#pragma unroll
                        for (int q = 0; q < kPer; ++q) {
                            const int c = lane + 32 * q;
                            while (r < nr - 1 && c >= rs + rl) {
                                rs += rl;
                                ++r;
                                rl = H.run_len[r];
                                rsrc = H.run_src[r];
                            }
                            idx[q] = c < ncols ? rsrc + (c - rs) : -1;
                        }
#pragma unroll
                        for (int q = 0; q < kPer; ++q) v[q] = idx[q] >= 0 ? __ldcg(in + idx[q]) : 0.0;
                        if (im == IN_FLUXI) {   // sharded flux prologue: w_j = eps_j T_j^4 (x region)
#pragma unroll
                            for (int q = 0; q < kPer; ++q)
                                if (idx[q] >= 0 && idx[q] < A.n_x) v[q] = __ldg(A.eps_int + idx[q]) * (A.eta_in ? v[q] : pow4(v[q]));
                        }
                    } else if (im == IN_PLAIN || im == IN_FLUXI) {
                        int32_t idx[kPer];
#pragma unroll
                        for (int q = 0; q < kPer; ++q) {
                            const int c = lane + 32 * q;
                            idx[q] = c < ncols ? __ldg(cs + c) : -1;
                        }
#pragma unroll
                        for (int q = 0; q < kPer; ++q) v[q] = idx[q] >= 0 ? __ldcg(in + idx[q]) : 0.0;
                        if (im == IN_FLUXI) {
#pragma unroll
                            for (int q = 0; q < kPer; ++q)
                                if (idx[q] >= 0 && idx[q] < A.n_x) v[q] = __ldg(A.eps_int + idx[q]) * (A.eta_in ? v[q] : pow4(v[q]));
                        }
                    } else {
                        // fused prologue: x-region inputs come straight from the caller's external-order
                        // vector (colsrc_ext holds -(external index + 1)); IN_FLUX: w = eps * T^4
                        // (eq:qi_new_location)
#pragma unroll
                        for (int q = 0; q < kPer; ++q) {
                            const int c = lane + 32 * q;
                            const int32_t j = c < ncols ? __ldg(cs + c) : 0;
                            if (c >= ncols) {
                                v[q] = 0.0;
                            } else if (j >= 0) {
                                v[q] = __ldcg(in + j);
                            } else {
                                const int64_t e = -(int64_t)j - 1;
                                // coherent load: after a copy-in pass the input is written earlier in
                                // this launch (the dependency wait is the acquire)
                                const double t = __ldcg(A.user_in + e * A.ld + A.col);
                                v[q] = im == IN_PERM ? t : __ldg(A.eps_ext + e) * (A.eta_in ? t : pow4(t));
                            }
                        }
                    }
#pragma unroll
                    for (int q = 0; q < kPer; ++q) {
                        const int c = lane + 32 * q;
                        if (c < ncols) S.gs[s].xs[c] = v[q];
                    }
                }
            }
            __syncwarp();
            if (type >= 0) st_gather += clock64() - c0;
            if (lane == 0) mbar_arrive(&S.gathered[s]);
            if (type < 0) break;
        }
        if (A.stats && lane == 0) {
            atomicAdd(A.stats + 3, st_full);
            atomicAdd(A.stats + 4, st_dep);
            atomicAdd(A.stats + 5, st_gather);
        }
        return;
    }
    if (warp >= kRetireWarp && warp < kRetireWarp + kRetireWarps) {
        // ------------------------------------------------ retire warp: per task, reduce the consumers'
        // partial sums in fixed order, emit (split panels: publish the partial, the last-finishing piece
        // adds all partials in piece order), then publish the task (release fence, dependency counters)
        unsigned long long st_rwait = 0, st_rwork = 0;
        for (int64_t k = warp - kRetireWarp;; k += kRetireWarps) {   // retire warp w: task ends k = w (mod kRetireWarps)
            const int r = (int)(k % kRetireSlots);
            long long c0 = clock64();
            mbar_wait(&S.rfull[r], (uint32_t)((k / kRetireSlots) & 1));
            long long c1 = clock64();
            st_rwait += c1 - c0;
            const RetireSlot& R = S.rs[r];
            struct { int32_t type, pass, nrows, ld, grp, nseg, seg; int64_t out0, part_off; } u;
            u.type = R.u.type; u.pass = R.u.pass; u.nrows = R.u.nrows; u.ld = R.u.ld; u.grp = R.u.grp;
            u.nseg = R.u.nseg; u.seg = R.u.seg; u.out0 = R.u.out0; u.part_off = R.u.part_off;
            if (u.type < 0) break;
            const int32_t inc0 = R.inc_id[0], inc1 = R.inc_id[1];
            const Pass& P = S.passes[u.pass];
            const int Pp = (u.nrows + 1) >> 1;
            const int G = kConsumers / Pp;
            double2 sum[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
            if (u.type == UNIT_STREAM) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int pp = lane + 32 * h;
                    if (pp < Pp) {
                        double2 t = R.red[pp];
                        for (int q = 1; q < G; ++q) {
                            const double2 v = R.red[q * Pp + pp];
                            t.x += v.x;
                            t.y += v.y;
                        }
                        sum[h] = t;
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.rempty[r]);   // slot free: the consumers may deposit the next task
            if (u.type == UNIT_STREAM) {
                if (u.grp < 0) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int pp = lane + 32 * h;
                        if (pp < Pp) {
                            emit(A, P, u.out0 + 2 * pp, sum[h].x);
                            if (2 * pp + 1 < u.nrows) emit(A, P, u.out0 + 2 * pp + 1, sum[h].y);
                        }
                    }
                } else {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int pp = lane + 32 * h;
                        if (pp < Pp) reinterpret_cast<double2*>(P.part + u.part_off)[pp] = sum[h];
                    }
                    __syncwarp();
                    int last = 0;
                    if (lane == 0) last = (atom_add_acq_rel(P.counters + u.grp, 1) == u.nseg - 1);
                    last = __shfl_sync(0xffffffffu, last, 0);
                    if (last) {
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int pp = lane + 32 * h;
                            if (pp < Pp) {
                                double2 t = make_double2(0.0, 0.0);
                                for (int q = 0; q < u.nseg; ++q) {  // piece q's partial sits (q - seg) * ld doubles away
                                    const double2 v = __ldcg(reinterpret_cast<const double2*>(P.part + u.part_off) +
                                                             (int64_t)(q - u.seg) * (u.ld >> 1) + pp);
                                    t.x += v.x;
                                    t.y += v.y;
                                }
                                emit(A, P, u.out0 + 2 * pp, t.x);
                                if (2 * pp + 1 < u.nrows) emit(A, P, u.out0 + 2 * pp + 1, t.y);
                            }
                        }
                        if (lane == 0) P.counters[u.grp] = 0;
                    }
                }
            }
            // ---- publish: outputs (this warp's, and the element-wise ones the consumers wrote before
            // their mbarrier release) visible GPU-wide before the counters move
            __syncwarp();
            if (lane == 0) {
                if (u.type != UNIT_STREAM) __threadfence();   // element-wise outputs were written by the consumers
                red_release(A.done + u.pass, 1ull);
                if (inc0 >= 0) red_release(A.done + inc0, 1ull);
                if (inc1 >= 0) red_release(A.done + inc1, 1ull);
                if (A.trace) atomicMax(A.trace + 2 * u.pass + 1, gtimer());
            }
            st_rwork += clock64() - c1;
        }
        if (A.stats && lane == 0) {
            atomicAdd(A.stats + 9, st_rwait);
            atomicAdd(A.stats + 10, st_rwork);
        }
        return;
    }
    // ---------------------------------------------------- consumers: accumulate a task's chunks in
    // registers; at the task's last chunk hand the per-thread partials to the retire warp
    const int ct = tid - kConsumer0;
    double2 acc = make_double2(0.0, 0.0), acc2 = acc;
    unsigned long long st_wait = 0, st_comp = 0, st_task = 0, st_wg = 0;
    int64_t ntask = 0;
    long long c0 = clock64();
    for (int64_t k = 0;; ++k) {
        const int gsl = (int)(k % kGSlots);
        const int s = (int)(k % kPStages);
        mbar_wait(&S.gathered[gsl], (uint32_t)((k / kGSlots) & 1));
        const long long cg = clock64();
        st_wg += cg - c0;
        const Unit& H = S.gs[gsl].hdr;
        struct { int32_t type, pass, nrows, ld, ncols, chunk, nchunks, grp, nseg, seg; int64_t out0, part_off; } u;
        u.type = H.type; u.pass = H.pass; u.nrows = H.nrows; u.ld = H.ld; u.ncols = H.ncols;
        u.chunk = H.chunk; u.nchunks = H.nchunks; u.out0 = H.out0;
        u.grp = H.grp; u.nseg = H.nseg; u.seg = H.seg; u.part_off = H.part_off;
        const int32_t inc0 = H.inc_id[0], inc1 = H.inc_id[1];
        if (u.type >= 0) mbar_wait(&S.full[s], (uint32_t)((k / kPStages) & 1));
        long long c1 = clock64();
        st_wait += c1 - c0;
        if (u.type < 0) {   // end of work: one marker per retire warp
            for (int w = 0; w < kRetireWarps; ++w, ++ntask) {
                const int r = (int)(ntask % kRetireSlots);
                if (ntask >= kRetireSlots) mbar_wait(&S.rempty[r], (uint32_t)(((ntask / kRetireSlots) - 1) & 1));
                if (ct == 0) S.rs[r].u.type = -1;
                asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");   // slot reuse across markers
                if (lane == 0) mbar_arrive(&S.rfull[r]);
            }
            break;
        }
        const Pass& P = S.passes[u.pass];
        const int Pp = (u.nrows + 1) >> 1;
        const int G = kConsumers / Pp;
        const int g = ct / Pp;
        const int p = ct - g * Pp;
        if (u.type == UNIT_STREAM) {
            if (u.chunk == 0) acc = acc2 = make_double2(0.0, 0.0);
            if (g < G) {
                const double2* a = reinterpret_cast<const double2*>(S.st[s].payload) + p;
                const double* xs = S.gs[gsl].xs;
                const int ld2 = u.ld >> 1;
                const int nc = u.ncols;
                int c = g;
                for (; c + 3 * G < nc; c += 4 * G) {
                    const double2 a0 = a[c * ld2], a1 = a[(c + G) * ld2];
                    const double2 a2 = a[(c + 2 * G) * ld2], a3 = a[(c + 3 * G) * ld2];
                    const double x0 = xs[c], x1 = xs[c + G], x2 = xs[c + 2 * G], x3 = xs[c + 3 * G];
                    acc.x = fma(a0.x, x0, acc.x);
                    acc.y = fma(a0.y, x0, acc.y);
                    acc2.x = fma(a1.x, x1, acc2.x);
                    acc2.y = fma(a1.y, x1, acc2.y);
                    acc.x = fma(a2.x, x2, acc.x);
                    acc.y = fma(a2.y, x2, acc.y);
                    acc2.x = fma(a3.x, x3, acc2.x);
                    acc2.y = fma(a3.y, x3, acc2.y);
                }
                for (; c < nc; c += G) {
                    const double2 a0 = a[c * ld2];
                    const double x0 = xs[c];
                    acc.x = fma(a0.x, x0, acc.x);
                    acc.y = fma(a0.y, x0, acc.y);
                }
            }
        } else {
            if (u.type == UNIT_COPYIN) {   // pinned host input -> device copy (overlaps the payload stream)
                // four PCIe reads in flight per thread (the unit is latency-bound)
                for (int i0 = ct; i0 < u.nrows; i0 += 4 * kConsumers) {
                    double v[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int i = i0 + q * kConsumers;
                        v[q] = i < u.nrows ? A.host_in[(u.out0 + i) * A.ld + A.col] : 0.0;
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int i = i0 + q * kConsumers;
                        if (i < u.nrows) P.out[(u.out0 + i) * A.ld + A.col] = v[q];
                    }
                }
            } else if (u.type == UNIT_PROLOGUE_INT) {   // sharded: w = eps T^4 in place on padded internal rows
                for (int i = ct; i < u.nrows; i += kConsumers) {
                    const int64_t row = u.out0 + i;
                    P.out[row] = A.eps_int[row] * (A.eta_in ? P.in[row] : pow4(P.in[row]));
                }
            } else {
                for (int i = ct; i < u.nrows; i += kConsumers) {   // element-wise: rows [out0, out0 + nrows)
                    const int64_t row = u.out0 + i;
                    const double v = A.user_in[(int64_t)A.perm[row] * A.ld + A.col];
                    P.out[row] = u.type == UNIT_PROLOGUE ? A.eps_int[row] * (A.eta_in ? v : pow4(v)) : v;
                }
            }
        }
        // chunk consumed: release its payload stage and header slot (per warp, no CTA-wide barrier)
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(&S.pempty[s]);
            mbar_arrive(&S.gempty[gsl]);
        }
        c0 = clock64();
        st_comp += c0 - c1;
        if (u.chunk != u.nchunks - 1) continue;
        // ---- last chunk of the task: deposit partials + descriptor, hand off to the retire warp
        const int r = (int)(ntask % kRetireSlots);
        if (ntask >= kRetireSlots) mbar_wait(&S.rempty[r], (uint32_t)(((ntask / kRetireSlots) - 1) & 1));
        ++ntask;
        RetireSlot& R = S.rs[r];
        if (u.type == UNIT_STREAM && g < G) R.red[g * Pp + p] = make_double2(acc.x + acc2.x, acc.y + acc2.y);
        if (ct == 0) {
            R.u = TaskEnd{u.type, u.pass, u.nrows, u.ld, u.grp, u.nseg, u.seg, 0, u.out0, u.part_off};
            R.inc_id[0] = inc0;
            R.inc_id[1] = inc1;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.rfull[r]);
        const long long c2 = clock64();
        st_task += c2 - c0;
        c0 = c2;
    }
    if (A.stats && ct == 0) {
        atomicAdd(A.stats + 6, st_wait);
        atomicAdd(A.stats + 7, st_comp);
        atomicAdd(A.stats + 8, st_task);
        atomicAdd(A.stats + 13, st_wg);
    }
}

}  // namespace

size_t engine_smem_bytes() { return sizeof(EngineSmem) + 128; }
int engine_max_passes() { return kMaxPasses; }

static void set_attr() {
    static bool attr = false;
    if (!attr) {
        HM_CUDA(cudaFuncSetAttribute(engine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)engine_smem_bytes()));
        attr = true;
    }
}

void engine_launch(const ProgArgs& A, int grid, cudaStream_t s) {
    set_attr();
    void* args[] = {const_cast<ProgArgs*>(&A)};
    HM_CUDA(cudaLaunchCooperativeKernel((const void*)engine_kernel, dim3(grid), dim3(kThreads), args,
                                        engine_smem_bytes(), s));
    debug_sync(s, "engine_kernel");
}

int engine_grid() {
    int dev = 0, sms = 0, per = 0;
    HM_CUDA(cudaGetDevice(&dev));
    HM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    set_attr();
    HM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, engine_kernel, kThreads, engine_smem_bytes()));
    if (per < 1) throw Error(HM_ERR_CUDA, "engine kernel does not fit on an SM");
    return sms * per;
}

}  // namespace hm
