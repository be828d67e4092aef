// Persistent pipelined stream engine: one cooperative launch executes a whole hot-path program
// (SURVEY.md §8(a) rows a1-a7): flux prologue / permute, the level-scheduled forward and backward
// substitution sweeps, the leaf inverses, both phases of the F apply and the flux epilogue.
//
// One CTA per SM (co-resident by cooperative launch), warp-specialised, through a kStages-deep
// shared-memory ring of 32 KB chunks:
//   warp 0 (producer): grabs tasks (a panel, or a piece of a big panel) from a monotone queue
//          counter in topological order and streams their chunks with 1-D TMA bulk copies
//          (cp.async.bulk, mbarrier transaction counts): payload + 16-byte aligned column sources;
//   warps 1-2 (gatherers; warp w owns the stages s = w-1 mod 2, so two gathers are in flight and
//          each warp still visits every phase of its barriers in order): before gathering for a
//          task, wait for the task's dependencies (per-pass or per-tree-node counters), then load
//          the chunk's inputs from L2 (ld.cg: written by other SMs) into the stage;
//   warps 3-7 (consumers): multiply from shared memory and accumulate the task in registers;
//          release each stage as soon as it is read; at the task's last chunk reduce in fixed
//          order, emit once (pieces of a split panel combine deterministically), retire the task
//          (cumulative fence, then the pass / node counters).
//
// Deadlock freedom: tasks are grabbed in increasing (topological) order and every wait refers to
// lower-numbered tasks, so the lowest unfinished task can always proceed.  Counters are monotone
// over launches (targets are epoch * count), so nothing is reset between launches.  Factor payload
// is constant, so the TMA ring keeps streaming while gatherers wait.
#include <cstdint>

#include "engine.h"
#include "hm_internal.h"

namespace hm {
namespace {

constexpr int kThreads = 288;      // warp 0 producer, warps 1-2 gatherers, warps 3..7 consumers, warp 8 L2 prefetcher
constexpr int kPrefetchWarp = 8;
constexpr int64_t kPrefetchWindow = 1536;   // chunks (~48 MB) ahead of the task-queue frontier
constexpr int kGatherers = 2;
constexpr int kConsumers = 160;
constexpr int kConsumerWarps = kConsumers / 32;
constexpr int kConsumer0 = 32 * (1 + kGatherers);
constexpr int kStages = 4;         // multiple of kGatherers
constexpr int kMaxCols = 512;      // per chunk; payload <= 32 KB
static_assert(kStages % kGatherers == 0, "stage ownership");

struct __align__(16) Stage {
    double payload[kUnitPayloadDoubles];
    double xs[kMaxCols];
    int32_t cs[kMaxCols];
};

struct EngineSmem {
    Stage st[kStages];
    int64_t hdr[kStages];      // chunk index in flight in each stage (-1: end of work)
    int64_t hdr_task[kStages]; // its task
    double2 red[kConsumers];
    unsigned long long full[kStages], gathered[kStages], empty[kStages];
    int last;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, unsigned long long* b) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(b))
        : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory"); }
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ double pow4(double T) {
    const double t2 = T * T;
    return t2 * t2;
}

__device__ __forceinline__ void emit(const ProgArgs& A, const Pass& P, int64_t row, double s) {
    switch (P.mode) {
        case OUT_ASSIGN: P.out[row] = s; break;
        case OUT_SUB: P.out[row] = __ldcg(P.out + row) - s; break;
        case OUT_PERM: A.user_out[(int64_t)A.perm[row] * A.ld + A.col] = s; break;
        default: {  // OUT_FLUX: q = sigma (eps/A) (F z - eta g)  (eq:qi_new_location, operator form)
            const int64_t e = A.perm[row];
            const double eta = pow4(A.user_in[e * A.ld + A.col]);
            A.user_out[e * A.ld + A.col] = A.sigma * (A.eps_int[row] / A.area_int[row]) * (s - eta * A.g_int[row]);
        }
    }
}

__device__ void wait_counter(const ProgArgs& A, int id, int cnt) {
    const unsigned long long target = A.epoch * (unsigned long long)cnt;
    const unsigned long long* d = A.done + id;
    unsigned ns = 20;
    while (true) {
        unsigned long long v;
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(d) : "memory");
        if (v >= target) break;
        __nanosleep(ns);
        if (ns < 160) ns <<= 1;
    }
}

__global__ void __launch_bounds__(kThreads, 1) engine_kernel(const ProgArgs A) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    EngineSmem& S = *reinterpret_cast<EngineSmem*>(smem_raw);
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&S.full[s], 1);
            mbar_init(&S.gathered[s], 1);
            mbar_init(&S.empty[s], kConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == 0) {
        // ------------------------------------------------ producer: grab tasks, TMA their chunks
        if (lane == 0) {
            int64_t k = 0;
            while (true) {
                const unsigned long long t = atomicAdd(A.queue, 1ull) - A.queue_base;
                const bool end = t >= (unsigned long long)A.n_tasks;
                const Task task = end ? Task{} : A.tasks[t];
                // end of work: one marker per gatherer warp (each owns its own stages)
                const int nch = end ? kGatherers : task.n_units;
                for (int c = 0; c < nch; ++c, ++k) {
                    const int s = (int)(k % kStages);
                    if (k >= kStages) mbar_wait(&S.empty[s], (uint32_t)(((k / kStages) - 1) & 1));
                    if (end) {
                        S.hdr[s] = -1;
                        mbar_arrive(&S.full[s]);
                        continue;
                    }
                    const int64_t ui = task.first_unit + c;
                    S.hdr[s] = ui;
                    S.hdr_task[s] = (int64_t)t;
                    const Unit& u = A.units[ui];
                    if (u.type != UNIT_STREAM) {
                        mbar_arrive(&S.full[s]);
                        continue;
                    }
                    const Pass& P = A.passes[u.pass];
                    const uint32_t pb = (uint32_t)u.ncols * (uint32_t)u.ld * 8u;
                    const uint32_t cb = (((uint32_t)u.ncols + 3u) & ~3u) * 4u;
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_expect_tx(&S.full[s], pb + cb);
                    tma_load_1d(S.st[s].payload, P.arena + u.a_off, pb, &S.full[s]);
                    tma_load_1d(S.st[s].cs, P.colsrc + u.cs_off, cb, &S.full[s]);
                }
                if (end) break;
            }
        }
        return;
    }
    if (warp == kPrefetchWarp) {
        // ------------------------------------------------ L2 prefetcher: stream the program's chunks into
        // L2 in program order, at most kPrefetchWindow chunks ahead of the task-queue frontier, so HBM
        // stays busy while tasks wait on their dependencies
        while (true) {
            const unsigned long long p = atomicAdd(A.pf_counter, 1ull) - A.pf_base;
            if (p >= (unsigned long long)A.n_units) break;
            unsigned ns = 64;
            while (true) {
                unsigned long long q;
                asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(q) : "l"(A.queue) : "memory");
                q -= A.queue_base;
                const int64_t frontier = q < (unsigned long long)A.n_tasks ? A.tasks[q].first_unit : A.n_units;
                if ((int64_t)p < frontier + kPrefetchWindow) break;
                __nanosleep(ns);
                if (ns < 1024) ns <<= 1;
            }
            const Unit& u = A.units[p];
            if (u.type == UNIT_STREAM) {
                const Pass& P = A.passes[u.pass];
                prefetch_l2(P.arena + u.a_off, (uint32_t)u.ncols * (uint32_t)u.ld * 8u);
            }
        }
        return;
    }
    if (warp <= kGatherers) {
        // ------------------------------------------------ gatherers: warp w owns stages s = w-1 (mod 2)
        int64_t verified = -1;  // last task whose waits this warp has checked
        for (int64_t k = warp - 1;; k += kGatherers) {
            const int s = (int)(k % kStages);
            mbar_wait(&S.full[s], (uint32_t)((k / kStages) & 1));
            const int64_t ui = S.hdr[s];
            if (ui >= 0) {
                const Unit& u = A.units[ui];
                const Pass& P = A.passes[u.pass];
                const int64_t ti = S.hdr_task[s];
                if (ti != verified) {
                    const Task& t = A.tasks[ti];
                    if (lane == 0) {
                        if (t.wait_id[0] >= 0) wait_counter(A, t.wait_id[0], t.wait_cnt[0]);
                        if (t.wait_id[1] >= 0) wait_counter(A, t.wait_id[1], t.wait_cnt[1]);
                        if (A.trace && u.chunk == 0) atomicMin(A.trace + 2 * u.pass, gtimer());
                    }
                    __syncwarp();
                    __threadfence();
                    verified = ti;
                }
                if (u.type == UNIT_STREAM) {
                    const double* in = P.in ? P.in : A.user_in;
                    const int32_t* cs = S.st[s].cs;
                    constexpr int kPer = kMaxCols / 32;
                    double v[kPer];
#pragma unroll
                    for (int q = 0; q < kPer; ++q) {
                        const int c = lane + 32 * q;
                        v[q] = c < u.ncols ? __ldcg(in + cs[c]) : 0.0;
                    }
#pragma unroll
                    for (int q = 0; q < kPer; ++q) {
                        const int c = lane + 32 * q;
                        if (c < u.ncols) S.st[s].xs[c] = v[q];
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.gathered[s]);
            if (ui < 0) break;
        }
        return;
    }
    // ---------------------------------------------------- consumers: accumulate a task's chunks in
    // registers, reduce and emit once per task
    const int ct = tid - kConsumer0;
    double2 acc = make_double2(0.0, 0.0), acc2 = acc;
    for (int64_t k = 0;; ++k) {
        const int s = (int)(k % kStages);
        mbar_wait(&S.gathered[s], (uint32_t)((k / kStages) & 1));
        const int64_t ui = S.hdr[s];
        if (ui < 0) break;
        const int64_t ti = S.hdr_task[s];
        const Unit u = A.units[ui];
        const Pass P = A.passes[u.pass];
        const int Pp = (u.nrows + 1) >> 1;
        const int G = kConsumers / Pp;
        const int g = ct / Pp;
        const int p = ct - g * Pp;
        if (u.type == UNIT_STREAM) {
            if (u.chunk == 0) acc = acc2 = make_double2(0.0, 0.0);
            if (g < G) {
                const double2* a = reinterpret_cast<const double2*>(S.st[s].payload) + p;
                const double* xs = S.st[s].xs;
                const int ld2 = u.ld >> 1;
                int c = g;
                for (; c + G < u.ncols; c += 2 * G) {
                    const double2 a0 = a[c * ld2], a1 = a[(c + G) * ld2];
                    const double x0 = xs[c], x1 = xs[c + G];
                    acc.x = fma(a0.x, x0, acc.x);
                    acc.y = fma(a0.y, x0, acc.y);
                    acc2.x = fma(a1.x, x1, acc2.x);
                    acc2.y = fma(a1.y, x1, acc2.y);
                }
                if (c < u.ncols) {
                    const double2 a0 = a[c * ld2];
                    const double x0 = xs[c];
                    acc.x = fma(a0.x, x0, acc.x);
                    acc.y = fma(a0.y, x0, acc.y);
                }
            }
        } else {
            for (int i = ct; i < u.nrows; i += kConsumers) {   // element-wise: rows [out0, out0 + nrows)
                const int64_t row = u.out0 + i;
                const double v = A.user_in[(int64_t)A.perm[row] * A.ld + A.col];
                P.out[row] = u.type == UNIT_PROLOGUE ? A.eps_int[row] * pow4(v) : v;
            }
        }
        // stage consumed: release it to the producer (per warp, no CTA-wide barrier)
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.empty[s]);
        if (u.chunk != u.nchunks - 1) continue;
        // ---- last chunk of the task
        if (u.type == UNIT_STREAM) {
            if (g < G) S.red[g * Pp + p] = make_double2(acc.x + acc2.x, acc.y + acc2.y);
            consumers_sync();
            const bool owner = ct < Pp;
            double2 sum = make_double2(0.0, 0.0);
            if (owner) {
                sum = S.red[ct];
                for (int q = 1; q < G; ++q) {
                    const double2 v = S.red[q * Pp + ct];
                    sum.x += v.x;
                    sum.y += v.y;
                }
            }
            if (u.grp < 0) {
                if (owner) {
                    emit(A, P, u.out0 + 2 * ct, sum.x);
                    if (2 * ct + 1 < u.nrows) emit(A, P, u.out0 + 2 * ct + 1, sum.y);
                }
            } else {  // panel split into pieces: the last-finishing piece adds the partials in order
                if (owner) reinterpret_cast<double2*>(P.part + u.part_off)[ct] = sum;
                consumers_sync();
                if (ct == 0) {
                    __threadfence();
                    S.last = (atomicAdd(P.counters + u.grp, 1) == u.nseg - 1);
                    if (S.last) __threadfence();
                }
                consumers_sync();
                if (S.last) {
                    if (owner) {
                        double2 t = make_double2(0.0, 0.0);
                        for (int q = 0; q < u.nseg; ++q) {  // piece q's partial sits (q - seg) * ld doubles away
                            const double2 v = __ldcg(reinterpret_cast<const double2*>(P.part + u.part_off) +
                                                     (int64_t)(q - u.seg) * (u.ld >> 1) + ct);
                            t.x += v.x;
                            t.y += v.y;
                        }
                        emit(A, P, u.out0 + 2 * ct, t.x);
                        if (2 * ct + 1 < u.nrows) emit(A, P, u.out0 + 2 * ct + 1, t.y);
                    }
                    if (ct == 0) P.counters[u.grp] = 0;
                }
            }
        }
        // ---- retire the task: outputs visible to other SMs (cumulative fence after the barrier)
        consumers_sync();
        if (ct == 0) {
            const Task& t = A.tasks[ti];
            __threadfence();
            atomicAdd(A.done + u.pass, 1ull);
            if (t.inc_id[0] >= 0) atomicAdd(A.done + t.inc_id[0], 1ull);
            if (t.inc_id[1] >= 0) atomicAdd(A.done + t.inc_id[1], 1ull);
            if (A.trace) atomicMax(A.trace + 2 * u.pass + 1, gtimer());
        }
    }
}

}  // namespace

size_t engine_smem_bytes() { return sizeof(EngineSmem) + 128; }

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
