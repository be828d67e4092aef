// Multi-RHS stream engine: the same programs as the single-vector engine
// (kernels_engine.cu) applied to a block of up to kMrhsMax = 64 right-hand sides at once, so every
// stored factor byte is read ONCE per 64 columns and the apply becomes a dense contraction
// (2 x 64 flop per 8 stored bytes = 16 flop/B, above the FP64 ridge): each chunk
//     out[rows, 0:r] += A[rows, cols] @ X[cols, 0:r]
// runs on the FP64 tensor pipe (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4; sm_100a's tcgen05 has no f64
// kind).  Vectors are row-major n x kMrhsMax (row i: its r values contiguous, 512 B).
//
// One CTA per SM, cooperative launch, warp-specialised over a 3-stage ring; each stage holds a
// chunk's descriptor, its payload (<= 32 KB, 1-D TMA) and its gathered X tile (<= 64 x 64):
//   warp 0      producer: tasks from the monotone queue, descriptors (lane-parallel loads), TMA;
//   warps 1-2   gatherers: dependency waits, then X rows (512 B each, coalesced) into the stage;
//   warps 3-10  consumers: DMMA over the chunk, accumulators (8x8 tiles) in registers across the
//               task; at the task's last chunk they emit (split panels: partial + last-arriver sum
//               in piece order) and publish the task (release fence, counters).
#include <cstdint>

#include "engine.h"
#include "engine_dev.cuh"
#include "hm_internal.h"

namespace hm {
namespace {
using namespace dev;

constexpr int kMGatherers = 2;
constexpr int kMConsumerWarps = 8;
constexpr int kMConsumers = 32 * kMConsumerWarps;
constexpr int kMConsumer0 = 32 * (1 + kMGatherers);
constexpr int kMPubWarp = 1 + kMGatherers + kMConsumerWarps;          // warp 11: publisher
constexpr int kMThreads = 32 * (kMPubWarp + 1);                        // 384
constexpr int kPubSlots = 8;          // task-end descriptors in flight (consumers -> publisher)
#ifndef HM_MRHS_STAGES
#define HM_MRHS_STAGES 3
#endif
constexpr int kMStages = HM_MRHS_STAGES;
// Shared-memory strides for conflict-free fragment loads: an 8-byte fragment load by a half-warp
// (lanes g = 0..3 row, t = 0..3 k) reads words t * stride + g; the 16 words fall into distinct bank
// pairs iff stride = 4 or 12 (mod 16).
// X tile row stride (doubles): 68, conflict-free B-fragment loads.  (Measured and removed: an unpadded
// stride 64, so that a run of consecutive input rows lands as ONE bulk copy -- C2 64-RHS flux 0.888 vs
// 0.779 ms: the 4-way B-fragment conflicts cost the consumers more than the per-row copy issue costs the
// gatherers.)
constexpr int kXStride = 68;
__host__ __device__ constexpr int padded_ld(int ld) {   // smem column stride of a chunk with ld rows
    return ld + ((ld & 15) <= 4 ? 4 - (ld & 15) : (ld & 15) <= 12 ? 12 - (ld & 15) : 20 - (ld & 15));
}
// shared-memory column stride of a chunk.  HM_MRHS_WHOLE_CHUNK = 2 (default): every chunk lands as ONE
// bulk copy of its contiguous payload (stride ld).  The producer is one warp, and per-column copies are
// issued lane by lane (a uniform-operand loop): at 64 copies per chunk that issue loop, not HBM, bounded
// the engine (C2 64-RHS flux 0.884 ms -> 0.779 ms).  The price is bank conflicts on the A-fragment
// loads of chunks whose ld is not 4, 8 or 12 (mod 16) (ncu: 1.63x the ideal shared wavefronts).  = 1: only
// those conflict-free chunks whole, the others per column at padded_ld(ld) (0.803 ms); = 0: all per
// column (0.884 ms)
#ifndef HM_MRHS_WHOLE_CHUNK
#define HM_MRHS_WHOLE_CHUNK 2
#endif
__host__ __device__ constexpr bool whole_chunk(int ld) {
    return HM_MRHS_WHOLE_CHUNK == 2 || (HM_MRHS_WHOLE_CHUNK && ((ld & 15) == 4 || (ld & 15) == 8 || (ld & 15) == 12));
}
__host__ __device__ constexpr int smem_ld(int ld) { return whole_chunk(ld) ? ld : padded_ld(ld); }
// payload columns land at stride padded_ld(ld) (one bulk copy per column): at most
// kMrhsPayloadDoubles + 6 * kMrhsMaxCols doubles
constexpr int kMPayload = kMrhsPayloadDoubles + (HM_MRHS_WHOLE_CHUNK == 2 ? 0 : 6 * kMrhsMaxCols);
constexpr int kMaxPassesM = 96;
constexpr int kMaxTiles = 16;         // 8x8 accumulator tiles per consumer warp (128 rows x 64 cols / 8 warps)

struct __align__(16) MStage {
    Unit hdr;
    double payload[kMPayload];
    double X[kMrhsMaxCols * kXStride];
};

struct PubDesc {        // what the publisher needs of a finished task
    int32_t type, pass, inc0, inc1;
};

struct MSmem {
    MStage st[kMStages];
    Pass passes[kMaxPassesM];
    PubDesc pub[kPubSlots];
    unsigned long long epoch;   // this launch's epoch (read_epoch)
    unsigned long long posted[kMStages], full[kMStages], gathered[kMStages], empty[kMStages];
    unsigned long long pfull[kPubSlots], pempty[kPubSlots];
    int last;
};

static_assert(sizeof(MSmem) + 128 <= 232448, "multi-RHS engine shared memory exceeds 227 KB");
static_assert(kMrhsMaxCols <= 64 && kMrhsMaxCols % 4 == 0, "X tile: the two gatherer warps cover <= 64 columns");
static_assert(padded_ld(40) == 44 && padded_ld(80) == 84 && padded_ld(126) == 132 && padded_ld(2) == 4, "padded_ld");

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

// One chunk's contraction for a warp owning TM tiles t = cw + 8 i: acc[i] += A[rows(t), :] X[:, cols(t)].
// Rows beyond the panel (garbage) only feed accumulator rows that are never emitted, so the full
// k-steps need no predicates; the k tail (ncols % 4) zeroes A (X rows there are zero, but stale A
// could be NaN).
template <int TM>
__device__ __forceinline__ void mma_chunk(double (&acc)[kMaxTiles][2], const double* __restrict__ Ap,
                                          const double* __restrict__ Xp, int ld, int ncols, int cw, int N8, int ar,
                                          int ak) {
    int arow[TM], bcol[TM];
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int t = cw + 8 * i;
        const int mt = N8 == 8 ? i : t / N8, nt = N8 == 8 ? cw : t - mt * N8;   // 64 RHS: no division
        arow[i] = mt * 8 + ar;
        bcol[i] = nt * 8 + ar;
    }
    const int nfull = ncols & ~3;
    if (8 % N8 == 0) {   // N8 in {1, 2, 4, 8}: nt = (cw + 8 i) mod N8 = cw mod N8 for every tile of the warp
        const int bc = bcol[0];
        for (int k4 = 0; k4 < nfull; k4 += 4) {
            const double* Ak = Ap + (k4 + ak) * ld;
            double a[TM];
#pragma unroll
            for (int i = 0; i < TM; ++i) a[i] = Ak[arow[i]];
            const double b = Xp[(k4 + ak) * kXStride + bc];
#pragma unroll
            for (int i = 0; i < TM; ++i) dmma(acc[i], a[i], b);
        }
    } else {
        for (int k4 = 0; k4 < nfull; k4 += 4) {
            const double* Ak = Ap + (k4 + ak) * ld;
            const double* Xk = Xp + (k4 + ak) * kXStride;
            double a[TM], b[TM];
#pragma unroll
            for (int i = 0; i < TM; ++i) {
                a[i] = Ak[arow[i]];
                b[i] = Xk[bcol[i]];
            }
#pragma unroll
            for (int i = 0; i < TM; ++i) dmma(acc[i], a[i], b[i]);
        }
    }
    if (nfull < ncols) {
        const int kk = nfull + ak;
        const bool kv = kk < ncols;
        const double* Ak = Ap + kk * ld;
        const double* Xk = Xp + kk * kXStride;
        double a[TM], b[TM];
#pragma unroll
        for (int i = 0; i < TM; ++i) {
            a[i] = kv ? Ak[arow[i]] : 0.0;
            b[i] = Xk[bcol[i]];
        }
#pragma unroll
        for (int i = 0; i < TM; ++i) dmma(acc[i], a[i], b[i]);
    }
}

// Warp tiling.  N8 == 8 (> 56 columns, the usual 64-RHS block): "2-D" -- consumer warp cw owns the
// column-tile pair {2 (cw & 3), 2 (cw & 3) + 1} and the row tiles mt = (cw >> 2) + 2 j, so each A
// fragment feeds two DMMAs and shared-memory fragment traffic per DMMA drops from (TM + 1) / TM to
// (TM / 2 + 2) / TM (shared memory is the co-bottleneck with the TMA writes).  Otherwise tiles
// t = cw + 8 i, (mt, nt) = (t / N8, t mod N8).  Tile i of the warp -> (mt, nt); false past the last.
// 64 columns and an odd number of row tiles <= 7 (40-row leaf panels: 5): one column tile per warp and
// every row tile ("1-D"), so all 8 warps issue the same M8 DMMAs per k-step (the 2-D tiling gives
// ceil(M8/2) and floor(M8/2) row tiles to the two warp halves).  Off by default: measured on C2 64-RHS
// flux 0.915 ms (1-D) vs 0.901 ms (2-D) -- the 2-D tiling's fewer shared-memory fragment loads per DMMA
// outweigh its imbalance; HM_MRHS_TILE1D=1 at build time selects 1-D
#ifndef HM_MRHS_GATHER_LDG
#define HM_MRHS_GATHER_LDG 0
#endif
#ifndef HM_MRHS_TILE1D
#define HM_MRHS_TILE1D 0
#endif
// rows in flight per consumer warp in the element-wise units (4: fewest register spills of the kernel)
// L2 policy of the phase-1 -> phase-2 scratch (t): 0 none; 1 evict-last stores of internal results;
// 2 also evict-last X-row gathers
#ifndef HM_MRHS_T_HINT
#define HM_MRHS_T_HINT 0
#endif
#ifndef HM_MRHS_EROWS
#define HM_MRHS_EROWS 4
#endif
__device__ __forceinline__ bool use_1d(int M8, int N8) { return HM_MRHS_TILE1D && N8 == 8 && (M8 & 1) && M8 <= 7; }

__device__ __forceinline__ bool warp_tile(int i, int cw, int M8, int N8, int& mt, int& nt) {
    if (use_1d(M8, N8)) {
        mt = i;
        nt = cw;
        return i < M8;
    }
    if (N8 == 8) {
        mt = (cw >> 2) + 2 * (i >> 1);
        nt = 2 * (cw & 3) + (i & 1);
        return mt < M8;
    }
    const int t = cw + 8 * i;
    mt = t / N8;
    nt = t - mt * N8;
    return t < M8 * N8;
}

// 2-D tiling (N8 == 8): RM row tiles x 2 column tiles, acc[2 j + c]
template <int RM>
__device__ __forceinline__ void mma_chunk2d(double (&acc)[kMaxTiles][2], const double* __restrict__ Ap,
                                            const double* __restrict__ Xp, int ld, int ncols, int cw, int ar,
                                            int ak) {
    int arow[RM];
#pragma unroll
    for (int j = 0; j < RM; ++j) arow[j] = ((cw >> 2) + 2 * j) * 8 + ar;
    const int bc = 2 * (cw & 3) * 8 + ar;
    const int nfull = ncols & ~3;
    for (int k4 = 0; k4 < nfull; k4 += 4) {
        const double* Ak = Ap + (k4 + ak) * ld;
        const double* Xk = Xp + (k4 + ak) * kXStride + bc;
        double a[RM];
#pragma unroll
        for (int j = 0; j < RM; ++j) a[j] = Ak[arow[j]];
        const double b0 = Xk[0], b1 = Xk[8];
#pragma unroll
        for (int j = 0; j < RM; ++j) {
            dmma(acc[2 * j], a[j], b0);
            dmma(acc[2 * j + 1], a[j], b1);
        }
    }
    if (nfull < ncols) {   // k tail: zero A past ncols (stale A could be NaN; X rows there are zero)
        const int kk = nfull + ak;
        const bool kv = kk < ncols;
        const double* Ak = Ap + kk * ld;
        const double* Xk = Xp + kk * kXStride + bc;
        double a[RM];
#pragma unroll
        for (int j = 0; j < RM; ++j) a[j] = kv ? Ak[arow[j]] : 0.0;
        const double b0 = Xk[0], b1 = Xk[8];
#pragma unroll
        for (int j = 0; j < RM; ++j) {
            dmma(acc[2 * j], a[j], b0);
            dmma(acc[2 * j + 1], a[j], b1);
        }
    }
}

// 1-D tiling: RM row tiles x this warp's column tile cw, acc[j]
template <int RM>
__device__ __forceinline__ void mma_chunk1d(double (&acc)[kMaxTiles][2], const double* __restrict__ Ap,
                                            const double* __restrict__ Xp, int ld, int ncols, int cw, int ar,
                                            int ak) {
    int arow[RM];
#pragma unroll
    for (int j = 0; j < RM; ++j) arow[j] = j * 8 + ar;
    const int bc = cw * 8 + ar;
    const int nfull = ncols & ~3;
    for (int k4 = 0; k4 < nfull; k4 += 4) {
        const double* Ak = Ap + (k4 + ak) * ld;
        double a[RM];
#pragma unroll
        for (int j = 0; j < RM; ++j) a[j] = Ak[arow[j]];
        const double b = Xp[(k4 + ak) * kXStride + bc];
#pragma unroll
        for (int j = 0; j < RM; ++j) dmma(acc[j], a[j], b);
    }
    if (nfull < ncols) {   // k tail: zero A past ncols (stale A could be NaN; X rows there are zero)
        const int kk = nfull + ak;
        const bool kv = kk < ncols;
        const double* Ak = Ap + kk * ld;
        double a[RM];
#pragma unroll
        for (int j = 0; j < RM; ++j) a[j] = kv ? Ak[arow[j]] : 0.0;
        const double b = Xp[kk * kXStride + bc];
#pragma unroll
        for (int j = 0; j < RM; ++j) dmma(acc[j], a[j], b);
    }
}

__device__ __forceinline__ void cons_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kMConsumers) : "memory"); }

// out[row, col] for the program's output mode; vectors inside the library are row-major with
// stride kMrhsMax, the caller's arrays with stride A.ld (external order)
__device__ __forceinline__ void emit_m(const ProgArgs& A, const Pass& P, int64_t row, int col, double s) {
    switch (P.mode) {
        case OUT_ASSIGN: P.out[row * kMrhsMax + col] = s; break;
        case OUT_SUB: P.out[row * kMrhsMax + col] = __ldcg(P.out + row * kMrhsMax + col) - s; break;
        case OUT_PERM: A.user_out[(int64_t)A.perm[row] * A.ld + col] = s; break;
        case OUT_LOCAL: A.user_out[(row - A.local0) * A.ld + col] = s; break;   // sharded: this rank's rows
        case OUT_FLUX_LOCAL: {   // sharded flux epilogue: T (padded rows x 64) and eps / A / g padded
            const double eta = pow4(__ldcg(A.T_pad + row * kMrhsMax + col));
            const double amb = A.amb ? A.amb[row] * (eta - A.t_inf4) : 0.0;   // eqn:flux_to_ambient (R34)
            A.user_out[(row - A.local0) * A.ld + col] =
                A.sigma * (A.eps_int[row] / A.area_int[row]) * (s - eta * A.g_int[row] + amb);
            break;
        }
        default: {  // OUT_FLUX: q = sigma (eps/A) (F z - eta g)  (eq:qi_new_location, operator form)
            const int64_t e = A.perm[row];
            const double eta = pow4(A.user_in[e * A.ld + col]);
            const double amb = A.amb ? A.amb[row] * (eta - A.t_inf4) : 0.0;   // eqn:flux_to_ambient (R34)
            A.user_out[e * A.ld + col] = A.sigma * (A.eps_int[row] / A.area_int[row]) * (s - eta * A.g_int[row] + amb);
        }
    }
}

__global__ void __launch_bounds__(kMThreads, 1) engine_mrhs_kernel(const ProgArgs A) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    MSmem& S = *reinterpret_cast<MSmem*>(smem_raw);
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int R = A.nrhs;                       // columns of this launch (<= 64)
    const int N8 = (R + 7) >> 3;                // 8-wide column tiles
    if (tid == 0) {
        for (int s = 0; s < kMStages; ++s) {
            mbar_init(&S.posted[s], 1);
            mbar_init(&S.full[s], 1);
            mbar_init(&S.gathered[s], kMGatherers);
            mbar_init(&S.empty[s], kMConsumerWarps);
        }
        for (int r = 0; r < kPubSlots; ++r) {
            mbar_init(&S.pfull[r], kMConsumerWarps);
            mbar_init(&S.pempty[r], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        read_epoch(A, &S.epoch);
    }
    for (int i = tid; i < A.n_passes; i += kMThreads) S.passes[i] = A.passes[i];
    __syncthreads();
    const unsigned long long epoch = S.epoch;
    const unsigned long long queue_base = (epoch - 1) * (unsigned long long)(A.n_tasks + gridDim.x);

    if (warp == 0) {
        // ------------------------------------------------ producer
        unsigned long long nxt = 0, st_e = 0, st_m = 0;
        const long long t0 = clock64();
        const uint64_t pol = l2_evict_first_policy();
        if (lane == 0) nxt = atomicAdd(A.queue, 1ull) - queue_base;
        nxt = __shfl_sync(0xffffffffu, nxt, 0);
        int64_t k = 0;
        while (true) {
            const unsigned long long t = nxt;
            const bool end = t >= (unsigned long long)A.n_tasks;
            Task task{};
            // element-wise units (prologue / permute / epilogue) are taken one at a time: the next task
            // index is grabbed only after the unit has been consumed.  Grabbing ahead let the first CTAs
            // to arrive hold up to four barrier-gated units each and run them back to back (C2 64-RHS
            // flux epilogue 42-50 us for 148 one-per-SM units)
            bool ew = false;
            if (!end) {
                task = A.tasks[t];
                ew = S.passes[task.pass].type != UNIT_STREAM;
                if (lane == 0 && !ew) nxt = atomicAdd(A.queue, 1ull) - queue_base;
            }
            const int nch = end ? 1 : task.n_units;
#if HM_DEVICE_CHECKS
            if (!end && (task.first_unit < 0 || nch < 1 || task.first_unit + nch > A.n_units)) {
                if (lane == 0)
                    printf("hm device check failed: task %llu units [%lld, +%d) of %lld\n", t, (long long)task.first_unit,
                           nch, (long long)A.n_units);
                __trap();
            }
#endif
            for (int base = 0; base < nch; base += 32) {
                long long c0 = clock64();
                Unit mine{};
                if (!end && base + lane < nch) mine = A.units[task.first_unit + base + lane];
                __syncwarp();
                st_m += clock64() - c0;
                const int cnt = min(32, nch - base);
                for (int c = 0; c < cnt; ++c, ++k) {
                    const int s = (int)(k % kMStages);
                    c0 = clock64();
                    if (k >= kMStages && lane == 0) mbar_wait(&S.empty[s], (uint32_t)(((k / kMStages) - 1) & 1));
                    __syncwarp();
                    st_e += clock64() - c0;
                    MStage& St = S.st[s];
                    const int utype = __shfl_sync(0xffffffffu, mine.type, c);
                    const int uncols = __shfl_sync(0xffffffffu, mine.ncols, c);
                    const int uld = __shfl_sync(0xffffffffu, mine.ld, c);
                    const int upass = __shfl_sync(0xffffffffu, mine.pass, c);
                    const long long uoff = __shfl_sync(0xffffffffu, (long long)mine.a_off, c);
                    // payload route (whole_chunk): one bulk copy of the chunk (default); else column by
                    // column at padded_ld(ld), one bulk copy per column issued lane by lane.  (Measured and
                    // removed: 16-byte cp.async from every lane for the padded chunks, 0.846 vs 0.796 ms.)
                    const bool stream = !end && utype == UNIT_STREAM;
#if HM_DEVICE_CHECKS
                    if (stream) check_payload(A, upass, uoff, uncols, uld);
#endif
                    const bool whole = stream && whole_chunk(uld);
                    if (lane == c) {
                        if (end) {
                            St.hdr.type = -1;
                            mbar_arrive(&S.posted[s]);
                            mbar_arrive(&S.full[s]);
                        } else {
                            St.hdr = mine;
                            mbar_arrive(&S.posted[s]);
                            if (stream)
                                mbar_expect_tx(&S.full[s], (uint32_t)mine.ncols * (uint32_t)mine.ld * 8u);
                            else if (!stream)
                                mbar_arrive(&S.full[s]);
                        }
                    }
                    __syncwarp();
                    if (whole) {   // one copy of the whole chunk
                        if (lane == 0) {
                            const double* src = S.passes[upass].arena + uoff;
                            const uint32_t pb = (uint32_t)uncols * (uint32_t)uld * 8u;
                            if (HM_PAYLOAD_EVICT_FIRST)
                                tma_load_1d_hint(St.payload, src, pb, &S.full[s], pol);
                            else
                                tma_load_1d(St.payload, src, pb, &S.full[s]);
                        }
                    } else if (stream) {   // column j -> payload + j * padded_ld(ld)
                        const double* src = S.passes[upass].arena + uoff;
                        const int ldp = padded_ld(uld);
                        for (int j = lane; j < uncols; j += 32) {
                            if (HM_PAYLOAD_EVICT_FIRST)
                                tma_load_1d_hint(St.payload + j * ldp, src + (int64_t)j * uld, (uint32_t)uld * 8u,
                                                 &S.full[s], pol);
                            else
                                tma_load_1d(St.payload + j * ldp, src + (int64_t)j * uld, (uint32_t)uld * 8u, &S.full[s]);
                        }
                    }
                }
                nxt = __shfl_sync(0xffffffffu, nxt, 0);
            }
            if (end) break;
            if (ew) {   // wait until the unit's (last) stage is released, then take the next task
                const int64_t kl = k - 1;
                if (lane == 0) {
                    mbar_wait(&S.empty[(int)(kl % kMStages)], (uint32_t)((kl / kMStages) & 1));
                    nxt = atomicAdd(A.queue, 1ull) - queue_base;
                }
                nxt = __shfl_sync(0xffffffffu, nxt, 0);
            }
        }
        if (A.stats && lane == 0) {
            atomicAdd(A.stats + 0, st_e);
            atomicAdd(A.stats + 1, st_m);
            atomicAdd(A.stats + 12, (unsigned long long)(clock64() - t0));
        }
        return;
    }
    if (warp <= kMGatherers) {
        // ------------------------------------------------ gatherers (both warps on every stage,
        // columns split between them): dependency waits, then the X rows of the chunk
        const int gw = warp - 1;
        int64_t verified = -1;
        unsigned long long st_p = 0, st_d = 0, st_g = 0;
        for (int64_t k = 0;; ++k) {
            const int s = (int)(k % kMStages);
            long long c0 = clock64();
            mbar_wait(&S.posted[s], (uint32_t)((k / kMStages) & 1));
            long long c1 = clock64();
            st_p += c1 - c0;
            MStage& St = S.st[s];
            const Unit& H = St.hdr;
            const int type = H.type;
            if (type >= 0 && H.task != verified) {
                if (lane == 0) {
                    if (H.wait_id[0] >= 0) wait_counter(A, epoch, H.wait_id[0], H.wait_cnt[0]);
                    if (H.wait_id[1] >= 0) wait_counter(A, epoch, H.wait_id[1], H.wait_cnt[1]);
                    if (A.trace && H.chunk == 0) atomicMin(A.trace + 2 * H.pass, gtimer());
                }
                __syncwarp();
                fence_proxy_async_global();
                verified = H.task;
            }
            c0 = clock64();
            st_d += c0 - c1;
#if HM_DEVICE_CHECKS
            if (type == UNIT_STREAM && gw == 0)
                check_chunk(A, H, S.passes[H.pass < A.n_passes ? H.pass : 0], kMrhsMaxCols, kMrhsPayloadDoubles, lane);
#endif
            if (type == UNIT_STREAM) {
                const Pass& P = S.passes[H.pass];
                const double* in = P.in;
                const int ncols = H.ncols;
                const int im = P.in_mode;
                const int32_t* cs = P.colsrc + H.cs_off;   // colsrc_ext for fused-prologue passes
                const int ncol4 = (ncols + 3) & ~3;
                if (im == IN_PLAIN && HM_MRHS_GATHER_LDG) {
                    // X rows (512 B each, written by an earlier pass: L2) by coalesced 16-byte loads, 16
                    // rows in flight per warp (HM_MRHS_GATHER_LDG=1 at build time).  Off: although the
                    // per-row TMA issue serialises over the lanes (8 % of the kernel's stall samples),
                    // the register path measured slower (C2 64-RHS flux 1.180 vs 0.913 ms): the gather
                    // warps then wait out the L2 latency themselves instead of moving on
                    for (int c0 = gw; c0 < ncol4; c0 += 16 * kMGatherers) {
                        double2 v[16];
#pragma unroll
                        for (int u = 0; u < 16; ++u) {
                            const int c = c0 + u * kMGatherers;
                            v[u] = make_double2(0.0, 0.0);
                            if (c < ncols)
                                v[u] = __ldcg(reinterpret_cast<const double2*>(in + (int64_t)__ldg(cs + c) * kMrhsMax) + lane);
                        }
#pragma unroll
                        for (int u = 0; u < 16; ++u) {
                            const int c = c0 + u * kMGatherers;
                            if (c < ncol4) reinterpret_cast<double2*>(St.X + c * kXStride)[lane] = v[u];
                        }
                    }
                } else if (im == IN_PLAIN) {
                    // each X row (512 B, written by an earlier pass) arrives by a 1-D TMA bulk copy:
                    // warp gw, lane l -> column c = gw + kMGatherers * l
                    const int c = gw + kMGatherers * lane;
                    const int mine = c < ncols ? 1 : 0;
                    const int cnt = __popc(__ballot_sync(0xffffffffu, mine));
                    if (lane == 0 && cnt) mbar_add_tx(&S.gathered[s], (uint32_t)cnt * kMrhsMax * 8u);
                    __syncwarp();
                    if (mine) {
                        const int32_t j = __ldg(cs + c);
                        if (HM_MRHS_T_HINT >= 2)
                            tma_load_1d_hint(St.X + c * kXStride, in + (int64_t)j * kMrhsMax, kMrhsMax * 8u, &S.gathered[s],
                                             l2_evict_last_policy());
                        else
                            tma_load_1d(St.X + c * kXStride, in + (int64_t)j * kMrhsMax, kMrhsMax * 8u, &S.gathered[s]);
                    } else if (c < ncol4) {   // k-step padding columns: zero (consumers multiply them)
#pragma unroll
                        for (int q = 0; q < kMrhsMax; ++q) St.X[c * kXStride + q] = 0.0;
                    }
                } else {
                    // fused prologue: rows of the caller's external-order array (stride ld), IN_FLUX:
                    // w = eps T^4; 8 columns in flight per warp, lanes cover the 64 values as double2
                    const int q = 2 * lane;
                    for (int c0 = gw; c0 < ncol4; c0 += 8 * kMGatherers) {
                        double2 v[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const int c = c0 + u * kMGatherers;
                            v[u] = make_double2(0.0, 0.0);
                            if (c < ncols) {
                                const int32_t j = __ldg(cs + c);
                                if (j >= 0) {
                                    v[u] = __ldcg(reinterpret_cast<const double2*>(in + (int64_t)j * kMrhsMax) + lane);
                                } else {
                                    const int64_t e = -(int64_t)j - 1;
                                    const double* src = A.user_in + e * A.ld;
                                    v[u].x = q < R ? __ldg(src + q) : 0.0;
                                    v[u].y = q + 1 < R ? __ldg(src + q + 1) : 0.0;
                                    if (im == IN_FLUX) {
                                        const double ee = __ldg(A.eps_ext + e);
                                        v[u].x = ee * pow4(v[u].x);
                                        v[u].y = ee * pow4(v[u].y);
                                    }
                                }
                                if (q >= R) v[u].x = 0.0;
                                if (q + 1 >= R) v[u].y = 0.0;
                            }
                        }
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const int c = c0 + u * kMGatherers;
                            if (c < ncol4) reinterpret_cast<double2*>(St.X + c * kXStride)[lane] = v[u];
                        }
                    }
                }
            }
            __syncwarp();
            st_g += clock64() - c0;
            if (lane == 0) mbar_arrive(&S.gathered[s]);
            if (type < 0) break;
        }
        if (A.stats && lane == 0) {
            atomicAdd(A.stats + 3, st_p);
            atomicAdd(A.stats + 4, st_d);
            atomicAdd(A.stats + 5, st_g);
        }
        return;
    }
    if (warp == kMPubWarp) {
        // ------------------------------------------------ publisher: per finished task, make its outputs
        // (written by the consumers before their mbarrier arrival) visible GPU-wide, then move the
        // dependency counters -- off the consumers' critical path
        unsigned long long st_pw = 0;
        for (int64_t j = 0;; ++j) {
            const int r = (int)(j % kPubSlots);
            const long long c0 = clock64();
            mbar_wait(&S.pfull[r], (uint32_t)((j / kPubSlots) & 1));
            st_pw += clock64() - c0;
            const PubDesc d = S.pub[r];
            if (d.type < 0) break;
            if (lane == 0) {
                __threadfence();
                if (A.trace) atomicMax(A.trace + 2 * d.pass + 1, gtimer());
                atomicAdd(A.done + d.pass, 1ull);
                if (d.inc0 >= 0) atomicAdd(A.done + d.inc0, 1ull);
                if (d.inc1 >= 0) atomicAdd(A.done + d.inc1, 1ull);
                mbar_arrive(&S.pempty[r]);
            }
            __syncwarp();
        }
        if (A.stats && lane == 0) atomicAdd(A.stats + 9, st_pw);
        return;
    }
    // ---------------------------------------------------- consumers: DMMA, task accumulators in registers
    const int cw = warp - 1 - kMGatherers;   // consumer warp 0..7
    const int ct = tid - kMConsumer0;
    double acc[kMaxTiles][2];
#pragma unroll
    for (int i = 0; i < kMaxTiles; ++i) acc[i][0] = acc[i][1] = 0.0;
    const int ar = lane >> 2, ak = lane & 3;     // fragment coordinates
    unsigned long long st_wg = 0, st_wf = 0, st_c = 0, st_t = 0;
    int64_t ntask = 0;     // tasks handed to the publisher
    // task-end handoff: every consumer warp waits for the slot's previous use to be published, warp 0
    // lane 0 writes the descriptor, every warp arrives after its own output stores
    auto hand_off = [&](int type, int pass, int32_t inc0, int32_t inc1) {
        const int r = (int)(ntask % kPubSlots);
        if (lane == 0 && ntask >= kPubSlots) mbar_wait(&S.pempty[r], (uint32_t)(((ntask / kPubSlots) - 1) & 1));
        if (ct == 0) S.pub[r] = PubDesc{type, pass, inc0, inc1};
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.pfull[r]);
        ++ntask;
    };
    long long c0 = clock64();
    for (int64_t k = 0;; ++k) {
        const int s = (int)(k % kMStages);
        mbar_wait(&S.gathered[s], (uint32_t)((k / kMStages) & 1));
        long long c1 = clock64();
        st_wg += c1 - c0;
        MStage& St = S.st[s];
        const int type = St.hdr.type;
        if (type < 0) {
            hand_off(-1, 0, -1, -1);
            break;
        }
        mbar_wait(&S.full[s], (uint32_t)((k / kMStages) & 1));
        long long c2 = clock64();
        st_wf += c2 - c1;
        const int pass = St.hdr.pass, nrows = St.hdr.nrows, ld = St.hdr.ld, ncols = St.hdr.ncols;
        const int chunk = St.hdr.chunk, nchunks = St.hdr.nchunks;
        const int grp = St.hdr.grp, nseg = St.hdr.nseg, seg = St.hdr.seg;
        const int64_t out0 = St.hdr.out0, part_off = St.hdr.part_off;
        const int32_t inc0 = St.hdr.inc_id[0], inc1 = St.hdr.inc_id[1];
        const Pass& P = S.passes[pass];
        const int M8 = (nrows + 7) >> 3;
        const int ntile = M8 * N8;
        if (type == UNIT_STREAM) {
            if (chunk == 0) {
#pragma unroll
                for (int i = 0; i < kMaxTiles; ++i) acc[i][0] = acc[i][1] = 0.0;
            }
            const double* Ap = St.payload;
            const double* Xp = St.X;
            const int ldp = smem_ld(ld);
            // this warp's tiles t = cw + 8 i (row tiles mt, column tile nt); the k loop is
            // specialised on the tile count so the fragments of a k-step are loaded as a batch into
            // distinct registers and then feed back-to-back DMMAs
            if (use_1d(M8, N8)) {
                switch (M8) {
                    case 1: mma_chunk1d<1>(acc, Ap, Xp, ldp, ncols, cw, ar, ak); break;
                    case 3: mma_chunk1d<3>(acc, Ap, Xp, ldp, ncols, cw, ar, ak); break;
                    case 5: mma_chunk1d<5>(acc, Ap, Xp, ldp, ncols, cw, ar, ak); break;
                    case 7: mma_chunk1d<7>(acc, Ap, Xp, ldp, ncols, cw, ar, ak); break;
                    default: break;
                }
            } else if (N8 == 8) {
                switch ((M8 - (cw >> 2) + 1) >> 1) {   // this warp's row tiles
#define HM_MMA2_CASE(RM) \
    case RM: mma_chunk2d<RM>(acc, Ap, Xp, ldp, ncols, cw, ar, ak); break;
                    HM_MMA2_CASE(1) HM_MMA2_CASE(2) HM_MMA2_CASE(3) HM_MMA2_CASE(4)
                    HM_MMA2_CASE(5) HM_MMA2_CASE(6) HM_MMA2_CASE(7) HM_MMA2_CASE(8)
#undef HM_MMA2_CASE
                    default: break;
                }
            } else {
            int nmine = 0;
#pragma unroll
            for (int i = 0; i < kMaxTiles; ++i)
                if (cw + 8 * i < ntile) nmine = i + 1;
            switch (nmine) {
#define HM_MMA_CASE(TM) \
    case TM: mma_chunk<TM>(acc, Ap, Xp, ldp, ncols, cw, N8, ar, ak); break;
                HM_MMA_CASE(1) HM_MMA_CASE(2) HM_MMA_CASE(3) HM_MMA_CASE(4)
                HM_MMA_CASE(5) HM_MMA_CASE(6) HM_MMA_CASE(7) HM_MMA_CASE(8)
                HM_MMA_CASE(9) HM_MMA_CASE(10) HM_MMA_CASE(11) HM_MMA_CASE(12)
                HM_MMA_CASE(13) HM_MMA_CASE(14) HM_MMA_CASE(15) HM_MMA_CASE(16)
#undef HM_MMA_CASE
                default: break;
            }
            }
        } else if (type == UNIT_EPILOGUE) {
            // rows x R of the internal result through the pass's output mode: warp cw takes rows
            // cw, cw + 8, ..., kERows of them in flight; lane l covers columns 2l, 2l + 1 (the internal
            // 64-wide row as one 16-byte load per lane).  The per-row scalars (perm, eps, A, g) are loaded
            // for all kERows rows first, so the dependent loads of T's row e = perm[row] are in flight
            // together (the unit is latency-bound: one round trip per batch, not per row)
            if (P.mode == OUT_PERM || P.mode == OUT_FLUX) {
                const bool flux = P.mode == OUT_FLUX;
                constexpr int kERows = HM_MRHS_EROWS;
                const int c2 = 2 * lane;
                for (int r0 = cw; r0 < nrows; r0 += kERows * kMConsumerWarps) {
                    int64_t e[kERows];
                    double sc[kERows], gg[kERows], am[kERows];
#pragma unroll
                    for (int u = 0; u < kERows; ++u) {
                        const int r = r0 + u * kMConsumerWarps;
                        const int64_t row = out0 + (r < nrows ? r : 0);
                        e[u] = __ldg(A.perm + row);
                        sc[u] = flux ? A.sigma * (__ldg(A.eps_int + row) / __ldg(A.area_int + row)) : 0.0;
                        gg[u] = flux ? __ldg(A.g_int + row) : 0.0;
                        am[u] = flux && A.amb ? __ldg(A.amb + row) : 0.0;
                    }
                    double2 v[kERows];
                    double t0[kERows], t1[kERows];
#pragma unroll
                    for (int u = 0; u < kERows; ++u) {
                        const int r = r0 + u * kMConsumerWarps;
                        const bool ok = r < nrows && c2 < R;
                        v[u] = ok ? __ldcg(reinterpret_cast<const double2*>(P.in + (out0 + r) * kMrhsMax + c2))
                                  : make_double2(0.0, 0.0);
                        t0[u] = ok && flux ? __ldg(A.user_in + e[u] * A.ld + c2) : 0.0;
                        t1[u] = ok && flux && c2 + 1 < R ? __ldg(A.user_in + e[u] * A.ld + c2 + 1) : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < kERows; ++u) {
                        const int r = r0 + u * kMConsumerWarps;
                        if (r >= nrows || c2 >= R) continue;
                        double* dst = A.user_out + e[u] * A.ld + c2;
                        if (flux) {
                            const double h0 = pow4(t0[u]), h1 = pow4(t1[u]);
                            dst[0] = sc[u] * (v[u].x - h0 * gg[u] + am[u] * (h0 - A.t_inf4));
                            if (c2 + 1 < R) dst[1] = sc[u] * (v[u].y - h1 * gg[u] + am[u] * (h1 - A.t_inf4));
                        } else {
                            dst[0] = v[u].x;
                            if (c2 + 1 < R) dst[1] = v[u].y;
                        }
                    }
                }
            } else {   // other modes (sharded): element by element, 4 in flight
                const int tot = nrows * R;
                for (int e0 = ct; e0 < tot; e0 += 4 * kMConsumers) {
                    double v[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int e = e0 + u * kMConsumers;
                        v[u] = e < tot ? __ldcg(P.in + (out0 + e / R) * kMrhsMax + (e % R)) : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int e = e0 + u * kMConsumers;
                        if (e < tot) emit_m(A, P, out0 + e / R, e % R, v[u]);
                    }
                }
            }
        } else if (type == UNIT_PROLOGUE_INT) {
            // sharded flux prologue: w = eps T^4 over padded rows, from the gathered T block
            const int tot = nrows * R;
            for (int e = ct; e < tot; e += kMConsumers) {
                const int64_t row = out0 + e / R;
                const int col = e % R;
                P.out[row * kMrhsMax + col] = __ldg(A.eps_int + row) * pow4(__ldcg(P.in + row * kMrhsMax + col));
            }
        } else {
            // element-wise prologue: rows x R of the caller's external-order array permuted into the
            // internal n x 64 layout (UNIT_PROLOGUE: w = eps T^4); as the epilogue: perm and eps for
            // kPRows rows first, then their T rows in flight together, lane l -> columns 2l, 2l + 1
            // (one 16-byte store per lane into the internal row)
            constexpr int kPRows = HM_MRHS_EROWS;
            const int c2 = 2 * lane;
            for (int r0 = cw; r0 < nrows; r0 += kPRows * kMConsumerWarps) {
                int64_t e[kPRows];
                double ep[kPRows];
#pragma unroll
                for (int u = 0; u < kPRows; ++u) {
                    const int r = r0 + u * kMConsumerWarps;
                    const int64_t row = out0 + (r < nrows ? r : 0);
                    e[u] = __ldg(A.perm + row);
                    ep[u] = type == UNIT_PROLOGUE ? __ldg(A.eps_int + row) : 1.0;
                }
                double t0[kPRows], t1[kPRows];
#pragma unroll
                for (int u = 0; u < kPRows; ++u) {
                    const int r = r0 + u * kMConsumerWarps;
                    const bool ok = r < nrows && c2 < R;
                    t0[u] = ok ? __ldg(A.user_in + e[u] * A.ld + c2) : 0.0;
                    t1[u] = ok && c2 + 1 < R ? __ldg(A.user_in + e[u] * A.ld + c2 + 1) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < kPRows; ++u) {
                    const int r = r0 + u * kMConsumerWarps;
                    if (r >= nrows || c2 >= R) continue;
                    const double2 w = type == UNIT_PROLOGUE ? make_double2(ep[u] * pow4(t0[u]), ep[u] * pow4(t1[u]))
                                                            : make_double2(t0[u], t1[u]);
                    *reinterpret_cast<double2*>(P.out + (out0 + r) * kMrhsMax + c2) = w;
                }
            }
            // the rest of the 64-wide rows stays zero-free of stale values: columns R..63 are never read
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.empty[s]);
        c0 = clock64();
        st_c += c0 - c2;
        if (chunk != nchunks - 1) continue;
        // ---- last chunk of the task: emit (split panels combine deterministically), publish
        if (type == UNIT_STREAM) {
            if (grp < 0 && P.mode == OUT_ASSIGN) {
                // internal n x 64 result (t or y): one 16-byte store per fragment pair (columns past R
                // hold values of the zero-free padding columns and are never read)
#pragma unroll
                for (int i = 0; i < kMaxTiles; ++i) {
                    int mt, nt;
                    if (!warp_tile(i, cw, M8, N8, mt, nt)) break;
                    const int row = mt * 8 + ar;
                    const int col = nt * 8 + 2 * ak;
                    if (row < nrows) {
                        if (HM_MRHS_T_HINT >= 1)
                            st_v2_hint(P.out + (out0 + row) * kMrhsMax + col, acc[i][0], acc[i][1], l2_evict_last_policy());
                        else
                            *reinterpret_cast<double2*>(P.out + (out0 + row) * kMrhsMax + col) = make_double2(acc[i][0], acc[i][1]);
                    }
                }
            } else if (grp < 0) {
#pragma unroll
                for (int i = 0; i < kMaxTiles; ++i) {
                    int mt, nt;
                    if (!warp_tile(i, cw, M8, N8, mt, nt)) break;
                    const int row = mt * 8 + ar;
                    const int col = nt * 8 + 2 * ak;
                    if (row < nrows) {
                        if (col < R) emit_m(A, P, out0 + row, col, acc[i][0]);
                        if (col + 1 < R) emit_m(A, P, out0 + row, col + 1, acc[i][1]);
                    }
                }
            } else {
                double* part = P.part + part_off;
#pragma unroll
                for (int i = 0; i < kMaxTiles; ++i) {
                    int mt, nt;
                    if (!warp_tile(i, cw, M8, N8, mt, nt)) break;
                    const int row = mt * 8 + ar;
                    const int col = nt * 8 + 2 * ak;
                    if (row < nrows) {
                        part[row * kMrhsMax + col] = acc[i][0];
                        part[row * kMrhsMax + col + 1] = acc[i][1];
                    }
                }
                cons_sync();
                if (ct == 0) {
                    __threadfence();
                    S.last = (atomicAdd(P.counters + grp, 1) == nseg - 1);
                    if (S.last) __threadfence();
                }
                cons_sync();
                if (S.last) {
                    const int64_t pstride = (int64_t)ld * kMrhsMax;   // piece q's partial: (q - seg) * pstride away
                    const int tot = nrows * R;
                    for (int e0 = ct; e0 < tot; e0 += 4 * kMConsumers) {   // 4 elements in flight
                        double v[4] = {0.0, 0.0, 0.0, 0.0};
                        for (int q = 0; q < nseg; ++q) {
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const int e = e0 + u * kMConsumers;
                                if (e < tot)
                                    v[u] += __ldcg(part + (int64_t)(q - seg) * pstride + (e / R) * kMrhsMax + (e % R));
                            }
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int e = e0 + u * kMConsumers;
                            if (e < tot) emit_m(A, P, out0 + e / R, e % R, v[u]);
                        }
                    }
                    if (ct == 0) P.counters[grp] = 0;
                }
            }
        }
        hand_off(type, pass, inc0, inc1);
        const long long c3 = clock64();
        st_t += c3 - c0;
        c0 = c3;
    }
    if (A.stats && ct == 0) {
        atomicAdd(A.stats + 6, st_wg);
        atomicAdd(A.stats + 13, st_wf);
        atomicAdd(A.stats + 7, st_c);
        atomicAdd(A.stats + 8, st_t);
    }
}

}  // namespace

static size_t mrhs_smem_bytes() { return sizeof(MSmem) + 128; }

static void mrhs_set_attr() {
    static bool attr = false;
    if (!attr) {
        HM_CUDA(cudaFuncSetAttribute(engine_mrhs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)mrhs_smem_bytes()));
        attr = true;
    }
}

void engine_mrhs_launch(const ProgArgs& A, int grid, cudaStream_t s) {
    mrhs_set_attr();
    void* args[] = {const_cast<ProgArgs*>(&A)};
    HM_CUDA(cudaLaunchCooperativeKernel((const void*)engine_mrhs_kernel, dim3(grid), dim3(kMThreads), args,
                                        mrhs_smem_bytes(), s));
    debug_sync(s, "engine_mrhs_kernel");
}

int engine_mrhs_max_passes() { return kMaxPassesM; }

int engine_mrhs_grid() {
    int dev = 0, sms = 0, per = 0;
    HM_CUDA(cudaGetDevice(&dev));
    HM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    mrhs_set_attr();
    HM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, engine_mrhs_kernel, kMThreads, mrhs_smem_bytes()));
    if (per < 1) throw Error(HM_ERR_CUDA, "multi-RHS engine kernel does not fit on an SM");
    return sms * per;
}

}  // namespace hm
