// Device helpers shared by the stream engines (kernels_engine.cu, kernels_mrhs.cu): mbarriers, 1-D
// TMA bulk copies, release/acquire counters.
#pragma once

#include <cstdint>

#include "hm_internal.h"

#ifndef HM_PAYLOAD_EVICT_FIRST
#define HM_PAYLOAD_EVICT_FIRST 1
#endif
// debug builds (HM_BUILD_DEFINES="HM_DEVICE_CHECKS=1"): every chunk descriptor and every gathered index
// is checked on the device against the program's bounds (compute-sanitizer is not available on the
// GPU pool); a violation prints the chunk and traps, and the call fails with HM_ERR_CUDA
#ifndef HM_DEVICE_CHECKS
#define HM_DEVICE_CHECKS 0
#endif

namespace hm {
namespace dev {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// expect `bytes` more transaction bytes in the current phase without arriving
__device__ __forceinline__ void mbar_add_tx(unsigned long long* b, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
// order this thread's generic-proxy view of global memory (acquired data) before its async-proxy
// (TMA) reads of it
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
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
__device__ __forceinline__ bool mbar_test(unsigned long long* b, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred P1;\nmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(ok) : "r"(smem_u32(b)), "r"(parity) : "memory");
    return ok != 0;
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, unsigned long long* b) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(b))
        : "memory");
}
// The factor payload is read once per apply and is larger than L2: stream it with an L2 evict-first
// policy so that the lines worth keeping (inputs, the phase-1 -> phase-2 scratch) stay resident
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// The multi-RHS phase-1 -> phase-2 scratch t (n_t x 64) is re-read by every leaf-row slice of its block:
// an L2 evict-last policy for its stores (and gathers) keeps it resident against the streamed payload
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void st_v2_hint(double* p, double a, double b, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(a), "d"(b), "l"(pol) : "memory");
}
__device__ __forceinline__ void tma_load_1d_hint(void* dst, const void* src, uint32_t bytes, unsigned long long* b,
                                                 uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(b)), "l"(pol)
        : "memory");
}
// split-K arrival: release this thread's (and, cumulatively, its warp's) partial-sum writes,
// acquire the other pieces' when last
__device__ __forceinline__ int atom_add_acq_rel(int* p, int v) {
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
// task publication: outputs visible GPU-wide before the counter moves (pairs with ld.acquire.gpu)
__device__ __forceinline__ void red_release(unsigned long long* p, unsigned long long v) {
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ double pow4(double T) {
    const double t2 = T * T;
    return t2 * t2;
}

// This launch's epoch (program launch number, 1-based) into *out_smem by thread 0 before the CTA
// barrier that follows; the last CTA to start advances the device epoch for the next launch.
__device__ __forceinline__ void read_epoch(const ProgArgs& A, unsigned long long* out_smem) {
    const unsigned long long e = *reinterpret_cast<volatile unsigned long long*>(A.epoch_dev);
    *out_smem = e;
    if (atomicAdd(A.epoch_dev + 1, 1ull) == e * gridDim.x - 1) {   // every CTA of this launch has read e
        *reinterpret_cast<volatile unsigned long long*>(A.epoch_dev) = e + 1;
        __threadfence();
    }
}

__device__ __forceinline__ void wait_counter(const ProgArgs& A, unsigned long long epoch, int id, int cnt) {
    const unsigned long long target = epoch * (unsigned long long)cnt;
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


#if HM_DEVICE_CHECKS
// producer side, before a payload copy: the chunk [a_off, a_off + ncols ld) inside pass `pass`'s arena
static __device__ __forceinline__ void check_payload(const ProgArgs& A, int pass, int64_t a_off, int ncols, int ld) {
    if (pass < 0 || pass >= A.n_passes || a_off < 0 || ncols < 0 || ld < 0 ||
        a_off + (int64_t)ncols * ld > A.chk[3 * pass]) {
        printf("hm device check failed: payload of pass %d at %lld + %d x %d outside its arena\n", pass, (long long)a_off,
               ncols, ld);
        __trap();
    }
}
// One warp: the chunk H of pass P against A.chk (arena doubles, column-source entries, input index
// bound of the pass), its stage limits, and every column source (lane-parallel); trap on a violation
static __device__ __noinline__ void check_chunk(const ProgArgs& A, const Unit& H, const Pass& P, int max_cols,
                                         int64_t max_payload, int lane) {
    int why = 0;
    if (H.pass < 0 || H.pass >= A.n_passes) why = 1;
    const int64_t* b = why ? nullptr : A.chk + 3 * H.pass;
    if (!why && (H.ncols <= 0 || H.ncols > max_cols || H.ld <= 0 || H.ld > 128 || (H.ld & 1) || H.nrows <= 0 ||
                 H.nrows > H.ld || (int64_t)H.ncols * H.ld > max_payload))
        why = 2;
    if (!why && (H.a_off < 0 || H.a_off + (int64_t)H.ncols * H.ld > b[0])) why = 3;
    const bool ext = P.in_mode == IN_PERM || P.in_mode == IN_FLUX;
    if (!why && H.nruns > 0 && !ext) {
        int64_t tot = 0;
        for (int r = 0; r < H.nruns && r < kMaxRuns; ++r) {
            if (H.run_src[r] < 0 || (int64_t)H.run_src[r] + H.run_len[r] > b[2]) why = 4;
            tot += H.run_len[r];
        }
        if (H.nruns > kMaxRuns || tot != H.ncols) why = 4;
    }
    if (!why && (!P.colsrc || H.cs_off < 0 || H.cs_off + H.ncols > b[1])) why = 5;
    int bad = why;
    if (!why) {
        for (int c = lane; c < H.ncols; c += 32) {
            const int32_t j = P.colsrc[H.cs_off + c];
            const bool ok = ext ? (j >= 0 ? (int64_t)j < b[2] : -(int64_t)j - 1 < A.n_x) : (j >= 0 && (int64_t)j < b[2]);
            if (!ok) bad = 6;
        }
    }
    bad = __reduce_max_sync(0xffffffffu, (unsigned)bad);
    if (bad) {
        if (lane == 0)
            printf("hm device check %d failed: pass %d (of %d) task %lld chunk %d: a_off %lld ncols %d ld %d nrows %d "
                   "cs_off %lld nruns %d\n",
                   bad, H.pass, A.n_passes, (long long)H.task, H.chunk, (long long)H.a_off, H.ncols, H.ld, H.nrows,
                   (long long)H.cs_off, H.nruns);
        __trap();
    }
}
#endif

}  // namespace dev
}  // namespace hm
