// Device helpers shared by the stream engines (kernels_engine.cu, kernels_mrhs.cu): mbarriers, 1-D
// TMA bulk copies, release/acquire counters.
#pragma once

#include <cstdint>

#include "hm_internal.h"

#ifndef HM_PAYLOAD_EVICT_FIRST
#define HM_PAYLOAD_EVICT_FIRST 1
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


}  // namespace dev
}  // namespace hm
