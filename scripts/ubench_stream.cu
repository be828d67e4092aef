// Streaming micro-benchmark for the hot-path design (not part of the library):
//   1. LDG.128 grid-stride read (the HBM read ceiling)
//   2. 1-D TMA bulk ring, one CTA per SM, S stages x B bytes, trivial consumer
//   3. same ring with CTAs/SM > 1
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench scripts/ubench_stream.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__global__ void ldg_read(const double2* __restrict__ a, size_t n2, double* out) {
    double s = 0;
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t st = (size_t)gridDim.x * blockDim.x;
    for (; i + 3 * st < n2; i += 4 * st) {
        double2 v0 = __ldcs(a + i), v1 = __ldcs(a + i + st), v2 = __ldcs(a + i + 2 * st), v3 = __ldcs(a + i + 3 * st);
        s += v0.x + v0.y + v1.x + v1.y + v2.x + v2.y + v3.x + v3.y;
    }
    for (; i < n2; i += st) { double2 v = a[i]; s += v.x + v.y; }
    if (s == 123.456) out[0] = s;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, uint32_t parity) {
    asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, unsigned long long* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory");
}

// ring: warp 0 lane 0 issues TMA of chunks blockIdx.x, blockIdx.x + grid, ...; warps 1..C consume
template <int CW>
__global__ void tma_ring(const char* __restrict__ a, int64_t nchunks, int chunk, int stages, double* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    unsigned long long* full = (unsigned long long*)sm;
    unsigned long long* empty = full + 32;
    char* buf = (char*)(sm + 1024);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, CW); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 0) {
        if (lane == 0) {
            int64_t k = 0;
            for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++k) {
                const int s = (int)(k % stages);
                if (k >= stages) mbar_wait(empty + s, (uint32_t)(((k / stages) - 1) & 1));
                mbar_expect_tx(full + s, chunk);
                tma_load_1d(buf + (size_t)s * chunk, a + c * chunk, chunk, full + s);
            }
        }
        return;
    }
    double acc = 0;
    int64_t k = 0;
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++k) {
        const int s = (int)(k % stages);
        mbar_wait(full + s, (uint32_t)((k / stages) & 1));
        const double2* p = (const double2*)(buf + (size_t)s * chunk);
        for (int i = threadIdx.x - 32; i < chunk / 16; i += 32 * CW) { double2 v = p[i]; acc += v.x + v.y; }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + s);
    }
    if (acc == 123.456) out[0] = acc;
}

// ring with (a) chunk byte offset `off` (16-B aligned, not 128-B), (b) permuted chunk order,
// (c) a gather step: after the payload lands the consumer warps first load `ng` x values from an
// L2-resident vector through the indices stored in the chunk's first bytes (like the engine)
__global__ void tma_ring2(const char* __restrict__ a, int64_t nchunks, int chunk, int stages, int off,
                          const int64_t* __restrict__ order, const double* __restrict__ xv, int ng, double* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    unsigned long long* full = (unsigned long long*)sm;
    unsigned long long* empty = full + 32;
    char* buf = (char*)(sm + 1024);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int CW = (blockDim.x >> 5) - 1;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, CW); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 0) {
        if (lane == 0) {
            int64_t k = 0;
            for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++k) {
                const int s = (int)(k % stages);
                if (k >= stages) mbar_wait(empty + s, (uint32_t)(((k / stages) - 1) & 1));
                mbar_expect_tx(full + s, chunk);
                const int64_t cc = order ? order[c] : c;
                tma_load_1d(buf + (size_t)s * chunk, a + cc * (chunk + off), chunk, full + s);
            }
        }
        return;
    }
    double acc = 0;
    int64_t k = 0;
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++k) {
        const int s = (int)(k % stages);
        mbar_wait(full + s, (uint32_t)((k / stages) & 1));
        const double2* p = (const double2*)(buf + (size_t)s * chunk);
        if (ng) {
            const int* idx = (const int*)p;
            for (int i = threadIdx.x - 32; i < ng; i += 32 * CW) acc += __ldcg(xv + (idx[i] & 262143));
        }
        for (int i = threadIdx.x - 32; i < chunk / 16; i += 32 * CW) { double2 v = p[i]; acc += v.x + v.y; }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + s);
    }
    if (acc == 123.456) out[0] = acc;
}

int main() {
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t bytes = size_t(1) << 31;  // 2 GiB
    char* a;
    double* out;
    CK(cudaMalloc(&a, bytes));
    CK(cudaMalloc(&out, 8));
    CK(cudaMemset(a, 0, bytes));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](auto fn) {
        fn();
        CK(cudaDeviceSynchronize());
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            fn();
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        return bytes / (best * 1e-3) / 1e9;
    };
    for (int per : {2, 4, 8, 16}) {
        double gbs = timeit([&] { ldg_read<<<sms * per, 512>>>((const double2*)a, bytes / 16, out); });
        printf("ldg_read grid %d x 512: %.0f GB/s\n", sms * per, gbs);
    }
    for (int chunk : {16384, 32768}) {
        for (int stages : {2, 4, 6, 8, 12}) {
            const size_t sm = 1024 + (size_t)stages * chunk;
            if (sm > 227 * 1024) continue;
            for (int ctas : {1, 2}) {
                if (sm * ctas > 228 * 1024) continue;
                CK(cudaFuncSetAttribute(tma_ring<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
                const int64_t nch = bytes / chunk;
                double gbs = timeit([&] { tma_ring<4><<<sms * ctas, 160, sm>>>(a, nch, chunk, stages, out); });
                printf("tma_ring chunk %6d stages %2d ctas/SM %d (in flight/SM %4zu KB): %.0f GB/s\n", chunk, stages, ctas,
                       (size_t)stages * chunk * ctas / 1024, gbs);
            }
        }
    }
    {
        const int chunk = 32768;
        const int64_t nch = bytes / (chunk + 16) - 1;
        std::vector<int64_t> h(nch);
        for (int64_t i = 0; i < nch; ++i) h[i] = i;
        uint64_t z = 12345;
        for (int64_t i = nch - 1; i > 0; --i) { z = z * 6364136223846793005ull + 1442695040888963407ull; int64_t j = (int64_t)((z >> 33) % (uint64_t)(i + 1)); std::swap(h[i], h[j]); }
        int64_t* ord;
        double* xv;
        CK(cudaMalloc(&ord, nch * 8));
        CK(cudaMalloc(&xv, 262144 * 8));
        CK(cudaMemset(xv, 0, 262144 * 8));
        CK(cudaMemcpy(ord, h.data(), nch * 8, cudaMemcpyHostToDevice));
        for (int stages : {4}) {
            const size_t sm = 1024 + (size_t)stages * chunk;
            CK(cudaFuncSetAttribute(tma_ring2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            for (int off : {0, 16}) for (int rnd : {0, 1}) for (int ng : {0, 128, 512}) for (int cw : {4, 8}) {
                double gbs = timeit([&] { tma_ring2<<<sms, 32 * (cw + 1), sm>>>(a, nch, chunk, stages, off, rnd ? ord : nullptr, xv, ng, out); });
                printf("tma_ring2 chunk 32K stages %d off %2d random %d gather %3d consumer warps %d: %.0f GB/s\n", stages, off, rnd, ng, cw, gbs * (double)nch * chunk / bytes);
            }
        }
    }
    return 0;
}
