// FP64 throughput micro-benchmark: DMMA (mma.sync.m8n8k4.f64) and DFMA from registers, 148 x k CTAs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/ubench_fp64 scripts/ubench_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void dmma_loop(double* out, int iters) {
    double c[CH][2];
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
#pragma unroll
    for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
    if (s == 1.2345) out[0] = s;
}

template <int CH>
__global__ void dfma_loop(double* out, int iters) {
    double c[CH];
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
#pragma unroll
    for (int i = 0; i < CH; ++i) c[i] = i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) c[i] = fma(a, b, c[i]);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s += c[i];
    if (s == 1.2345) out[0] = s;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int warps : {4, 8, 16, 32}) {
        auto run = [&](auto kern, double flop_per_inst_warp, const char* name, int ch) {
            kern<<<sms, 32 * warps>>>(out, 10);
            cudaDeviceSynchronize();
            cudaEventRecord(e0);
            kern<<<sms, 32 * warps>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double fl = (double)sms * warps * iters * ch * flop_per_inst_warp;
            printf("%s warps/SM %2d chains %d: %.2f TFLOP/s\n", name, warps, ch, fl / (ms * 1e-3) / 1e12);
        };
        run(dmma_loop<4>, 2.0 * 8 * 8 * 4, "DMMA", 4);
        run(dmma_loop<8>, 2.0 * 8 * 8 * 4, "DMMA", 8);
        run(dfma_loop<8>, 2.0 * 32, "DFMA", 8);
    }
    return 0;
}
