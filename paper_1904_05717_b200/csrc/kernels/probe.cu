// FP64 tensor-pipe (DMMA) issue-rate probe: the roofline denominator for the
// FP64 GEMM, measured on the device the bench runs on (MEASURED_PEAKS.json
// carries no FP64 figure). 8 independent m8n8k4 chains per warp, 2 CTAs of
// 256 threads per SM; reports 2*256 flop per mma per warp.
#include <cstdint>

#include "gpu.hpp"

namespace mmm {
namespace gpu {
namespace {

__global__ void __launch_bounds__(256) k_dmma_peak(double* sink, int iters) {
    double acc[8][2];
    const double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c][0] = acc[c][1] = c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(acc[c][0]), "+d"(acc[c][1])
                         : "d"(a), "d"(b));
    }
    double t = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) t += acc[c][0] + acc[c][1];
    if (t == -1.2345) sink[threadIdx.x] = t;
}

}  // namespace

cudaError_t measure_fp64_peak(int launches, double* tflops) {
    int dev = 0, sms = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* sink = nullptr;
    if ((e = cudaMalloc(&sink, 256 * sizeof(double))) != cudaSuccess) return e;
    const int grid = sms * 2, iters = 5000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_dmma_peak<<<grid, 256>>>(sink, iters);  // warm
    cudaEventRecord(e0);
    for (int i = 0; i < launches; ++i) k_dmma_peak<<<grid, 256>>>(sink, iters);
    cudaEventRecord(e1);
    e = cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    *tflops = 2.0 * 256.0 * 8.0 * iters * (double)grid * 8.0 * launches / (ms * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace gpu
}  // namespace mmm
