// FP64 peak microbenchmark for sm_100a: DFMA vs DMMA (mma.sync .f64) issue rates,
// plus the device properties the GPU cache hierarchy is built from.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double s) {
    double a[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) a[c] = threadIdx.x * 1e-9 + c;
    const double b = s, d = 1e-12;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) a[c] = fma(a[c], b, d);
    }
    double t = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) t += a[c];
    if (t == 123.456) out[threadIdx.x] = t;
}

// m8n8k4: 256 FMA per warp-instruction
template <int CHAINS>
__global__ void dmma884_kernel(double* out, int iters) {
    double acc[CHAINS][2];
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c][0] = acc[c][1] = c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
    }
    double t = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) t += acc[c][0] + acc[c][1];
    if (t == 123.456) out[threadIdx.x] = t;
}

// m16n8k4: 512 FMA per warp-instruction
template <int CHAINS>
__global__ void dmma1684_kernel(double* out, int iters) {
    double acc[CHAINS][4];
    double a0 = threadIdx.x * 1e-3, a1 = 0.5, b = 1.0 - threadIdx.x * 1e-4;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c][0] = acc[c][1] = acc[c][2] = acc[c][3] = c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c)
            asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                         : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3])
                         : "d"(a0), "d"(a1), "d"(b));
    }
    double t = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) t += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
    if (t == 123.456) out[threadIdx.x] = t;
}

// m16n8k16: 2048 FMA per warp-instruction
template <int CHAINS>
__global__ void dmma16816_kernel(double* out, int iters) {
    double acc[CHAINS][4];
    double a[8], b[4];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
    for (int i = 0; i < 4; ++i) b[i] = 1.0 - threadIdx.x * 1e-4 * i;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c][0] = acc[c][1] = acc[c][2] = acc[c][3] = c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                         : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3])
                         : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                           "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
    double t = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) t += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
    if (t == 123.456) out[threadIdx.x] = t;
}

template <typename F>
static float time_it(F launch, int reps) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    launch();  // warm
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, 0));
    int l2 = 0, smem_optin = 0, smem_sm = 0, clk = 0, memclk = 0, persist = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaDeviceGetAttribute(&memclk, cudaDevAttrMemoryClockRate, 0);
    cudaDeviceGetAttribute(&persist, cudaDevAttrMaxPersistingL2CacheSize, 0);
    printf("{\"name\":\"%s\",\"cc\":\"%d.%d\",\"sms\":%d,\"l2_bytes\":%d,\"persist_l2_max\":%d,\"smem_optin\":%d,\"smem_per_sm\":%d,"
           "\"regs_per_sm\":%d,\"hbm_bytes\":%zu,\"clock_khz\":%d,\"memclk_khz\":%d,\"bus_bits\":%d}\n",
           p.name, p.major, p.minor, p.multiProcessorCount, l2, persist, smem_optin, smem_sm, p.regsPerMultiprocessor,
           p.totalGlobalMem, clk, memclk, p.memoryBusWidth);
    double* out;
    CK(cudaMalloc(&out, 1 << 20));
    const int sms = p.multiProcessorCount;
    const int iters = 20000;
    for (int bpsm : {1, 2, 4}) {
        for (int threads : {128, 256, 512}) {
            if (bpsm * threads > 2048) continue;
            int grid = sms * bpsm;
            float ms = time_it([&] { dfma_kernel<8><<<grid, threads>>>(out, iters, 1.0000001); }, 5);
            double fl = 2.0 * 8 * iters * (double)grid * threads;
            printf("{\"kind\":\"dfma\",\"chains\":8,\"blocks_per_sm\":%d,\"threads\":%d,\"ms\":%.4f,\"tflops\":%.3f}\n",
                   bpsm, threads, ms, fl / ms / 1e9);
        }
    }
    for (int bpsm : {1, 2, 4}) {
        int threads = 256, grid = sms * bpsm;
        float ms = time_it([&] { dfma_kernel<16><<<grid, threads>>>(out, iters, 1.0000001); }, 5);
        double fl = 2.0 * 16 * iters * (double)grid * threads;
        printf("{\"kind\":\"dfma\",\"chains\":16,\"blocks_per_sm\":%d,\"threads\":%d,\"ms\":%.4f,\"tflops\":%.3f}\n",
               bpsm, threads, ms, fl / ms / 1e9);
    }
    for (int bpsm : {1, 2, 4}) {
        for (int threads : {128, 256}) {
            int grid = sms * bpsm;
            int it = iters / 4;
            float ms = time_it([&] { dmma884_kernel<8><<<grid, threads>>>(out, it); }, 5);
            double fl = 2.0 * 256 * 8 * (double)it * grid * (threads / 32);
            printf("{\"kind\":\"dmma_m8n8k4\",\"chains\":8,\"blocks_per_sm\":%d,\"threads\":%d,\"ms\":%.4f,\"tflops\":%.3f}\n",
                   bpsm, threads, ms, fl / ms / 1e9);
            ms = time_it([&] { dmma1684_kernel<8><<<grid, threads>>>(out, it); }, 5);
            fl = 2.0 * 512 * 8 * (double)it * grid * (threads / 32);
            printf("{\"kind\":\"dmma_m16n8k4\",\"chains\":8,\"blocks_per_sm\":%d,\"threads\":%d,\"ms\":%.4f,\"tflops\":%.3f}\n",
                   bpsm, threads, ms, fl / ms / 1e9);
            ms = time_it([&] { dmma16816_kernel<4><<<grid, threads>>>(out, it / 4); }, 5);
            fl = 2.0 * 2048 * 4 * (double)(it / 4) * grid * (threads / 32);
            printf("{\"kind\":\"dmma_m16n8k16\",\"chains\":4,\"blocks_per_sm\":%d,\"threads\":%d,\"ms\":%.4f,\"tflops\":%.3f}\n",
                   bpsm, threads, ms, fl / ms / 1e9);
        }
    }
    // sustained DFMA for ~3 s (power-cap behaviour)
    {
        int grid = sms * 2, threads = 256;
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        int n = 0;
        for (; n < 200; ++n) dfma_kernel<8><<<grid, threads>>>(out, iters, 1.0000001);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 8 * iters * (double)grid * threads * n;
        printf("{\"kind\":\"dfma_sustained\",\"launches\":%d,\"ms\":%.2f,\"tflops\":%.3f}\n", n, ms, fl / ms / 1e9);
        cudaEventRecord(e0);
        int it = iters / 4;
        for (n = 0; n < 200; ++n) dmma884_kernel<8><<<grid, threads>>>(out, it);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        fl = 2.0 * 256 * 8 * (double)it * grid * (threads / 32) * n;
        printf("{\"kind\":\"dmma884_sustained\",\"launches\":%d,\"ms\":%.2f,\"tflops\":%.3f}\n", n, ms, fl / ms / 1e9);
    }
    CK(cudaGetLastError());
    return 0;
}
