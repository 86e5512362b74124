#include <algorithm>
// BF16 / TF32-input C(fp32) += A·B on the 5th-generation tensor cores
// (tcgen05 + TMEM), BASELINE.json configs[3]. sm_100a only.
//
// Same task model as the FP64 kernels (gpu.hpp): a persistent grid walks the
// lowered task list; each task is one 128 x 256 C tile over a k range.
// Warp roles (256 threads):
//   warp 0      TMA producer: A (column-major = M-major) and B (column-major =
//               K-major) k-slabs -> 128B-swizzled shared memory, 4-stage ring
//               of full/empty mbarriers;
//   warp 1      MMA issuer: one thread issues tcgen05.mma (M=128, N=256,
//               K=32 bytes) into a TMEM accumulator, commits to the ring's
//               empty barriers and, per tile, to the accumulator-full barrier;
//   warp 2      TMEM allocator (512 columns = two 256-column accumulators);
//   warps 4..7  epilogue: tcgen05.ld 32 lanes x 32 columns per warp, C += acc
//               with coalesced fp32 column accesses, then release the
//               accumulator so the next tile's MMAs overlap this epilogue.
// The SMEM level of the MOMMS member is the TMA ring; the register level is
// the TMEM accumulator (128 x 256 fp32 per tile).
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "gpu.hpp"

namespace mmm {
namespace gpu {
namespace {

#ifndef TC_CPF_AHEAD
#define TC_CPF_AHEAD 8  // k-blocks before the end of a tile at which the pair kernel prefetches its C
#endif
constexpr int kTcStages = 4;
constexpr int kTcBM = 128, kTcBN = 256;

__device__ __forceinline__ uint32_t saddr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(saddr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "TC_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra TC_DONE;\n\t"
        "bra TC_WAIT;\n"
        "TC_DONE:\n\t}\n" ::"r"(saddr(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];\n" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(src), "r"(c0), "r"(c1)
                 : "memory");
}
// C += box, the add done by the L2 (TMA reduction): the epilogue never reads C into the SM
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* map, uint32_t src, int c0, int c1) {
    asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];\n" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(src), "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void tma_load_2d_cta(uint32_t dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(saddr(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::
            "r"(saddr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(saddr(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// Shared-memory matrix descriptor (SM100 UMMA): start, LBO, SBO in 16-byte
// units, version 1, layout type 2 = SWIZZLE_128B (16-byte atoms, 8-row
// period) or 1 = SWIZZLE_128B_BASE32B (32-byte atoms, 4-row period; the only
// M-major layout tf32 operands accept).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout = 2) {
    return static_cast<uint64_t>((addr >> 4) & 0x3FFF) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
           (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) |
           (static_cast<uint64_t>(layout) << 61);
}

// Instruction descriptor: D fp32, A/B format (BF16 = 1, TF32 = 2), A M-major,
// B K-major, N = 256, M = 128.
template <bool TF32>
__host__ __device__ constexpr uint32_t instr_desc() {
    return (1u << 4) | ((TF32 ? 2u : 1u) << 7) | ((TF32 ? 2u : 1u) << 10) | (1u << 15) | (0u << 16) |
           (static_cast<uint32_t>(kTcBN >> 3) << 17) | (static_cast<uint32_t>(kTcBM >> 4) << 24);
}

template <bool TF32>
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accumulate) {
    if constexpr (TF32) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
            "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
            : "memory");
    } else {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
            "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
            : "memory");
    }
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(saddr(bar))
                 : "memory");
}

#define TC_LD32(taddr, r)                                                                                           \
    asm volatile(                                                                                                   \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18," \
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"                                            \
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),          \
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),    \
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),  \
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])   \
        : "r"(taddr))

// C(row, c0 .. c0+31) += acc for one thread's row: all 32 loads are issued
// before any add (a dependent load/add/store per column would serialise
// ~32 memory latencies per chunk and make the epilogue, not the MMA, the
// critical path). Consecutive lanes own consecutive rows, so every column
// access of a warp is one coalesced 128-byte line.
__device__ __forceinline__ void epilogue_chunk(float* c, int64_t ldc, int ncols, const uint32_t (&r)[32]) {
    if (ncols >= 32) {
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __ldcs(c + j * ldc);
#pragma unroll
        for (int j = 0; j < 32; ++j) __stcs(c + j * ldc, v[j] + __uint_as_float(r[j]));
    } else {
        for (int j = 0; j < ncols; ++j) c[j * ldc] = c[j * ldc] + __uint_as_float(r[j]);
    }
}

struct TcArgs {
    float* C;
    int64_t ldc;
    const Task* tasks;
    int32_t ntasks;
    int64_t m = 0, n = 0;   // C extents (the TMA epilogue's clipping bounds)
    int32_t tma_c = 0;      // 256 x 512 pair kernel: tmC maps C (16-byte aligned columns) for the TMA epilogue
    int32_t tma_red = 0;    // 256 x 512 TMA epilogue: C += acc by TMA reduce-add in L2 (no C load)
    int32_t clc = 0;        // pair kernels: tiles by cluster launch control (one cluster launched per tile,
                            // running clusters cancel not-yet-started ones and take their tiles)
};

template <bool TF32>
struct TcGeo {
    static constexpr int E = TF32 ? 4 : 2;     // bytes per input element
    static constexpr int BK = 128 / E;          // k per stage: one 128-byte swizzle row of K-major B
    static constexpr int MATOM = 128 / E;       // m per 128-byte row of M-major A
    static constexpr int A_BOXES = kTcBM / MATOM;
    static constexpr int A_BOX_BYTES = 128 * BK;
    static constexpr int A_BYTES = kTcBM * BK * E;
    static constexpr int B_BYTES = kTcBN * BK * E;
    static constexpr int STAGE = A_BYTES + B_BYTES;
    static constexpr int UK = 32 / E;           // k per MMA instruction
    static constexpr int NMMA = BK / UK;
    // M-major A: bf16 uses SWIZZLE_128B (8-row groups), tf32 SWIZZLE_128B_BASE32B (4-row groups)
    static constexpr uint32_t A_LAYOUT = TF32 ? 1u : 2u;
    static constexpr uint32_t A_SBO = TF32 ? 512u : 1024u;
    static constexpr int SMEM = kTcStages * STAGE + 1024 /*align*/ + 256 /*barriers*/;
};

template <bool TF32>
__global__ void __launch_bounds__(256, 1) k_tc(const __grid_constant__ CUtensorMap tmA,
                                               const __grid_constant__ CUtensorMap tmB, TcArgs a) {
    using G = TcGeo<TF32>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kTcStages * G::STAGE);
    uint64_t* empty = full + kTcStages;
    uint64_t* tfull = empty + kTcStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    }
    if (warp == 1 && lane == 0) {
        for (int s = 0; s < kTcStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(saddr(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer
            int stage = 0;
            uint32_t phase = 0;
            for (int ti = blockIdx.x; ti < a.ntasks; ti += gridDim.x) {
                const Task t = a.tasks[ti];
                const int nk = (t.k + G::BK - 1) / G::BK;
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* sa = smem + stage * G::STAGE;
                    uint8_t* sb = sa + G::A_BYTES;
                    mbar_expect_tx(&full[stage], G::STAGE);
                    const int kc = t.p0 + kb * G::BK;
#pragma unroll
                    for (int h = 0; h < G::A_BOXES; ++h)
                        tma_load_2d(sa + h * G::A_BOX_BYTES, &tmA, &full[stage], t.i0 + h * G::MATOM, kc);
                    tma_load_2d(sb, &tmB, &full[stage], kc, t.j0);
                    if (++stage == kTcStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---------------- MMA issuer
            constexpr uint32_t idesc = instr_desc<TF32>();
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t aphase = 0;
            for (int ti = blockIdx.x; ti < a.ntasks; ti += gridDim.x) {
                const Task t = a.tasks[ti];
                const int nk = (t.k + G::BK - 1) / G::BK;
                mbar_wait(&tempty[acc], aphase ^ 1);
                tc_fence_after();
                const uint32_t tmem_d = tmem_base + static_cast<uint32_t>(acc * kTcBN);
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t sa = saddr(smem + stage * G::STAGE);
                    const uint32_t sb = sa + G::A_BYTES;
#pragma unroll
                    for (int kk = 0; kk < G::NMMA; ++kk) {
                        // A: M-major SW128 — LBO = next 128-byte M chunk (one TMA box), SBO = next 8 k rows.
                        const uint64_t da = smem_desc(sa + kk * G::UK * 128, G::A_BOX_BYTES, G::A_SBO, G::A_LAYOUT);
                        // B: K-major SW128 — advance 32 bytes of k inside the swizzled row, SBO = 8 n rows.
                        const uint64_t db = smem_desc(sb + kk * 32, 16, 1024);
                        umma<TF32>(tmem_d, da, db, idesc, (kb | kk) != 0 ? 1u : 0u);
                    }
                    umma_commit(&empty[stage]);
                    if (++stage == kTcStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma_commit(&tfull[acc]);
                if (++acc == 2) {
                    acc = 0;
                    aphase ^= 1;
                }
            }
        }
    } else if (warp >= 4) {  // ---------------- epilogue
        const int ew = warp - 4;
        const int row = ew * 32 + lane;
        int acc = 0;
        uint32_t aphase = 0;
        for (int ti = blockIdx.x; ti < a.ntasks; ti += gridDim.x) {
            const Task t = a.tasks[ti];
            mbar_wait(&tfull[acc], aphase);
            tc_fence_after();
            const bool live = row < t.m;
            float* crow = a.C + (static_cast<int64_t>(t.i0) + row) + static_cast<int64_t>(t.j0) * a.ldc;
#pragma unroll 1
            for (int cb = 0; cb < kTcBN / 32; ++cb) {
                uint32_t r[32];
                const uint32_t taddr = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) +
                                       static_cast<uint32_t>(acc * kTcBN + cb * 32);
                TC_LD32(taddr, r);
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                if (live) epilogue_chunk(crow + static_cast<int64_t>(cb * 32) * a.ldc, a.ldc, t.n - cb * 32, r);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            if (++acc == 2) {
                acc = 0;
                aphase ^= 1;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem_base) : "memory");
    }
}

// ======================= tensor-pipe peak probe =======================
// One CTA per SM, one thread issuing M=128 x N=256 tcgen05.mma back to back
// from fixed shared-memory operands (contents irrelevant to throughput) into
// one TMEM accumulator: the issue-rate ceiling of the MMA path the GEMM
// kernels use, measured on this device under its own clocks and power cap.
template <bool TF32>
__global__ void __launch_bounds__(128, 1) k_tc_peak(int iters) {
    using G = TcGeo<TF32>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* done = reinterpret_cast<uint64_t*>(smem + G::STAGE);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(saddr(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) {
        constexpr uint32_t idesc = instr_desc<TF32>();
        const uint32_t sa = saddr(smem), sb = sa + G::A_BYTES;
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int kk = 0; kk < G::NMMA; ++kk)
                umma<TF32>(tmem, smem_desc(sa + kk * G::UK * 128, G::A_BOX_BYTES, G::A_SBO, G::A_LAYOUT),
                           smem_desc(sb + kk * 32, 16, 1024), idesc, (i | kk) != 0 ? 1u : 0u);
        }
        umma_commit(done);
        mbar_wait(done, 0);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tmem) : "memory");
    }
}

template <bool TF32>
cudaError_t measure_tc_peak_t(int launches, bool sustained, double* tflops) {
    using G = TcGeo<TF32>;
    int dev = 0, sms = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // ~half the opt-in shared memory: one CTA per SM
    const int smem = 110 * 1024;
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_tc_peak<TF32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    // ~5 ms per launch (burst: full clocks), or ~200 ms (sustained: under the power cap, like a long GEMM)
    const int iters = (TF32 ? 2048 : 4096) * (sustained ? 40 : 1);
    const double flops = 2.0 * kTcBM * kTcBN * G::BK * static_cast<double>(iters) * sms;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_tc_peak<TF32><<<sms, 128, smem>>>(iters);  // warm-up
    double best = 0;
    for (int l = 0; l < launches && e == cudaSuccess; ++l) {
        cudaEventRecord(e0);
        k_tc_peak<TF32><<<sms, 128, smem>>>(iters);
        cudaEventRecord(e1);
        e = cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms > 0) best = std::max(best, flops / (ms * 1e-3) / 1e12);
    }
    if (e == cudaSuccess) e = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *tflops = best;
    return e;
}

// ======================= 2-SM pair kernel (cta_group::2) =======================
// A cluster of two CTAs on one TPC computes a 256 x 256 C tile with
// tcgen05.mma.cta_group::2 (M = 256): each CTA stages its 128 rows of A and
// its 128 columns of B (so each SM ingests 32 KB per 64-deep bf16 stage for a
// 128 x 256 result, two thirds of the single-CTA kernel's 48 KB), the leader
// (rank 0) issues the MMAs, each CTA's TMEM holds its own 128 accumulator
// rows. Barrier protocol (the one CUTLASS's 2-SM pipelines use):
//   full[s]   leader only; armed by the leader's producer with both CTAs'
//             bytes; both CTAs' 2-SM TMA loads complete_tx on it;
//   empty[s]  both CTAs; the leader's MMA commit multicasts to both;
//   tfull[a]  both CTAs; the leader's per-tile commit multicasts to both;
//   tempty[a] leader only; the 4 epilogue warps of both CTAs arrive (count 8).
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa_rank(const void* p, uint32_t rank) {
    uint32_t out;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(out) : "r"(saddr(p)), "r"(rank));
    return out;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t leader_bar, int c0,
                                                 int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
        "%4}], [%2];\n" ::"r"(saddr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1)
        : "memory");
}
template <bool TF32>
__device__ __forceinline__ void umma_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
    if constexpr (TF32) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
            "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
            : "memory");
    } else {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
            "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
            : "memory");
    }
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
            saddr(bar)),
        "h"(static_cast<uint16_t>(3))
        : "memory");
}

// ---- cluster launch control (sm_100): dynamic persistent tiles ----
// The grid launches one cluster per tile. A running cluster asks the hardware
// to cancel a cluster that has not started yet (clusterlaunchcontrol.try_cancel)
// and, if that succeeds, computes the canceled cluster's tile next. Tiles are
// taken in launch order, by whichever cluster is free first -- the window of
// tiles in flight stays a run of consecutive raster tiles, as with fresh
// clusters -- while the running cluster keeps its TMEM, barriers and pipeline
// (no launch, no refill, and the next tile's loads and MMAs overlap this
// tile's epilogue). Query j (j = 1, 2, ...) has its 16-byte response
// multicast into both CTAs' resp[(j-1) % 4] and completes their
// clc_full[(j-1) % 4]; every role (both producers, the MMA issuer, every
// epilogue warp) reads it and arrives on the leader's clc_empty[(j-1) % 4]
// before the slot is reused four queries later.
constexpr int kClcSlots = 4;
__device__ __forceinline__ void clc_try_cancel(uint32_t resp, uint64_t* bar) {
    asm volatile(
        "clusterlaunchcontrol.try_cancel.async.shared::cta.mbarrier::complete_tx::bytes.multicast::cluster::all.b128 "
        "[%0], [%1];\n" ::"r"(resp),
        "r"(saddr(bar))
        : "memory");
}
// -1: no cluster was left to cancel; else the canceled cluster's index
__device__ __forceinline__ int clc_decode(uint32_t resp) {
    uint32_t ok, x = 0;
    asm volatile(
        "{\n .reg .pred p;\n .reg .b128 r;\n ld.shared.b128 r, [%2];\n"
        " clusterlaunchcontrol.query_cancel.is_canceled.pred.b128 p, r;\n selp.u32 %0, 1, 0, p;\n"
        " @p clusterlaunchcontrol.query_cancel.get_first_ctaid::x.b32.b128 %1, r;\n}\n"
        : "=r"(ok), "+r"(x)
        : "r"(resp)
        : "memory");
    return ok ? static_cast<int>(x >> 1) : -1;
}
__device__ __forceinline__ void mbar_arrive_expect_tx_remote(uint32_t cluster_addr, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;\n" ::"r"(cluster_addr),
                 "r"(bytes)
                 : "memory");
}

// NH = 256-column halves of the pair tile: 1 -> 256 x 256 per pair, two
// TMEM accumulators (the next tile's MMAs overlap this tile's epilogue);
// 2 -> 256 x 512 per pair, one accumulator filling TMEM (512 columns), 25 %
// fewer L2->SMEM bytes per flop, epilogue by 8 warps and not overlapped.
template <bool TF32, int NH = 1>
struct Tc2Geo {
    static constexpr int E = TF32 ? 4 : 2;
    static constexpr int BK = 128 / E;
    static constexpr int MATOM = 128 / E;
    static constexpr int A_BOXES = 128 / MATOM;  // this CTA's 128 rows
    static constexpr int A_BOX_BYTES = 128 * BK;
    static constexpr int A_BYTES = 128 * BK * E;
    static constexpr int B_HALF_BYTES = 128 * BK * E;  // this CTA's 128 columns of one 256-column half
    static constexpr int B_BYTES = NH * B_HALF_BYTES;
    static constexpr int STAGE = A_BYTES + B_BYTES;
    static constexpr int PAIR_STAGE_BYTES = 2 * STAGE;
    static constexpr int UK = 32 / E;
    static constexpr int NMMA = BK / UK;
    static constexpr int STAGES = NH == 1 ? 6 : 4;
    static constexpr int NACC = NH == 1 ? 2 : 1;      // TMEM accumulators of 256 * NH columns
    static constexpr int EPI_WARPS = 4 * NH;
    static constexpr int THREADS = 128 + 32 * EPI_WARPS;
    static constexpr uint32_t A_LAYOUT = TF32 ? 1u : 2u;
    static constexpr uint32_t A_SBO = TF32 ? 512u : 1024u;
    static constexpr int SMEM = STAGES * STAGE + 1024 + 512;
};

template <bool TF32>
__host__ __device__ constexpr uint32_t instr_desc_pair() {
    return (1u << 4) | ((TF32 ? 2u : 1u) << 7) | ((TF32 ? 2u : 1u) << 10) | (1u << 15) | (0u << 16) |
           (static_cast<uint32_t>(256 >> 3) << 17) | (static_cast<uint32_t>(256 >> 4) << 24);
}

template <bool TF32, int NH = 1>
__global__ void __launch_bounds__(Tc2Geo<TF32, NH>::THREADS, 1) k_tc2(const __grid_constant__ CUtensorMap tmA,
                                                                  const __grid_constant__ CUtensorMap tmB, TcArgs a,
                                                                  const __grid_constant__ CUtensorMap tmC) {
    using G = Tc2Geo<TF32, NH>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + G::STAGES * G::STAGE);
    uint64_t* empty = full + G::STAGES;
    uint64_t* tfull = empty + G::STAGES;
    uint64_t* tempty = tfull + 2;
    uint64_t* cl = tempty + 2;  // TMA epilogue: C quarter loads into the (then idle) stage ring, 3 buffers
    uint64_t* clc_full = cl + 3;                // cluster launch control: response landed (both CTAs)
    uint64_t* clc_empty = clc_full + kClcSlots;  // response read by every role (leader's copy counts)
    uint4* clc_resp = reinterpret_cast<uint4*>((reinterpret_cast<uintptr_t>(clc_empty + kClcSlots) + 15) & ~uintptr_t(15));
    // clc + TMA epilogue (256 x 512): the epilogue stages C through the stage ring, so the producer starts a
    // cluster's next tile only once this CTA's epilogue is done with the ring (it warms L2 with the tile's
    // first k-blocks meanwhile)
    uint64_t* ring_free = reinterpret_cast<uint64_t*>(clc_resp + kClcSlots);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ring_free + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    }
    if (warp == 1 && lane == 0) {
        for (int s = 0; s < G::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], 2 * G::EPI_WARPS);
        }
        for (int s = 0; s < 3; ++s) mbar_init(&cl[s], 1);
        mbar_init(ring_free, 1);
        for (int s = 0; s < kClcSlots; ++s) {
            mbar_init(&clc_full[s], 1);
            mbar_init(&clc_empty[s], 3 + 2 * G::EPI_WARPS);  // 2 producers, the MMA issuer, every epilogue warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(saddr(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
    }
    tc_fence_before();
    cluster_sync_all();  // barriers of both CTAs initialised and TMEM allocated before any remote traffic
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    // The cluster's tile sequence: its own tile, then (clc) the tiles of the clusters it cancels, or
    // (static) every nclusters-th tile. Every role walks the same sequence.
    // queries are numbered from 1 (the cluster's own tile needs none): query q uses slot (q-1) % kClcSlots,
    // phase (q-1) / kClcSlots of its barriers
    auto clc_issue = [&](int q) {  // leader's producer: query q, once query q - kClcSlots has been read by all
        const int sl = (q - 1) % kClcSlots;
        if (q > kClcSlots) mbar_wait(&clc_empty[sl], ((q - 1) / kClcSlots - 1) & 1);
        mbar_expect_tx(&clc_full[sl], 16);
        mbar_arrive_expect_tx_remote(mapa_rank(&clc_full[sl], 1), 16);
        clc_try_cancel(saddr(&clc_resp[sl]), &clc_full[sl]);
    };
    auto next_tile = [&](int ti, int& j, bool arrive) {  // arrive: this thread is its role's counted one
        if (!a.clc) return ti + nclusters;
        ++j;
        const int sl = (j - 1) % kClcSlots;
        mbar_wait(&clc_full[sl], ((j - 1) / kClcSlots) & 1);
        const int t = clc_decode(saddr(&clc_resp[sl]));
        if (arrive) mbar_arrive_remote(mapa_rank(&clc_empty[sl], 0));
        return t < 0 ? a.ntasks : t;
    };

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer (both CTAs)
            int stage = 0;
            uint32_t phase = 0;
            int j = 0;
            uint32_t ntile = 0;
            const bool gate = NH == 2 && a.clc && a.tma_c;
            if (a.clc && leader) clc_issue(1);
            for (int ti = cluster; ti < a.ntasks; ++ntile) {
                const Task t = a.tasks[ti];
                const int nk = (t.k + G::BK - 1) / G::BK;
                if (gate && ntile > 0) {
                    for (int kb = 0; kb < nk && kb < G::STAGES; ++kb) {
                        const int kc = t.p0 + kb * G::BK;
                        for (int h = 0; h < G::A_BOXES; ++h)
                            asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];\n" ::"l"(
                                             reinterpret_cast<uint64_t>(&tmA)),
                                         "r"(t.i0 + static_cast<int>(rank) * 128 + h * G::MATOM), "r"(kc)
                                         : "memory");
                        for (int h = 0; h < NH; ++h)
                            asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];\n" ::"l"(
                                             reinterpret_cast<uint64_t>(&tmB)),
                                         "r"(kc), "r"(t.j0 + h * 256 + static_cast<int>(rank) * 128)
                                         : "memory");
                    }
                    mbar_wait(ring_free, (ntile - 1) & 1);
                }
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (NH == 2 && a.tma_c && kb == nk - TC_CPF_AHEAD) {
                        // the TMA epilogue reads this CTA's C quarters right after the k loop: warm L2 with them
                        for (int q = 0; q < 4; ++q)
                            asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];\n" ::"l"(
                                             reinterpret_cast<uint64_t>(&tmC)),
                                         "r"(t.i0 + static_cast<int>(rank) * 128), "r"(t.j0 + q * 128)
                                         : "memory");
                    }
                    uint8_t* sa = smem + stage * G::STAGE;
                    uint8_t* sb = sa + G::A_BYTES;
                    if (leader) mbar_expect_tx(&full[stage], G::PAIR_STAGE_BYTES);
                    const uint32_t bar = mapa_rank(&full[stage], 0);
                    const int kc = t.p0 + kb * G::BK;
#pragma unroll
                    for (int h = 0; h < G::A_BOXES; ++h)
                        tma_load_2d_pair(sa + h * G::A_BOX_BYTES, &tmA, bar,
                                         t.i0 + static_cast<int>(rank) * 128 + h * G::MATOM, kc);
#pragma unroll
                    for (int h = 0; h < NH; ++h)
                        tma_load_2d_pair(sb + h * G::B_HALF_BYTES, &tmB, bar, kc,
                                         t.j0 + h * 256 + static_cast<int>(rank) * 128);
                    if (++stage == G::STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                ti = next_tile(ti, j, true);
                if (a.clc && leader && ti < a.ntasks) clc_issue(j + 1);  // one tile ahead
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && leader) {  // ---------------- MMA issuer (leader only)
            constexpr uint32_t idesc = instr_desc_pair<TF32>();
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t aphase = 0;
            int j = 0;
            for (int ti = cluster; ti < a.ntasks; ti = next_tile(ti, j, true)) {
                const Task t = a.tasks[ti];
                const int nk = (t.k + G::BK - 1) / G::BK;
                mbar_wait(&tempty[acc], aphase ^ 1);
                tc_fence_after();
                const uint32_t tmem_d = tmem_base + static_cast<uint32_t>(acc * 256);
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t sa = saddr(smem + stage * G::STAGE);
                    const uint32_t sb = sa + G::A_BYTES;
#pragma unroll
                    for (int kk = 0; kk < G::NMMA; ++kk) {
                        const uint64_t da = smem_desc(sa + kk * G::UK * 128, G::A_BOX_BYTES, G::A_SBO, G::A_LAYOUT);
#pragma unroll
                        for (int h = 0; h < NH; ++h) {
                            const uint64_t db = smem_desc(sb + h * G::B_HALF_BYTES + kk * 32, 16, 1024);
                            umma_pair<TF32>(tmem_d + h * 256, da, db, idesc, (kb | kk) != 0 ? 1u : 0u);
                        }
                    }
                    umma_commit_pair(&empty[stage]);
                    if (++stage == G::STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma_commit_pair(&tfull[acc]);
                if (++acc == G::NACC) {
                    acc = 0;
                    aphase ^= 1;
                }
            }
        }
    } else if (warp >= 4) {  // ---------------- epilogue (both CTAs, own 128 rows; warp group h: columns of half h)
        const int ew = warp & 3, h = (warp - 4) >> 2;  // TMEM lanes 32*(warp%4).. are this warp's
        const int row = static_cast<int>(rank) * 128 + ew * 32 + lane;
        int acc = 0;
        uint32_t aphase = 0;
        uint32_t ntask = 0;
        int j = 0;
        for (int ti = cluster; ti < a.ntasks; ti = next_tile(ti, j, lane == 0), ++ntask) {
            const Task t = a.tasks[ti];
            mbar_wait(&tfull[acc], aphase);
            tc_fence_after();
            // TMA epilogue (256 x 512 pair tiles, one task per cluster so the stage ring is idle): C moves
            // between L2 and shared memory in 128-row x 128-column quarters by bulk tensor copies, three
            // buffers in the ring, and each lane adds its TMEM row into shared memory. A box store writes
            // its whole box, clipped only at C's edges, so the task must cover its box region.
            if constexpr (NH == 2) {
                const bool covers = (t.m == 256 || static_cast<int64_t>(t.i0) + t.m == a.m) &&
                                    (t.n == 512 || static_cast<int64_t>(t.j0) + t.n == a.n);
                if (a.tma_c && covers && (a.ntasks <= nclusters || a.clc)) {
                    constexpr uint32_t QB = 128 * 128 * 4;  // bytes of one quarter
                    const uint32_t cbase = saddr(smem);
                    const int r0 = t.i0 + static_cast<int>(rank) * 128;
                    const bool issuer = warp == 4 && lane == 0;
                    const uint32_t ph = ntask & 1;  // cl[1], cl[2] complete once per task, cl[0] twice
                    if (a.tma_red) {
                        // Reduction epilogue: each lane writes its TMEM row of a quarter into a ring buffer and
                        // one thread issues a TMA reduce-add of the quarter onto C -- the L2 adds, so C is
                        // never loaded into the SM (one SMEM pass per quarter instead of load + read + write +
                        // store). Quarter 3 reuses buffer 0 once quarter 0's reduction has read it.
                        const int g = (warp - 4) >> 2;
                        for (int q = 0; q < 4; ++q) {
                            const int buf = q % 3;
                            if (q == 3) {
                                if (issuer) asm volatile("cp.async.bulk.wait_group.read 2;\n" ::: "memory");
                                asm volatile("bar.sync 1, %0;\n" ::"n"(32 * G::EPI_WARPS) : "memory");
                            }
                            float* cs = reinterpret_cast<float*>(smem + buf * QB);
#pragma unroll 1
                            for (int cc = 0; cc < 2; ++cc) {
                                const int col = g * 64 + cc * 32;
                                uint32_t r[32];
                                TC_LD32(tmem_base + (static_cast<uint32_t>(ew * 32) << 16) +
                                            static_cast<uint32_t>(q * 128 + col), r);
                                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
                                for (int j = 0; j < 32; ++j) cs[(col + j) * 128 + ew * 32 + lane] = __uint_as_float(r[j]);
                            }
                            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                            asm volatile("bar.sync 1, %0;\n" ::"n"(32 * G::EPI_WARPS) : "memory");
                            if (issuer) {
                                tma_reduce_add_2d(&tmC, cbase + buf * QB, r0, t.j0 + q * 128);
                                asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
                            }
                        }
                        if (issuer) {
                            asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
                            if (a.clc) mbar_arrive(ring_free);  // the ring is the producer's again
                        }
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive_remote(mapa_rank(&tempty[acc], 0));
                        if (++acc == G::NACC) {
                            acc = 0;
                            aphase ^= 1;
                        }
                        continue;
                    }
                    if (issuer) {
                        for (int q = 0; q < 3; ++q) {
                            mbar_expect_tx(&cl[q], QB);
                            tma_load_2d_cta(cbase + q * QB, &tmC, &cl[q], r0, t.j0 + q * 128);
                        }
                    }
                    const int g = (warp - 4) >> 2;  // this warp's 64 columns of each quarter
                    for (int q = 0; q < 4; ++q) {
                        const int buf = q % 3;
                        mbar_wait(&cl[buf], buf == 0 ? (q == 0 ? 0u : 1u) : ph);
                        float* cs = reinterpret_cast<float*>(smem + buf * QB);
#pragma unroll 1
                        for (int cc = 0; cc < 2; ++cc) {
                            const int col = g * 64 + cc * 32;
                            uint32_t r[32];
                            TC_LD32(tmem_base + (static_cast<uint32_t>(ew * 32) << 16) +
                                        static_cast<uint32_t>(q * 128 + col), r);
                            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
                            for (int j = 0; j < 32; ++j) cs[(col + j) * 128 + ew * 32 + lane] += __uint_as_float(r[j]);
                        }
                        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                        asm volatile("bar.sync 1, %0;\n" ::"n"(32 * G::EPI_WARPS) : "memory");
                        if (issuer) {
                            tma_store_2d(&tmC, cbase + buf * QB, r0, t.j0 + q * 128);
                            asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
                            if (q == 0) {  // quarter 3 reuses buffer 0 once the store has read it
                                asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
                                mbar_expect_tx(&cl[0], QB);
                                tma_load_2d_cta(cbase, &tmC, &cl[0], r0, t.j0 + 3 * 128);
                            }
                        }
                    }
                    if (issuer) {
                        asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
                        if (a.clc) mbar_arrive(ring_free);  // the ring is the producer's again
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_remote(mapa_rank(&tempty[acc], 0));
                    if (++acc == G::NACC) {
                        acc = 0;
                        aphase ^= 1;
                    }
                    continue;
                }
            }
            if (NH == 2 && a.clc && a.tma_c && warp == 4 && lane == 0) mbar_arrive(ring_free);  // (ring untouched)
            const bool live = row < t.m;
            float* crow = a.C + (static_cast<int64_t>(t.i0) + row) + static_cast<int64_t>(t.j0 + h * 256) * a.ldc;
#pragma unroll 1
            for (int cb = 0; cb < 256 / 32; ++cb) {
                uint32_t r[32];
                const uint32_t taddr = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) +
                                       static_cast<uint32_t>(acc * 256 + h * 256 + cb * 32);
                TC_LD32(taddr, r);
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                if (live) epilogue_chunk(crow + static_cast<int64_t>(cb * 32) * a.ldc, a.ldc, t.n - h * 256 - cb * 32, r);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(mapa_rank(&tempty[acc], 0));
            if (++acc == G::NACC) {
                acc = 0;
                aphase ^= 1;
            }
        }
    }
    tc_fence_before();
    cluster_sync_all();  // no CTA leaves (or frees TMEM) while its peer may still signal it
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem_base) : "memory");
    }
}

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::mutex g_tc_mu;  // lazy driver-entry lookup and per-kernel attribute setup

cudaError_t encoder() {
    std::lock_guard<std::mutex> lk(g_tc_mu);
    if (g_encode) return cudaSuccess;
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess) return e;
    if (q != cudaDriverEntryPointSuccess || fn == nullptr) return cudaErrorNotSupported;
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    return cudaSuccess;
}

}  // namespace

void* tensor_map_encoder() { return encoder() == cudaSuccess ? reinterpret_cast<void*>(g_encode) : nullptr; }

namespace {

// 2-D column-major tensor map: dim0 contiguous (rows), box {box0, box1}, 128B swizzle.
cudaError_t make_map(CUtensorMap* m, const void* base, bool tf32, int64_t rows, int64_t cols, int64_t ld, int box0,
                     int box1, CUtensorMapSwizzle swz) {
    const int E = tf32 ? 4 : 2;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(cols)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * E};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(box0), static_cast<cuuint32_t>(box1)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = g_encode(m, tf32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                          const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <bool TF32>
cudaError_t launch_tc_t(const void* A, int64_t lda, const void* B, int64_t ldb, float* C, int64_t ldc, int64_t m,
                        int64_t n, int64_t k, const Task* tasks, int ntasks, int grid, cudaStream_t stream) {
    using G = TcGeo<TF32>;
    cudaError_t e = encoder();
    if (e != cudaSuccess) return e;
    if ((lda * G::E) % 16 || (ldb * G::E) % 16 || reinterpret_cast<uintptr_t>(A) % 16 ||
        reinterpret_cast<uintptr_t>(B) % 16)
        return cudaErrorInvalidValue;  // TMA: 16-byte aligned bases and row strides
    CUtensorMap ma, mb;
    if ((e = make_map(&ma, A, TF32, m, k, lda, G::MATOM, G::BK,
                      TF32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B)) != cudaSuccess)
        return e;
    if ((e = make_map(&mb, B, TF32, k, n, ldb, G::BK, kTcBN, CU_TENSOR_MAP_SWIZZLE_128B)) != cudaSuccess) return e;
    static bool attr[2] = {false, false};
    std::lock_guard<std::mutex> lk(g_tc_mu);
    if (!attr[TF32]) {
        if ((e = cudaFuncSetAttribute(k_tc<TF32>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM)) != cudaSuccess)
            return e;
        attr[TF32] = true;
    }
    TcArgs args{C, ldc, tasks, ntasks};
    k_tc<TF32><<<grid, 256, G::SMEM, stream>>>(ma, mb, args);
    return cudaGetLastError();
}

// Round fp64 values to bf16 (RNE) or to tf32-in-fp32 (RNE to 10 mantissa bits).
__global__ void k_round_bf16(const double* x, uint16_t* y, int64_t count) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        // exact RNE of the double to 8 significant bits (bf16), no double rounding via fp32
        int ex;
        const double mant = frexp(x[i], &ex);  // x = mant * 2^ex, 0.5 <= |mant| < 1
        const float r = static_cast<float>(ldexp(rint(ldexp(mant, 8)), ex - 8));
        y[i] = static_cast<uint16_t>(__float_as_uint(r) >> 16);
    }
}
__global__ void k_round_tf32(const double* x, float* y, int64_t count) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int ex;
        const double mant = frexp(x[i], &ex);
        const double q = rint(ldexp(mant, 11));       // tf32: 10 stored + implicit = 11 significant bits
        y[i] = static_cast<float>(ldexp(q, ex - 11));
    }
}

template <bool TF32, int NH>
cudaError_t launch_tc2_t(const void* A, int64_t lda, const void* B, int64_t ldb, float* C, int64_t ldc, int64_t m,
                         int64_t n, int64_t k, const Task* tasks, int ntasks, int grid, cudaStream_t stream) {
    using G = Tc2Geo<TF32, NH>;
    cudaError_t e = encoder();
    if (e != cudaSuccess) return e;
    if ((lda * G::E) % 16 || (ldb * G::E) % 16 || reinterpret_cast<uintptr_t>(A) % 16 ||
        reinterpret_cast<uintptr_t>(B) % 16)
        return cudaErrorInvalidValue;
    CUtensorMap ma, mb;
    if ((e = make_map(&ma, A, TF32, m, k, lda, G::MATOM, G::BK,
                      TF32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B)) != cudaSuccess)
        return e;
    if ((e = make_map(&mb, B, TF32, k, n, ldb, G::BK, 128, CU_TENSOR_MAP_SWIZZLE_128B)) != cudaSuccess) return e;
    static bool attr[2] = {false, false};
    std::lock_guard<std::mutex> lk(g_tc_mu);
    if (!attr[TF32]) {
        if ((e = cudaFuncSetAttribute(k_tc2<TF32, NH>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM)) !=
            cudaSuccess)
            return e;
        attr[TF32] = true;
    }
    TcArgs args{C, ldc, tasks, ntasks};
    args.m = m;
    args.n = n;
    CUtensorMap mc;
    std::memset(&mc, 0, sizeof(mc));
    if (NH == 2 && (ldc * 4) % 16 == 0 && reinterpret_cast<uintptr_t>(C) % 16 == 0) {
        // C quarters for the TMA epilogue: 128 rows x 128 columns of fp32, unswizzled ([col][128 rows])
        const cuuint64_t dims[2] = {static_cast<cuuint64_t>(m), static_cast<cuuint64_t>(n)};
        const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldc) * 4};
        const cuuint32_t box[2] = {128, 128}, estr[2] = {1, 1};
        args.tma_c = g_encode(&mc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, C, dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
        static const int tma_epilogue_knob = [] {  // TILEMUL_TC_TMA_EPILOGUE=0: A/B knob
            const char* env = std::getenv("TILEMUL_TC_TMA_EPILOGUE");
            return env ? std::atoi(env) : 1;
        }();
        args.tma_c &= tma_epilogue_knob;
        static const int tma_red_knob = [] {  // TILEMUL_TC_TMA_REDUCE: A/B knob
            const char* env = std::getenv("TILEMUL_TC_TMA_REDUCE");
            return env ? std::atoi(env) : 1;
        }();
        args.tma_red = args.tma_c && tma_red_knob;
    }
    // Cluster launch control: on for the persistent 256 x 256 kernel (its static stride let the clusters
    // drift apart: 16384^3 bf16 18.6 -> 12.0 GB of HBM reads, 1250 -> 1300 TF/s; tf32 681 -> 712), off for
    // the 256 x 512 kernel, which already runs one fresh cluster per tile (CLC measured neutral there:
    // 1353 vs 1345-1372 TF/s, the TMA epilogue then gated on the stage ring; profiles/ab_r02_tc_clc.json).
    static const int clc_knob = [] {  // TILEMUL_TC_CLC=0/1: A/B knob for both kernels
        const char* env = std::getenv("TILEMUL_TC_CLC");
        return env ? std::atoi(env) : -1;
    }();
    args.clc = clc_knob < 0 ? (NH == 1 ? 1 : 0) : clc_knob;
    if (args.clc) grid = 2 * ntasks;  // one cluster per tile; running clusters take the unstarted ones' tiles
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(grid & ~1));
    cfg.blockDim = dim3(G::THREADS);
    cfg.dynamicSmemBytes = G::SMEM;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_tc2<TF32, NH>, ma, mb, args, mc);
}

}  // namespace

cudaError_t launch_tc_pair(bool tf32, const void* A, int64_t lda, const void* B, int64_t ldb, float* C, int64_t ldc,
                           int64_t m, int64_t n, int64_t k, const Task* tasks, int ntasks, int grid,
                           cudaStream_t stream, bool wide) {
    if (ntasks <= 0) return cudaSuccess;
    if (wide)
        return tf32 ? launch_tc2_t<true, 2>(A, lda, B, ldb, C, ldc, m, n, k, tasks, ntasks, grid, stream)
                    : launch_tc2_t<false, 2>(A, lda, B, ldb, C, ldc, m, n, k, tasks, ntasks, grid, stream);
    return tf32 ? launch_tc2_t<true, 1>(A, lda, B, ldb, C, ldc, m, n, k, tasks, ntasks, grid, stream)
                : launch_tc2_t<false, 1>(A, lda, B, ldb, C, ldc, m, n, k, tasks, ntasks, grid, stream);
}

int tc2_smem_bytes(bool tf32, bool wide) {
    return wide ? (tf32 ? Tc2Geo<true, 2>::SMEM : Tc2Geo<false, 2>::SMEM)
                : (tf32 ? Tc2Geo<true, 1>::SMEM : Tc2Geo<false, 1>::SMEM);
}

cudaError_t launch_tc(bool tf32, const void* A, int64_t lda, const void* B, int64_t ldb, float* C, int64_t ldc,
                      int64_t m, int64_t n, int64_t k, const Task* tasks, int ntasks, int grid, cudaStream_t stream) {
    if (ntasks <= 0) return cudaSuccess;
    return tf32 ? launch_tc_t<true>(A, lda, B, ldb, C, ldc, m, n, k, tasks, ntasks, grid, stream)
                : launch_tc_t<false>(A, lda, B, ldb, C, ldc, m, n, k, tasks, ntasks, grid, stream);
}

cudaError_t launch_round(bool tf32, const double* x, void* y, int64_t count, cudaStream_t stream) {
    if (count <= 0) return cudaSuccess;
    const int blocks = static_cast<int>(std::min<int64_t>((count + 255) / 256, 148 * 32));
    if (tf32)
        k_round_tf32<<<blocks, 256, 0, stream>>>(x, static_cast<float*>(y), count);
    else
        k_round_bf16<<<blocks, 256, 0, stream>>>(x, static_cast<uint16_t*>(y), count);
    return cudaGetLastError();
}

int tc_smem_bytes(bool tf32) { return tf32 ? TcGeo<true>::SMEM : TcGeo<false>::SMEM; }

cudaError_t measure_tc_peak(bool tf32, int launches, bool sustained, double* tflops) {
    return tf32 ? measure_tc_peak_t<true>(launches, sustained, tflops)
                : measure_tc_peak_t<false>(launches, sustained, tflops);
}

}  // namespace gpu
}  // namespace mmm
