// Interface between the host lowering (capi.cpp) and the sm_100a kernels
// (dgemm_sm100.cu). A launch is a list of CTA tasks processed by a
// persistent grid in list order (task t runs on CTA t mod grid).
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace mmm {
namespace gpu {

// One CTA task: C(i0:i0+m, j0:j0+n) += A(i0:, p0:p0+k) · B(p0:, j0:j0+n),
// accumulated in ascending k from the incoming C value (the reference's cell,
// exec.hpp:35-46, at CTA granularity).
struct Task {
    int32_t i0, j0, p0;
    int32_t m, n, k;
    int32_t tile;   // progress counter of this C region (-1: no ordering needed)
    int32_t seq;    // chunks of this region that must finish first
    int32_t slice;  // -1: read/write C; s >= 0: split-k partial into workspace slice s
    int32_t from_c; // slice tasks: 1 = start from C's value, 0 = start from zero
    // In-kernel split-k fix-up (DMMA kernels; replaces the reduce launch):
    //   0 — none (slice semantics above);
    //   1 — contributor: the part's partial goes to workspace slot `slice`,
    //       then counter (-2 - tile) is incremented (release);
    //   2 — owner (the part that starts from C): after its k loop it waits
    //       until counter (-2 - tile) reaches `seq`, adds slots slice ..
    //       slice+seq-1 in slot order, writes C and resets the counter to 0.
    //   (tile < 0 keeps fix-up tasks out of the faithful-order protocol.)
    int32_t fixup;
    // Copy-engine-fed pipeline (tm_execute_host): ready = 1 + index of the
    // data flag the task waits for before touching A/B/C (0 = none); done =
    // 1 + index of the counter it increments once its C tile is final
    // (0 = none). Both are read only at task boundaries.
    int32_t ready;
    int32_t done;
};

struct Args {
    const double* A;
    int64_t lda;
    const double* B;
    int64_t ldb;
    double* C;
    int64_t ldc;
    const Task* tasks;
    int32_t ntasks;
    int32_t* progress;   // one counter per ordered region (faithful schedule)
    double* work;        // split-k partials: one compact slot per (tile, k-part), tile-local, ld = work_ld
    int64_t work_ld;
    int64_t work_slice;  // elements per slot
    const int32_t* cta_first;  // blocked assignment: CTA c runs tasks [cta_first[c], cta_first[c+1]);
                               // nullptr = strided (task t on CTA t mod grid)
    const int32_t* ready;      // data flags written by the copy stream (Task::ready), or nullptr
    int32_t* done;             // per-block completion counters (Task::done), or nullptr
    int32_t prefetch_c = 0;    // TMA kernels: warm L2 with each task's C tile when the producer reaches it
    int32_t pdl_trigger = 0;   // TMA kernels: griddepcontrol.launch_dependents at each CTA's last task
    int32_t zero = 0;          // always 0, but only known at run time: ties a stage's release to its last fragment loads
};

// One k-split C tile: its partials live in slots slot0 .. slot0+nslots-1 and
// are summed in slot order (slot0 started from C's incoming value).
struct ReduceTile {
    int32_t i0, j0, m, n;
    int32_t slot0, nslots;
};

enum Kernel : int {
    kDmma128 = 0,   // 128x128 C tile, 16 warps of 32x32 (4 per SM sub-partition), mma.sync m8n8k4 f64
                    // (its TMA variant adds a producer warpgroup: 640 threads)
    kDmma64 = 1,    // 64x64 C tile, 4 warps of 32x32
    kFma64 = 2,     // 64x64, DFMA chain per entry (bit-exact vs sequential fma)
    kExact64 = 3,   // 64x64, DMUL + DADD per step (bit-exact vs the reference)
    kFma128 = 4,    // 128x128, 8x8 per thread DFMA chain
    kDmma128x64 = 5,  // 128x64 C tile, 4 warps of 64x32, two CTAs per SM (prologue/epilogue overlap)
    kKernelCount = 6,
    kTcBf16 = 100,    // tcgen05 BF16 inputs, fp32 TMEM accumulate, 128x256 tile (tc_gemm_sm100.cu)
    kTcTf32 = 101,    // tcgen05 TF32 inputs
    kTc2Bf16 = 102,   // tcgen05.mma.cta_group::2: 2-CTA cluster, 256x256 tile per pair
    kTc2Tf32 = 103,
    kTc2wBf16 = 104,  // 2-CTA cluster, 256x512 tile per pair (25 % fewer L2->SMEM bytes per flop)
    kTc2wTf32 = 105
};

struct KernelInfo {
    int tile_m, tile_n, threads;
    int smem_bytes;
    int ctas_per_sm;  // occupancy measured at first use
};

// Launch `kernel` over args.tasks with `grid` persistent CTAs. vec16 selects
// 16-byte cp.async staging (all task origins even, ld even, 16B-aligned bases).
cudaError_t launch(Kernel kernel, bool vec16, const Args& args, int grid, cudaStream_t stream);
// TMA-fed variant of a DMMA kernel (k_dmma_tma): A (M x K) and B (K x N) are
// read through tensor maps built per launch, so the task list must not need
// a k limit inside a slab: every task's k range is a multiple of tma_bk() or
// ends at K (out-of-range rows/columns are zero-filled by the TMA unit).
// cudaErrorNotSupported: no TMA variant, unaligned operands, or lower
// occupancy than the cp.async kernel the grid was sized for.
// pdl: programmatic dependent launch after the previous kernel on the stream (a later segment of the same
// task list): its CTAs may start as the previous launch's CTAs retire (they trigger at their last task).
cudaError_t launch_tma(Kernel kernel, const Args& args, int64_t M, int64_t N, int64_t K, int grid,
                       cudaStream_t stream, bool pdl = false);
int tma_bk(Kernel kernel);  // k-slab depth of the TMA variant (0 = none)
// cuTensorMapEncodeTiled from the driver (nullptr if unavailable).
void* tensor_map_encoder();
// Occupancy-derived info (queries the device on first call).
cudaError_t kernel_info(Kernel kernel, KernelInfo* info);
// C(tile) = slot0 + slot1 + ... in slot order for every listed tile
// (deterministic split-k reduction).
cudaError_t launch_reduce_tiles(double* C, int64_t ldc, const double* work, int64_t work_ld, int64_t work_slice,
                                const ReduceTile* tiles, int ntiles, cudaStream_t stream);
// Peak tcgen05 MMA rate of the current device (M=128 x N=256, BF16 or TF32
// inputs, fp32 accumulate), best of `launches` launches of ~5 ms (burst) or
// ~200 ms (sustained, power-capped), TFLOP/s.
cudaError_t measure_tc_peak(bool tf32, int launches, bool sustained, double* tflops);
// Sustained FP64 DMMA rate of this device (TFLOP/s) over `launches` probe launches.
cudaError_t measure_fp64_peak(int launches, double* tflops);
// tcgen05 BF16/TF32-input GEMM over a task list (C fp32, column-major).
cudaError_t launch_tc(bool tf32, const void* A, int64_t lda, const void* B, int64_t ldb, float* C, int64_t ldc,
                      int64_t m, int64_t n, int64_t k, const Task* tasks, int ntasks, int grid, cudaStream_t stream);
// fp64 -> bf16 (RNE) or fp64 -> tf32-valued fp32 (RNE to 11 significant bits).
cudaError_t launch_round(bool tf32, const double* x, void* y, int64_t count, cudaStream_t stream);
int tc_smem_bytes(bool tf32);
// Same contract, 2-SM pair kernel: tasks are 256 x 256 tiles (wide: 256 x
// 512, one TMEM accumulator of 512 columns), grid even (clusters of 2).
cudaError_t launch_tc_pair(bool tf32, const void* A, int64_t lda, const void* B, int64_t ldb, float* C, int64_t ldc,
                           int64_t m, int64_t n, int64_t k, const Task* tasks, int ntasks, int grid,
                           cudaStream_t stream, bool wide = false);
int tc2_smem_bytes(bool tf32, bool wide = false);
// A hierarchical layout for the relayout kernel (<= kMaxCuts partition steps).
struct LayoutDev {
    static constexpr int kMaxCuts = 24;
    int64_t rows, cols;
    int32_t ncuts;
    uint8_t on_rows[kMaxCuts];
    int64_t size[kMaxCuts];
};
// pack: column-major src -> blocked dst; unpack: blocked src -> column-major dst.
cudaError_t launch_relayout(const double* src, double* dst, const LayoutDev& L, bool pack, cudaStream_t stream);
cudaError_t launch_fill_block(double* x, int64_t rows, int64_t cols, int64_t ld, uint64_t seed, int64_t row0,
                              int64_t col0, int64_t gld, cudaStream_t stream);
cudaError_t launch_fill(double* x, int64_t count, uint64_t seed, uint64_t offset, cudaStream_t stream);

}  // namespace gpu
}  // namespace mmm
