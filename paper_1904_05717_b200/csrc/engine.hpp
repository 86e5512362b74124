// Internal interface between the C ABI (capi.cpp), the lowering of a loop
// nest onto CTA tasks (lower.cpp) and the host-buffer pipelines
// (host_pipe.cpp). Not installed; callers use include/tilemul_b200.h.
#pragma once

#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/tilemul_b200.h"
#include "host/mmm.hpp"
#include "kernels/gpu.hpp"

namespace mmm {
namespace engine {

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Failure(kDevice, "", std::string(what) + ": " + cudaGetErrorString(e));
}

struct Schedule {
    gpu::Kernel kernel = gpu::kDmma128;
    bool vec16 = false;
    int grid = 1;
    int slices = 0;          // number of k-split tiles to reduce (fused)
    gpu::ReduceTile* reduce = nullptr;
    int32_t* cta_first = nullptr;  // stream-K: per-CTA task ranges
    bool blocked = false;
    int grid_fixed = 0;
    int regions = 0;         // progress counters (faithful)
    int counters = 0;        // split-k fix-up counters (DMMA kernels), self-resetting
    std::vector<gpu::Task> host_tasks;
    gpu::Task* tasks = nullptr;
    int32_t* progress = nullptr;
    double* work = nullptr;
    int64_t work_ld = 0, work_slice = 0;
    int device = -1;
    int tma_ok = -1;         // task list fits the TMA kernel's slab grid (-1 = not yet checked)
    int64_t slabs_per_cta = 0;  // k-slabs a CTA streams in one launch, on average (set with tma_ok)
    std::vector<int32_t> segments;  // TMA launches of a long task list: task index boundaries (whole rounds)
    int last_launches = 1;          // task-kernel launches the last launch_tasks issued
    ~Schedule() {
        if (tasks) cudaFree(tasks);
        if (progress) cudaFree(progress);
        if (work) cudaFree(work);
        if (reduce) cudaFree(reduce);
        if (cta_first) cudaFree(cta_first);
    }
};

struct Key {
    int schedule, kernel, split, ctas;
    bool vec16;
    int par;  // faithful: parallel loop (+1, 0 = auto)
    bool operator<(const Key& o) const {
        return std::tie(schedule, kernel, split, ctas, vec16, par) <
               std::tie(o.schedule, o.kernel, o.split, o.ctas, o.vec16, o.par);
    }
};

// Copy-engine-fed host pipeline (tm_execute_host): one persistent launch
// over the tasks of every (C column block, k-chunk) unit; the copy stream
// writes a per-unit flag after the unit's uploads, tasks wait on it, and
// the download of a block waits on its completion counter.
struct HostPipe {
    tm_exec_opts opts{};
    std::vector<i64> mcut, kcut, ncut;
    // One upload step: its pieces go up on the copy stream, then the step's
    // data flag is written; the tasks the step enables wait for that flag.
    struct Piece {
        char op;        // 'A', 'B' or 'C'
        i64 r0, rows;   // row range of the operand (A: m, B: k, C: m)
        i64 c0, cols;   // column range (A: k, B: n, C: n)
    };
    struct Step {
        std::vector<Piece> pieces;
        i64 i0 = 0, i1 = 0, j0 = 0, j1 = 0;  // the cell box the step enables: rows x columns ...
        int q = 0;                           // ... of k-chunk q
    };
    std::vector<Step> steps;                 // in issue order
    int done_rows = 1;                       // row blocks the downloads are cut into (1: whole column blocks)
    std::vector<int32_t> block_tasks;        // last-chunk tasks of each C cell (column block b, row block i): [b * done_rows + i]
    std::vector<std::pair<int, int>> cells;  // the C cells (b, i) in the order their last chunk is scheduled (download order)
    std::unique_ptr<Schedule> sched;
    int32_t* flags = nullptr;  // [steps] data-ready flags, then [column blocks x row blocks] done counters
    int regions = 0;
    ~HostPipe() {
        if (flags) cudaFree(flags);
    }
};

// The pipeline's cuts and upload steps for extents e (pure host logic, no device calls).
void pipe_order(const Extents& e, HostPipe& P);
int sm_count();
// Launch the schedule's task kernel: the TMA-fed DMMA variant when the
// options allow and the operands/task list fit it, else the cp.async one.
// Returns the staging used (TM_STAGING_*; 0 = kernel without variants).
int launch_tasks(Schedule& s, const gpu::Args& a, int64_t M, int64_t N, int64_t K, bool vec16, int32_t staging,
                 cudaStream_t stream, bool long_ok = false);
// `tma`: the operands allow TMA staging (16-byte aligned bases and leading
// dimensions, staging not forced to cp.async).
gpu::Kernel pick_kernel(const Nest& nest, const tm_exec_opts& o, bool tma);
// The host half of the lowering (no device calls): the task list of the
// nest for a kernel with tile_m x tile_n tiles on a machine with `slots`
// resident CTAs, plus what the device half allocates for it. Also the input
// of the GPU-mode I/O model (gpu_model.cpp), which runs without a GPU.
struct HostSchedule {
    std::vector<gpu::Task> tasks;
    bool blocked = false;            // stream-K: CTA c runs tasks first[c] .. first[c+1]-1
    int grid_fixed = 0;
    std::vector<int32_t> first;
    bool fixup = false;              // split tiles finished in-kernel (Task::fixup)
    int32_t slots = 0;               // split-k workspace slots
    int32_t counters = 0;            // fix-up counters
    std::vector<gpu::ReduceTile> red;  // tiles summed by the reduce launch (kernels without the fix-up)
    int regions = 0;                 // faithful: per-region progress counters
};
HostSchedule plan_tasks(const Nest& nest, const tm_exec_opts& o, gpu::Kernel kernel, int tile_m, int tile_n,
                        int slots);
// GPU-mode I/O model of the schedule the kernel runs (gpu_model.cpp):
// elements into the SMEM level per operand (exact over the task list) and
// bytes crossing the HBM boundary from a lockstep run of the task list
// through an LRU of the L2's capacity.
struct GpuIo {
    LevelFlow smem;
    int64_t hbm_read_bytes[3] = {0, 0, 0}, hbm_write_bytes[3] = {0, 0, 0};
    i64 tasks = 0, lockstep_slabs = 0;
    int grid = 0, kernel = 0, tile_m = 0, tile_n = 0;
};
// kernel < 0: the kernel execute() picks for `o`; else that kernel (the tensor-core path's tiles: for the
// SM-pair kernels one task per cluster, sms / 2 clusters in flight).
GpuIo gpu_io(const Nest& nest, const tm_exec_opts& o, int sms, int64_t l2_bytes, const double elem_bytes[3],
             int policy = 0, int kernel = -1);
// The tcgen05 kernel tm_execute_tc runs for `dtype` and the tile options (TM_DTYPE_*).
gpu::Kernel pick_tc_kernel(int dtype, const tm_exec_opts& o);
// Tile shape and occupancy of a kernel: measured on the device (query) or
// the compiled-in values (the model's CPU path).
gpu::KernelInfo kernel_tiles(gpu::Kernel kernel, bool query);
// Lowers the nest onto CTA tasks for `kernel` (schedule, split and fix-up
// per opts). upload = false builds the host task list only.
std::unique_ptr<Schedule> lower(const Nest& nest, const tm_exec_opts& o, gpu::Kernel kernel, cudaStream_t stream,
                                bool upload = true);
bool origins_even(const std::vector<gpu::Task>& T);

}  // namespace engine
}  // namespace mmm

// The opaque plan handle of the C ABI.
struct tm_plan {
    mmm::Nest nest;
    mmm::Hierarchy hier;
    std::map<mmm::engine::Key, std::unique_ptr<mmm::engine::Schedule>> schedules;
    std::mutex mu;
    std::mutex host_mu;  // one tm_execute_host at a time per plan (it owns the plan's staging buffers and streams)
    // device-operand launches share the schedules' scratch (task lists,
    // progress / fix-up counters, split-k slots): each launch's stream waits
    // for the previous launch of this plan (on any stream) to finish with it
    cudaEvent_t order = nullptr;
    // tm_execute_packed's column-major scratch, ordered across streams by packed_done
    std::mutex packed_mu;
    double *pA = nullptr, *pB = nullptr, *pC = nullptr;
    cudaEvent_t packed_done = nullptr;
    // host-buffer execution
    double *dA = nullptr, *dB = nullptr, *dC = nullptr;
    cudaStream_t host_stream = nullptr, copy_stream = nullptr, d2h_stream = nullptr;
    std::vector<cudaEvent_t> chunk_ready;
    // sub-plans of the host-buffer pipeline, keyed by (n, k) extent of one
    // (column block, k-chunk) piece: same family and blocksizes
    std::map<std::pair<int64_t, int64_t>, std::unique_ptr<tm_plan>> chunk_plans;
    std::unique_ptr<mmm::engine::HostPipe> pipe;
    int64_t last_tasks = 0;
    int32_t last_launches = 0, last_ctas = 0;
    int32_t last_staging = 0;
    ~tm_plan() {
        if (dA) cudaFree(dA);
        if (dB) cudaFree(dB);
        if (dC) cudaFree(dC);
        if (pA) cudaFree(pA);
        if (pB) cudaFree(pB);
        if (pC) cudaFree(pC);
        if (order) cudaEventDestroy(order);
        if (packed_done) cudaEventDestroy(packed_done);
        for (auto ev : chunk_ready) cudaEventDestroy(ev);
        if (host_stream) cudaStreamDestroy(host_stream);
        if (copy_stream) cudaStreamDestroy(copy_stream);
        if (d2h_stream) cudaStreamDestroy(d2h_stream);
    }
};

namespace mmm {
namespace engine {
// execute(): device operands, asynchronous on `stream` (tm_execute).
void run(tm_plan* plan, const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
         const tm_exec_opts* opts, cudaStream_t stream);
// execute() on host buffers: copies in, runs, copies C back (tm_execute_host).
void execute_host(tm_plan* plan, const double* A, const double* B, double* C, const tm_exec_opts* opts);
}  // namespace engine
}  // namespace mmm
