// C ABI (include/tilemul_b200.h) over the host library and the sm_100a task
// kernels, plus the lowering of a loop nest onto CTA tasks.
//
// Lowering (the blocked-loop driver, reference plan.hpp:61-84 +
// exec.hpp:94-138, re-targeted): a task is one C region x k range run by one
// CTA with its accumulators in registers. Two schedules:
//   fused    — every k loop of the nest is sunk below its m/n loops, so each
//              register-level C block is visited once, in the order of its
//              first appearance in the nest (the m/n loops above it become the
//              CTA raster: the L2-level plan sets which tiles share a wave).
//              Optional split-k adds a deterministic slice reduction.
//   faithful — one task per nest cell, in nest order; cells of the same C
//              block run in ascending k (per-region progress counters), so
//              the C block round-trips to memory per cell exactly as the
//              reference's micro-kernel does.
// Either way every C entry is accumulated in ascending k from its incoming
// value, which is what makes the result independent of the schedule.
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/tilemul_b200.h"
#include "host/cachesim.hpp"
#include "host/mmm.hpp"
#include "kernels/gpu.hpp"

using namespace mmm;

namespace {

thread_local std::string g_error;
thread_local std::string g_rules;

void record(const Failure& f) {
    g_error = f.what();
    g_rules.clear();
    for (const auto& v : f.issues)
        g_rules += v.rule + ":" + std::to_string(v.level) + ":" + std::to_string(v.lhs) + ":" + std::to_string(v.rhs) + "\n";
    if (f.issues.empty() && !f.rule.empty()) g_rules = f.rule + ":-1:0:0\n";
}

template <typename F>
int guard(F&& f) {
    try {
        g_error.clear();
        g_rules.clear();
        f();
        return kOk;
    } catch (const Failure& e) {
        record(e);
        return e.status;
    } catch (const std::exception& e) {
        g_error = e.what();
        return kUsage;
    }
}

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Failure(kDevice, "", std::string(what) + ": " + cudaGetErrorString(e));
}

Hierarchy hierarchy_from(const tm_level* levels, int n) {
    if (n < 1 || levels == nullptr) fail_usage("hierarchy needs at least one level");
    std::vector<MemLevel> lv;
    for (int i = 0; i < n; ++i)
        lv.push_back({levels[i].capacity_elements, levels[i].granularity < 1 ? 1 : levels[i].granularity,
                      levels[i].inclusive != 0, levels[i].write_allocate != 0, levels[i].write_back != 0});
    return make_hierarchy(std::move(lv));
}

Blocks blocks_from(const tm_blocksize* bs, int n) {
    Blocks b;
    for (int i = 0; i < n; ++i) b.put(bs[i].level, dim_of_char(bs[i].dim), bs[i].value);
    return b;
}

void put_tiers(const Family& f, tm_tier* tiers, int cap, int* count) {
    if (count) *count = static_cast<int>(f.tiers.size());
    if (tiers == nullptr) return;
    if (static_cast<int>(f.tiers.size()) > cap) fail_usage("tier buffer too small");
    for (std::size_t i = 0; i < f.tiers.size(); ++i)
        tiers[i] = tm_tier{f.tiers[i].level, opnd_char(f.tiers[i].resident), dim_char(f.tiers[i].outer),
                           dim_char(f.tiers[i].inner)};
}

void put_name(const std::string& s, char* out, int cap) {
    if (out == nullptr) return;
    if (static_cast<int>(s.size()) + 1 > cap) fail_usage("name buffer too small");
    std::memcpy(out, s.c_str(), s.size() + 1);
}

// ------------------------------------------------------------- lowering

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
    bool operator<(const Key& o) const {
        return std::tie(schedule, kernel, split, ctas, vec16) < std::tie(o.schedule, o.kernel, o.split, o.ctas, o.vec16);
    }
};

}  // namespace

// Copy-engine-fed host pipeline (tm_execute_host): one persistent launch
// over the tasks of every (C column block, k-chunk) unit; the copy stream
// writes a per-unit flag after the unit's uploads, tasks wait on it, and
// the download of a block waits on its completion counter.
struct HostPipe {
    tm_exec_opts opts{};
    std::vector<i64> kcut, ncut;
    std::vector<std::pair<int, int>> units;  // (block, chunk) in issue order
    std::vector<int32_t> block_tasks;        // tasks of each block's last unit
    std::unique_ptr<Schedule> sched;
    int32_t* flags = nullptr;  // [units] data-ready flags, then [blocks] done counters
    int regions = 0;
    ~HostPipe() {
        if (flags) cudaFree(flags);
    }
};

struct tm_plan {
    Nest nest;
    Hierarchy hier;
    std::map<Key, std::unique_ptr<Schedule>> schedules;
    std::mutex mu;
    std::mutex host_mu;  // one tm_execute_host at a time per plan (it owns the plan's staging buffers and streams)
    // host-buffer execution
    double *dA = nullptr, *dB = nullptr, *dC = nullptr;
    cudaStream_t host_stream = nullptr, copy_stream = nullptr, d2h_stream = nullptr;
    std::vector<cudaEvent_t> chunk_ready;
    // sub-plans of the host-buffer pipeline, keyed by (n, k) extent of one
    // (column block, k-chunk) piece: same family and blocksizes
    std::map<std::pair<int64_t, int64_t>, std::unique_ptr<tm_plan>> chunk_plans;
    std::unique_ptr<HostPipe> pipe;
    int64_t last_tasks = 0;
    int32_t last_launches = 0, last_ctas = 0;
    ~tm_plan() {
        if (dA) cudaFree(dA);
        if (dB) cudaFree(dB);
        if (dC) cudaFree(dC);
        for (auto ev : chunk_ready) cudaEventDestroy(ev);
        if (host_stream) cudaStreamDestroy(host_stream);
        if (copy_stream) cudaStreamDestroy(copy_stream);
        if (d2h_stream) cudaStreamDestroy(d2h_stream);
    }
};

namespace {

int sm_count() {
    int dev = 0, sms = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "cudaDeviceGetAttribute");
    return sms;
}

gpu::Kernel pick_kernel(const Nest& nest, const tm_exec_opts& o) {
    const bool small_tile = o.tile == 64 || (o.tile == 0 && (nest.m_r < 128 || nest.n_r < 128));
    if (o.tile != 0 && o.tile != 64 && o.tile != 128) fail_usage("tile must be 0, 64 or 128");
    const int tn = o.tile_n == 0 ? o.tile : o.tile_n;
    if (o.tile_n != 0 && !((o.tile == 128 && (tn == 64 || tn == 128)) || (o.tile == 64 && tn == 64)))
        fail_usage("tile x tile_n must be 128x128, 128x64 or 64x64");
    switch (o.numerics) {
        case TM_NUMERICS_DMMA:
            if (o.tile == 128 && tn == 64) return gpu::kDmma128x64;
            // short k: every task is mostly C load/store; two CTAs per SM
            // (128 x 64 tiles) hide one CTA's C traffic behind the other's DMMAs
            if (o.tile == 0 && !small_tile && nest.ext.k <= 512 && o.schedule == TM_SCHEDULE_FUSED)
                return gpu::kDmma128x64;
            return small_tile ? gpu::kDmma64 : gpu::kDmma128;
        case TM_NUMERICS_FMA:
            if (tn == 64 && o.tile == 128) fail_usage("fma numerics run on square tiles");
            return small_tile ? gpu::kFma64 : gpu::kFma128;
        case TM_NUMERICS_EXACT:
            if (o.tile == 128) fail_usage("exact numerics run on the 64x64 tile only");
            return gpu::kExact64;
        default: fail_usage("unknown numerics");
    }
}

// Splits one C region into kernel tiles, n outer / m inner (the register
// plan's own loop order, C0 = n then m).
template <typename F>
void for_each_subtile(i64 i0, i64 m, i64 j0, i64 n, int tm, int tn, F&& f) {
    for (i64 jj = 0; jj < n; jj += tn)
        for (i64 ii = 0; ii < m; ii += tm) f(i0 + ii, std::min<i64>(tm, m - ii), j0 + jj, std::min<i64>(tn, n - jj));
}

void check_i32(i64 v, const char* what) {
    if (v > INT32_MAX) fail_usage(std::string(what) + " exceeds the 32-bit task range");
}

// Workspace slots and self-resetting counters of the in-kernel fix-up.
void alloc_fixup(Schedule& s, const gpu::KernelInfo& info, int32_t slots, int32_t counters, cudaStream_t stream) {
    if (counters == 0) return;
    s.work_ld = info.tile_m;
    s.work_slice = static_cast<i64>(info.tile_m) * info.tile_n;
    cuda_check(cudaMalloc(&s.work, sizeof(double) * static_cast<std::size_t>(s.work_slice) * slots),
               "cudaMalloc(split-k workspace)");
    cuda_check(cudaMalloc(&s.progress, sizeof(int32_t) * static_cast<std::size_t>(counters)), "cudaMalloc(fix-up counters)");
    cuda_check(cudaMemsetAsync(s.progress, 0, sizeof(int32_t) * static_cast<std::size_t>(counters), stream),
               "zero fix-up counters");
    s.counters = counters;
}

std::unique_ptr<Schedule> lower(const Nest& nest, const tm_exec_opts& o, gpu::Kernel kernel, cudaStream_t stream,
                                bool upload = true) {
    auto s = std::make_unique<Schedule>();
    s->kernel = kernel;
    gpu::KernelInfo info{};
    const bool pair = kernel == gpu::kTc2Bf16 || kernel == gpu::kTc2Tf32;
    if (kernel == gpu::kTcBf16 || kernel == gpu::kTcTf32)
        info = gpu::KernelInfo{128, 256, 256, gpu::tc_smem_bytes(kernel == gpu::kTcTf32), 1};
    else if (pair)
        info = gpu::KernelInfo{256, 256, 256, gpu::tc2_smem_bytes(kernel == gpu::kTc2Tf32), 1};
    else
        cuda_check(gpu::kernel_info(kernel, &info), "kernel_info");
    const int slots = sm_count() * std::max(1, info.ctas_per_sm);
    const Extents& e = nest.ext;
    check_i32(e.m, "m");
    check_i32(e.n, "n");
    check_i32(e.k, "k");
    auto& T = s->host_tasks;

    if (o.schedule == TM_SCHEDULE_FUSED) {
        // First-appearance order of the register-level C blocks = the walk of
        // the nest with its k loops removed.
        Nest mn = nest;
        mn.loops.clear();
        for (const auto& L : nest.loops)
            if (L.dim != kK) mn.loops.push_back(L);
        std::vector<std::array<i64, 4>> tiles;
        mn.walk([&](const Cell& c) {
            for_each_subtile(c.i0, c.m, c.j0, c.n, info.tile_m, info.tile_n,
                             [&](i64 i0, i64 m, i64 j0, i64 n) { tiles.push_back({i0, m, j0, n}); });
        });
        const bool dmma = o.numerics == TM_NUMERICS_DMMA && kernel < gpu::kTcBf16;
        const i64 ntiles = static_cast<i64>(tiles.size());
        // Stream-K (split_k == -1, or auto when C fills only a few waves with
        // a ragged last one): every CTA gets an equal contiguous range of
        // (tile, 32-deep k-slab) iterations; a tile cut by a range boundary
        // becomes several k-parts reduced in fixed slot order afterwards.
        // Balances the machine exactly and staggers the tile boundaries
        // (C loads/stores) of different CTAs in time.
        const bool ragged = ntiles % slots != 0 && ntiles < 8 * slots && ntiles * 2 > slots;
        if (dmma && (o.split_k == -1 || (o.split_k == 0 && ragged && e.k >= 2048))) {
            const i64 slab = 32, nks = cdiv(e.k, slab), U = ntiles * nks;
            const int G = static_cast<int>(std::min<i64>(slots, U));
            std::vector<std::vector<std::array<i64, 2>>> pieces(tiles.size());  // per tile: (slab_lo, slab_hi)
            std::vector<std::vector<std::pair<i64, i64>>> per_cta(static_cast<std::size_t>(G));  // (tile, piece#)
            for (int c = 0; c < G; ++c) {
                const i64 lo = U * c / G, hi = U * (c + 1) / G;
                for (i64 u = lo; u < hi;) {
                    const i64 tile = u / nks, end = std::min(hi, (tile + 1) * nks);
                    auto& pc = pieces[static_cast<std::size_t>(tile)];
                    per_cta[static_cast<std::size_t>(c)].push_back({tile, static_cast<i64>(pc.size())});
                    pc.push_back({u - tile * nks, end - tile * nks});
                    u = end;
                }
            }
            // A cut tile is finished inside the kernel: its head piece (k from
            // 0, from C) is the owner and runs last in its CTA's range; the
            // later pieces run first in the following CTAs' ranges and leave
            // partials in slots slot0 .. slot0+pieces-2 (Task::fixup).
            // Kernels built without the fix-up keep one slot per piece and a
            // fixed-order reduce launch afterwards.
            const bool fixk = kernel == gpu::kDmma128 || kernel == gpu::kDmma64;
            std::vector<int32_t> slot0(tiles.size(), -1), counter(tiles.size(), -1);
            std::vector<gpu::ReduceTile> red;
            int32_t next_slot = 0, ncounters = 0;
            for (std::size_t t = 0; t < tiles.size(); ++t)
                if (pieces[t].size() > 1) {
                    const int32_t np = static_cast<int32_t>(pieces[t].size());
                    slot0[t] = next_slot;
                    counter[t] = ncounters++;
                    if (!fixk)
                        red.push_back(gpu::ReduceTile{static_cast<int32_t>(tiles[t][0]), static_cast<int32_t>(tiles[t][2]),
                                                      static_cast<int32_t>(tiles[t][1]), static_cast<int32_t>(tiles[t][3]),
                                                      next_slot, np});
                    next_slot += fixk ? np - 1 : np;
                }
            std::vector<int32_t> first(static_cast<std::size_t>(G) + 1, 0);
            for (int c = 0; c < G; ++c) {
                first[static_cast<std::size_t>(c)] = static_cast<int32_t>(T.size());
                for (auto [tile, pi] : per_cta[static_cast<std::size_t>(c)]) {
                    const auto& t = tiles[static_cast<std::size_t>(tile)];
                    const auto& pr = pieces[static_cast<std::size_t>(tile)][static_cast<std::size_t>(pi)];
                    gpu::Task tk{};
                    tk.i0 = static_cast<int32_t>(t[0]);
                    tk.m = static_cast<int32_t>(t[1]);
                    tk.j0 = static_cast<int32_t>(t[2]);
                    tk.n = static_cast<int32_t>(t[3]);
                    tk.p0 = static_cast<int32_t>(pr[0] * slab);
                    tk.k = static_cast<int32_t>(std::min(pr[1] * slab, e.k) - pr[0] * slab);
                    const int32_t s0 = slot0[static_cast<std::size_t>(tile)];
                    const int32_t np = static_cast<int32_t>(pieces[static_cast<std::size_t>(tile)].size());
                    tk.tile = s0 < 0 ? -1 : -2 - counter[static_cast<std::size_t>(tile)];
                    tk.from_c = pr[0] == 0 ? 1 : 0;
                    if (s0 < 0) {
                        tk.seq = 0;
                        tk.slice = -1;
                        tk.fixup = 0;
                    } else if (!fixk) {  // every piece into its slot; the reduce launch sums them
                        tk.tile = -1;
                        tk.seq = 0;
                        tk.slice = s0 + static_cast<int32_t>(pi);
                        tk.fixup = 0;
                    } else if (pi == 0) {  // owner
                        tk.seq = np - 1;
                        tk.slice = s0;
                        tk.fixup = 2;
                    } else {
                        tk.seq = 0;
                        tk.slice = s0 + static_cast<int32_t>(pi) - 1;
                        tk.fixup = 1;
                    }
                    T.push_back(tk);
                }
            }
            first[static_cast<std::size_t>(G)] = static_cast<int32_t>(T.size());
            s->blocked = true;
            s->grid_fixed = G;
            cuda_check(cudaMalloc(&s->cta_first, sizeof(int32_t) * first.size()), "cudaMalloc(cta ranges)");
            cuda_check(cudaMemcpyAsync(s->cta_first, first.data(), sizeof(int32_t) * first.size(),
                                       cudaMemcpyHostToDevice, stream),
                       "upload cta ranges");
            if (fixk) {
                alloc_fixup(*s, info, next_slot, ncounters, stream);
            } else if (!red.empty()) {
                s->slices = static_cast<int>(red.size());
                s->work_ld = info.tile_m;
                s->work_slice = static_cast<i64>(info.tile_m) * info.tile_n;
                cuda_check(cudaMalloc(&s->work, sizeof(double) * static_cast<std::size_t>(s->work_slice) * next_slot),
                           "cudaMalloc(stream-k workspace)");
                cuda_check(cudaMalloc(&s->reduce, sizeof(gpu::ReduceTile) * red.size()), "cudaMalloc(reduce list)");
                cuda_check(cudaMemcpyAsync(s->reduce, red.data(), sizeof(gpu::ReduceTile) * red.size(),
                                           cudaMemcpyHostToDevice, stream),
                           "upload reduce list");
            }
            cuda_check(cudaStreamSynchronize(stream), "upload stream-k lists (sync)");
        } else {
        // k parts per tile. split_k > 1: every tile; split_k == 0 (auto):
        // every tile when C has too few tiles to fill the machine, otherwise
        // only the tiles of the last, partial wave (a "tail split": the full
        // waves run unsplit, the tail's parts fill the idle SMs).
        const i64 slab = (kernel >= gpu::kTcBf16) ? 64 : 32;
        const i64 nt = static_cast<i64>(tiles.size());
        const i64 max_parts = std::max<i64>(1, std::min<i64>(8, e.k / (16 * slab)));
        std::vector<int> parts(tiles.size(), 1);
        if (o.split_k > 1) {
            std::fill(parts.begin(), parts.end(), static_cast<int>(std::min<i64>(o.split_k, cdiv(e.k, slab))));
        } else if (o.split_k == 0 && nt > 0 && o.numerics == TM_NUMERICS_DMMA) {
            // (auto-splitting changes the summation order, so it is only
            // applied where results are bound-checked, never for the
            // bit-reproducible fma/exact numerics)
            if (nt * 2 <= slots) {
                const int sp = static_cast<int>(std::min<i64>(slots / nt, std::max<i64>(1, e.k / 1024)));
                std::fill(parts.begin(), parts.end(), std::max(1, std::min<int>(sp, static_cast<int>(cdiv(e.k, slab)))));
            } else {
                const i64 full = (nt / slots) * slots, rem = nt - full;
                // tail time in tile units: ceil(rem*S/slots)/S, plus a small
                // charge per extra part for its partial store and reduction
                double best = 1.0;
                int bestS = 1;
                for (i64 S = 2; S <= max_parts && rem > 0; ++S) {
                    const double cost = static_cast<double>(cdiv(rem * S, slots)) / static_cast<double>(S) +
                                        0.03 * static_cast<double>(S - 1);
                    if (cost < best - 1e-9) {
                        best = cost;
                        bestS = static_cast<int>(S);
                    }
                }
                for (i64 i = full; i < nt; ++i) parts[static_cast<std::size_t>(i)] = bestS;
            }
        }
        // DMMA kernels finish split tiles in-kernel (Task::fixup): the owner
        // part (k from 0, from C) is listed after its contributors, so every
        // wait points at an earlier task of the persistent grid (no cycle).
        // (the 128x64 short-k kernel is built without the fix-up: its register
        // budget is two CTAs per SM; its few tail splits use the reduce launch)
        const bool fix = kernel == gpu::kDmma128 || kernel == gpu::kDmma64;
        int32_t next_slot = 0, ncounters = 0;
        std::vector<gpu::ReduceTile> red;
        for (std::size_t ti = 0; ti < tiles.size(); ++ti) {
            const auto& t = tiles[ti];
            const i64 per = cdiv(cdiv(e.k, parts[ti]), slab) * slab;
            const int used = static_cast<int>(cdiv(e.k, per));
            gpu::Task tk{};
            tk.i0 = static_cast<int32_t>(t[0]);
            tk.m = static_cast<int32_t>(t[1]);
            tk.j0 = static_cast<int32_t>(t[2]);
            tk.n = static_cast<int32_t>(t[3]);
            tk.tile = -1;
            tk.seq = 0;
            if (used == 1) {
                tk.p0 = 0;
                tk.k = static_cast<int32_t>(e.k);
                tk.slice = -1;
                tk.from_c = 1;
                T.push_back(tk);
                continue;
            }
            if (fix) {
                const int32_t ctr = ncounters++;
                for (int q = 1; q <= used; ++q) {
                    const int part = q % used;  // contributors 1..used-1, then the owner (part 0)
                    const i64 p0 = part * per;
                    tk.p0 = static_cast<int32_t>(p0);
                    tk.k = static_cast<int32_t>(std::min(per, e.k - p0));
                    tk.tile = -2 - ctr;
                    tk.from_c = part == 0 ? 1 : 0;
                    tk.fixup = part == 0 ? 2 : 1;
                    tk.seq = part == 0 ? used - 1 : 0;
                    tk.slice = part == 0 ? next_slot : next_slot + part - 1;
                    T.push_back(tk);
                }
                next_slot += used - 1;
                continue;
            }
            red.push_back(gpu::ReduceTile{tk.i0, tk.j0, tk.m, tk.n, next_slot, used});
            for (int q = 0; q < used; ++q) {
                const i64 p0 = q * per;
                tk.p0 = static_cast<int32_t>(p0);
                tk.k = static_cast<int32_t>(std::min(per, e.k - p0));
                tk.slice = next_slot + q;
                tk.from_c = q == 0 ? 1 : 0;
                T.push_back(tk);
            }
            next_slot += used;
        }
        if (fix) alloc_fixup(*s, info, next_slot, ncounters, stream);
        s->slices = static_cast<int>(red.size());
        if (!red.empty()) {
            s->work_ld = info.tile_m;
            s->work_slice = static_cast<i64>(info.tile_m) * info.tile_n;
            cuda_check(cudaMalloc(&s->work, sizeof(double) * static_cast<std::size_t>(s->work_slice) * next_slot),
                       "cudaMalloc(split-k workspace)");
            cuda_check(cudaMalloc(&s->reduce, sizeof(gpu::ReduceTile) * red.size()), "cudaMalloc(reduce list)");
            cuda_check(cudaMemcpyAsync(s->reduce, red.data(), sizeof(gpu::ReduceTile) * red.size(),
                                       cudaMemcpyHostToDevice, stream),
                       "upload reduce list");
            cuda_check(cudaStreamSynchronize(stream), "upload reduce list (sync)");
        }
        }  // uniform / tail split
    } else if (o.schedule == TM_SCHEDULE_FAITHFUL) {
        const i64 cells = nest.cells();
        if (cells > 64LL * 1000 * 1000) fail_usage("faithful schedule limited to 64M cells; use the fused schedule");
        std::unordered_map<i64, std::pair<int32_t, int32_t>> regions;  // key -> (id, next seq)
        nest.walk([&](const Cell& c) {
            for_each_subtile(c.i0, c.m, c.j0, c.n, info.tile_m, info.tile_n, [&](i64 i0, i64 m, i64 j0, i64 n) {
                const i64 key = i0 * (e.n + 1) + j0;
                auto it = regions.find(key);
                if (it == regions.end()) it = regions.emplace(key, std::make_pair(static_cast<int32_t>(regions.size()), 0)).first;
                gpu::Task tk{};
                tk.i0 = static_cast<int32_t>(i0);
                tk.m = static_cast<int32_t>(m);
                tk.j0 = static_cast<int32_t>(j0);
                tk.n = static_cast<int32_t>(n);
                tk.p0 = static_cast<int32_t>(c.p0);
                tk.k = static_cast<int32_t>(c.k);
                tk.tile = it->second.first;
                tk.seq = it->second.second++;
                tk.slice = -1;
                tk.from_c = 1;
                T.push_back(tk);
            });
        });
        s->regions = static_cast<int>(regions.size());
        cuda_check(cudaMalloc(&s->progress, sizeof(int32_t) * static_cast<std::size_t>(std::max(1, s->regions))),
                   "cudaMalloc(progress)");
    } else {
        fail_usage("unknown schedule");
    }
    if (T.size() > static_cast<std::size_t>(INT32_MAX)) fail_usage("too many tasks");
    if (!upload) return s;  // host task list only (callers that splice task lists)
    // Persistent grid: every CTA must be co-resident for the faithful
    // schedule's waits to make progress.
    int grid = o.ctas > 0 ? std::min(o.ctas, slots) : slots;
    s->grid = std::max(1, std::min<int>(grid, static_cast<int>(T.size())));
    if (pair) s->grid = 2 * std::max(1, std::min<int>(slots / 2, static_cast<int>(T.size())));  // clusters of 2
    if (s->blocked) s->grid = s->grid_fixed;  // one task range per CTA
    cuda_check(cudaGetDevice(&s->device), "cudaGetDevice");
    cuda_check(cudaMalloc(&s->tasks, sizeof(gpu::Task) * std::max<std::size_t>(1, T.size())), "cudaMalloc(tasks)");
    // Stream-ordered upload, completed before the schedule is used: a plain
    // cudaMemcpy from pageable memory may return before the DMA lands, and the
    // launch streams are non-blocking (no ordering with the legacy stream).
    cuda_check(cudaMemcpyAsync(s->tasks, T.data(), sizeof(gpu::Task) * T.size(), cudaMemcpyHostToDevice, stream),
               "upload tasks");
    cuda_check(cudaStreamSynchronize(stream), "upload tasks (sync)");
    return s;
}

bool origins_even(const std::vector<gpu::Task>& T) {
    for (const auto& t : T)
        if ((t.i0 | t.p0) & 1) return false;
    return true;
}

void run(tm_plan* plan, const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
         const tm_exec_opts* opts, cudaStream_t stream) {
    const Extents& e = plan->nest.ext;
    if (!A || !B || !C) fail_usage("null operand pointer");
    if (lda < e.m || ldb < e.k || ldc < e.m) fail_usage("leading dimension smaller than the operand's row count");
    tm_exec_opts o{};
    if (opts) o = *opts;
    const gpu::Kernel kernel = pick_kernel(plan->nest, o);
    std::lock_guard<std::mutex> lk(plan->mu);
    Key key{o.schedule, kernel, o.schedule == TM_SCHEDULE_FUSED ? o.split_k : 0, o.ctas, false};
    auto& slot = plan->schedules[key];
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    if (!slot || slot->device != dev) slot = lower(plan->nest, o, kernel, stream);
    Schedule& s = *slot;
    const bool vec16 = (lda % 2 == 0) && (ldb % 2 == 0) && (reinterpret_cast<uintptr_t>(A) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(B) % 16 == 0) && origins_even(s.host_tasks);
    if (s.regions > 0)
        cuda_check(cudaMemsetAsync(s.progress, 0, sizeof(int32_t) * static_cast<std::size_t>(s.regions), stream),
                   "reset progress");
    gpu::Args a{A, lda, B, ldb, C, ldc, s.tasks, static_cast<int32_t>(s.host_tasks.size()), s.progress, s.work,
                s.work_ld, s.work_slice, s.blocked ? s.cta_first : nullptr};
    cuda_check(gpu::launch(s.kernel, vec16, a, s.grid, stream), "task kernel launch");
    int launches = 1;
    if (s.slices > 0) {
        cuda_check(gpu::launch_reduce_tiles(C, ldc, s.work, s.work_ld, s.work_slice, s.reduce, s.slices, stream),
                   "split-k reduce launch");
        ++launches;
    }
    plan->last_tasks = static_cast<int64_t>(s.host_tasks.size());
    plan->last_launches = launches;
    plan->last_ctas = s.grid;
}

// ---------------------------------------------- copy-engine-fed pipeline
using StreamValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
struct MemOps {
    StreamValueFn write = nullptr, wait = nullptr;
};
// cuStreamWriteValue32 / cuStreamWaitValue32 through the runtime's driver
// entry point (the library links the static runtime, not libcuda); null
// when the driver does not provide them.
const MemOps& memops() {
    static const MemOps m = [] {
        MemOps r;
        void* fw = nullptr;
        void* fv = nullptr;
        cudaDriverEntryPointQueryResult qw{}, qv{};
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fw, cudaEnableDefault, &qw) == cudaSuccess &&
            qw == cudaDriverEntryPointSuccess &&
            cudaGetDriverEntryPoint("cuStreamWaitValue32", &fv, cudaEnableDefault, &qv) == cudaSuccess &&
            qv == cudaDriverEntryPointSuccess) {
            r.write = reinterpret_cast<StreamValueFn>(fw);
            r.wait = reinterpret_cast<StreamValueFn>(fv);
        }
        return r;
    }();
    return m;
}

// The persistent pipeline's tasks wait on flags written by another stream's
// copies: that needs the kernel and the copies to run concurrently, which
// CUDA_LAUNCH_BLOCKING=1 (the launch returns only when the kernel is done)
// and injected tools that serialize GPU work (Nsight Compute, sanitizers:
// CUDA_INJECTION64_PATH) rule out. Those get the one-launch-per-unit path.
bool serialized_launches() {
    const char* lb = std::getenv("CUDA_LAUNCH_BLOCKING");
    return (lb != nullptr && std::atoi(lb) != 0) || std::getenv("CUDA_INJECTION64_PATH") != nullptr;
}

void cu_check(CUresult r, const char* what) {
    if (r != CUDA_SUCCESS) throw Failure(kDevice, "", std::string(what) + ": CUresult " + std::to_string(static_cast<int>(r)));
}

// Cut points of [0, total) into `pieces` equal pieces, aligned.
std::vector<i64> even_cuts(i64 total, int pieces, i64 align) {
    const i64 each = cdiv(cdiv(total, std::max(1, pieces)), align) * align;
    std::vector<i64> start{0};
    while (start.back() < total) start.push_back(std::min(total, start.back() + each));
    return start;
}

// Lowers every unit's sub-nest (fused, unsplit) and splices the task lists
// into one, in unit order, with global coordinates; each task waits for its
// unit's data flag and for the previous chunk of its C tile (progress
// counters, as in the faithful schedule), so every C entry still sees its k
// chunks in ascending order.
std::unique_ptr<HostPipe> build_pipe(const tm_plan& plan, const tm_exec_opts& o, cudaStream_t st) {
    const Extents& e = plan.nest.ext;
    auto P = std::make_unique<HostPipe>();
    P->opts = o;
    // k-chunks of >= 4096 (at most 4) and column blocks of >= 256 (at most
    // 64): at 16384^3 on PCIe Gen5 these measured best among 4..16 chunks x
    // 8..64 blocks (tools/e2e_probe.py); smaller k-chunks cost more C round
    // trips, larger first pieces delay the first GEMM.
    P->kcut = even_cuts(e.k, static_cast<int>(std::max<i64>(1, std::min<i64>(4, e.k / 4096))), 32);
    P->ncut = even_cuts(e.n, static_cast<int>(std::max<i64>(1, std::min<i64>(64, e.n / 256))), 128);
    const int nq = static_cast<int>(P->kcut.size()) - 1, nbk = static_cast<int>(P->ncut.size()) - 1;
    // Growing-rectangle order: after (A_0, C_0), load next whichever of the
    // next A k-chunk or the next C column block enables more GEMM work per
    // byte copied, then run the (block, chunk) units it enables: a new A
    // chunk adds column q for every loaded block, a new C block adds row b
    // for every loaded chunk (ascending q, so each C entry still sees its k
    // chunks in order). Early on this keeps the copy stream ahead of the
    // math instead of front-loading all of A.
    {
        int na = 1, nc = 1;
        P->units.push_back({0, 0});
        const double mm = static_cast<double>(e.m);
        while (na < nq || nc < nbk) {
            const double kq = static_cast<double>(na < nq ? P->kcut[static_cast<std::size_t>(na) + 1] - P->kcut[static_cast<std::size_t>(na)] : 1);
            const double wb = static_cast<double>(nc < nbk ? P->ncut[static_cast<std::size_t>(nc) + 1] - P->ncut[static_cast<std::size_t>(nc)] : 1);
            const double wavg = static_cast<double>(P->ncut[static_cast<std::size_t>(nc)]) / nc;   // loaded columns per block
            const double kavg = static_cast<double>(P->kcut[static_cast<std::size_t>(na)]) / na;  // loaded k per chunk
            // flops per byte of the copies each choice needs
            const double ra = na < nq ? (nc * mm * kq * wavg) / (mm * kq + nc * kq * wavg) : -1.0;
            const double rc = nc < nbk ? (na * mm * kavg * wb) / (mm * wb + na * kavg * wb) : -1.0;
            if (ra > rc) {
                for (int b2 = 0; b2 < nc; ++b2) P->units.push_back({b2, na});
                ++na;
            } else {
                for (int q2 = 0; q2 < na; ++q2) P->units.push_back({nc, q2});
                ++nc;
            }
        }
    }
    tm_exec_opts uo = o;
    uo.split_k = 1;
    Nest first = plan.nest;
    first.ext.n = P->ncut[1];
    first.ext.k = P->kcut[1];
    const gpu::Kernel kernel = pick_kernel(first, uo);
    gpu::KernelInfo info{};
    cuda_check(gpu::kernel_info(kernel, &info), "kernel_info");
    const i64 mt = cdiv(e.m, info.tile_m);
    P->regions = static_cast<int>(mt * cdiv(e.n, info.tile_n));
    P->block_tasks.assign(static_cast<std::size_t>(nbk), 0);
    auto sched = std::make_unique<Schedule>();
    sched->kernel = kernel;
    auto& T = sched->host_tasks;
    for (std::size_t u = 0; u < P->units.size(); ++u) {
        const auto [b, q] = P->units[u];
        const i64 j0 = P->ncut[static_cast<std::size_t>(b)], p0 = P->kcut[static_cast<std::size_t>(q)];
        Nest sn = plan.nest;
        sn.ext.n = P->ncut[static_cast<std::size_t>(b) + 1] - j0;
        sn.ext.k = P->kcut[static_cast<std::size_t>(q) + 1] - p0;
        const auto part = lower(sn, uo, kernel, st, false);
        for (gpu::Task tk : part->host_tasks) {
            tk.j0 += static_cast<int32_t>(j0);
            tk.p0 += static_cast<int32_t>(p0);
            tk.tile = static_cast<int32_t>(tk.i0 / info.tile_m + (tk.j0 / info.tile_n) * mt);
            tk.seq = q;
            tk.ready = static_cast<int32_t>(u) + 1;
            tk.done = q == nq - 1 ? b + 1 : 0;
            T.push_back(tk);
        }
        if (q == nq - 1) P->block_tasks[static_cast<std::size_t>(b)] = static_cast<int32_t>(part->host_tasks.size());
    }
    if (T.size() > static_cast<std::size_t>(INT32_MAX)) fail_usage("too many tasks");
    sched->grid = std::max(1, std::min<int>(sm_count() * std::max(1, info.ctas_per_sm), static_cast<int>(T.size())));
    sched->regions = P->regions;
    cuda_check(cudaGetDevice(&sched->device), "cudaGetDevice");
    cuda_check(cudaMalloc(&sched->progress, sizeof(int32_t) * static_cast<std::size_t>(P->regions)), "cudaMalloc(progress)");
    cuda_check(cudaMalloc(&sched->tasks, sizeof(gpu::Task) * T.size()), "cudaMalloc(tasks)");
    cuda_check(cudaMemcpyAsync(sched->tasks, T.data(), sizeof(gpu::Task) * T.size(), cudaMemcpyHostToDevice, st),
               "upload tasks");
    cuda_check(cudaMalloc(&P->flags, sizeof(int32_t) * (P->units.size() + static_cast<std::size_t>(nbk))),
               "cudaMalloc(pipeline flags)");
    cuda_check(cudaStreamSynchronize(st), "upload tasks (sync)");
    P->sched = std::move(sched);
    return P;
}

bool same_opts(const tm_exec_opts& a, const tm_exec_opts& b) {
    return a.numerics == b.numerics && a.schedule == b.schedule && a.split_k == b.split_k && a.ctas == b.ctas &&
           a.tile == b.tile && a.tile_n == b.tile_n;
}

void run_pipe(tm_plan* plan, const double* A, const double* B, double* C, const tm_exec_opts& o) {
    const Extents& e = plan->nest.ext;
    cudaStream_t st = plan->host_stream, cs = plan->copy_stream, ds = plan->d2h_stream;
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    if (!plan->pipe || !same_opts(plan->pipe->opts, o) || plan->pipe->sched->device != dev)
        plan->pipe = build_pipe(*plan, o, st);
    HostPipe& P = *plan->pipe;
    Schedule& S = *P.sched;
    const std::size_t nu = P.units.size(), nbk = P.ncut.size() - 1;
    if (plan->chunk_ready.empty()) {
        cudaEvent_t ev;
        cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
        plan->chunk_ready.push_back(ev);
    }
    cudaEvent_t zero = plan->chunk_ready[0];
    cuda_check(cudaMemsetAsync(S.progress, 0, sizeof(int32_t) * static_cast<std::size_t>(P.regions), st), "reset progress");
    cuda_check(cudaMemsetAsync(P.flags, 0, sizeof(int32_t) * (nu + nbk), st), "reset flags");
    cuda_check(cudaEventRecord(zero, st), "event");
    const bool vec16 = e.m % 2 == 0 && e.k % 2 == 0 && origins_even(S.host_tasks);
    gpu::Args a{plan->dA, e.m, plan->dB, e.k, plan->dC, e.m, S.tasks, static_cast<int32_t>(S.host_tasks.size()),
                S.progress, nullptr, 0, 0, nullptr, P.flags, P.flags + nu};
    cuda_check(gpu::launch(S.kernel, vec16, a, S.grid, st), "pipeline kernel launch");

    // uploads in first-need order, a flag after each unit's pieces
    const std::size_t ldb = static_cast<std::size_t>(e.k) * sizeof(double);
    cuda_check(cudaStreamWaitEvent(cs, zero, 0), "wait flags reset");
    std::vector<char> have_a(P.kcut.size(), 0);
    for (std::size_t u = 0; u < nu; ++u) {
        const auto [b, q] = P.units[u];
        const i64 j0 = P.ncut[static_cast<std::size_t>(b)], w = P.ncut[static_cast<std::size_t>(b) + 1] - j0;
        const i64 p0 = P.kcut[static_cast<std::size_t>(q)], kq = P.kcut[static_cast<std::size_t>(q) + 1] - p0;
        if (q == 0)
            cuda_check(cudaMemcpyAsync(plan->dC + j0 * e.m, C + j0 * e.m, static_cast<std::size_t>(w * e.m) * 8,
                                       cudaMemcpyHostToDevice, cs),
                       "H2D C block");
        if (!have_a[static_cast<std::size_t>(q)]) {
            have_a[static_cast<std::size_t>(q)] = 1;
            cuda_check(cudaMemcpyAsync(plan->dA + p0 * e.m, A + p0 * e.m, static_cast<std::size_t>(kq * e.m) * 8,
                                       cudaMemcpyHostToDevice, cs),
                       "H2D A chunk");
        }
        cuda_check(cudaMemcpy2DAsync(plan->dB + p0 + j0 * e.k, ldb, B + p0 + j0 * e.k, ldb,
                                     static_cast<std::size_t>(kq) * 8, static_cast<std::size_t>(w),
                                     cudaMemcpyHostToDevice, cs),
                   "H2D B piece");
        cu_check(memops().write(reinterpret_cast<CUstream>(cs), reinterpret_cast<CUdeviceptr>(P.flags + u), 1, 0),
                 "cuStreamWriteValue32");
    }
    // each block goes back once its last unit's tasks are done
    cuda_check(cudaStreamWaitEvent(ds, zero, 0), "wait flags reset");
    for (std::size_t b = 0; b < nbk; ++b) {
        const i64 j0 = P.ncut[b], w = P.ncut[b + 1] - j0;
        cu_check(memops().wait(reinterpret_cast<CUstream>(ds), reinterpret_cast<CUdeviceptr>(P.flags + nu + b),
                               static_cast<cuuint32_t>(P.block_tasks[b]), CU_STREAM_WAIT_VALUE_GEQ),
                 "cuStreamWaitValue32");
        cuda_check(cudaMemcpyAsync(C + j0 * e.m, plan->dC + j0 * e.m, static_cast<std::size_t>(w * e.m) * 8,
                                   cudaMemcpyDeviceToHost, ds),
                   "D2H C block");
    }
    cuda_check(cudaStreamSynchronize(ds), "execute_host sync");
    cuda_check(cudaStreamSynchronize(st), "execute_host sync");
    plan->last_tasks = static_cast<int64_t>(S.host_tasks.size());
    plan->last_launches = 1;
    plan->last_ctas = S.grid;
}

}  // namespace

extern "C" {

const char* tm_last_error(void) { return g_error.c_str(); }
const char* tm_last_rules(void) { return g_rules.c_str(); }
const char* tm_version(void) { return "tilemul_b200 0.1 (sm_100a)"; }

int tm_parse_name(const char* name, int allow_non_c, tm_tier* tiers, int cap, int* count) {
    return guard([&] {
        if (!name) fail_usage("null name");
        put_tiers(family_from_name(name, allow_non_c != 0), tiers, cap, count);
    });
}

int tm_compose(const int32_t* levels, const char* residents, int count, int allow_non_c, char* name_out, int name_cap,
               tm_tier* tiers, int cap, int* tier_count) {
    return guard([&] {
        std::vector<std::pair<int, Opnd>> r;
        for (int i = 0; i < count; ++i) r.emplace_back(levels[i], opnd_of_char(residents[i]));
        Family f = compose(r, allow_non_c != 0);
        put_name(family_name(f), name_out, name_cap);
        put_tiers(f, tiers, cap, tier_count);
    });
}

int tm_validate_structure(const tm_tier* tiers, int count, int allow_non_c) {
    int n = 0;
    int rc = guard([&] {
        Family f;
        f.free_registers = allow_non_c != 0;
        for (int i = 0; i < count; ++i)
            f.tiers.push_back(Tier{tiers[i].level, opnd_of_char(tiers[i].resident), dim_of_char(tiers[i].outer_dim),
                                   dim_of_char(tiers[i].inner_dim)});
        auto issues = structure_issues(f);
        n = static_cast<int>(issues.size());
        for (const auto& v : issues)
            g_rules += v.rule + ":" + std::to_string(v.level) + ":" + std::to_string(v.lhs) + ":" + std::to_string(v.rhs) + "\n";
    });
    return rc == kOk ? n : -rc;
}

int tm_skip_level(const char* name, int level, char* name_out, int name_cap) {
    return guard([&] { put_name(family_name(without_level(family_from_name(name), level)), name_out, name_cap); });
}

int tm_select_outer(int64_t m, int64_t n, int64_t k, int64_t cap, char* resident) {
    return guard([&] { *resident = opnd_char(outer_resident_for(make_extents(m, n, k), cap)); });
}

int tm_derive(const char* name, const tm_level* levels, int nlevels, int64_t m, int64_t n, int64_t k,
              const tm_derive_opts* opts, const tm_blocksize* pinned, int npinned, tm_blocksize* out, int cap,
              int* count) {
    return guard([&] {
        DeriveOpts d;
        Weights w;
        if (opts) {
            d.slack = opts->slack;
            d.m_r = opts->m_r;
            d.n_r = opts->n_r;
            w = Weights{opts->beta_a, opts->beta_b, opts->beta_c};
        }
        Blocks bs = derive(family_from_name(name), hierarchy_from(levels, nlevels), make_extents(m, n, k), w, d,
                           blocks_from(pinned, npinned));
        auto ent = bs.entries();
        if (count) *count = static_cast<int>(ent.size());
        if (static_cast<int>(ent.size()) > cap) fail_usage("blocksize buffer too small");
        for (std::size_t i = 0; i < ent.size(); ++i)
            out[i] = tm_blocksize{std::get<0>(ent[i]), dim_char(std::get<1>(ent[i])), std::get<2>(ent[i])};
    });
}

int tm_validate(const char* name, const tm_level* levels, int nlevels, int64_t m, int64_t n, int64_t k,
                const tm_blocksize* bs, int nbs) {
    int count = 0;
    int rc = guard([&] {
        (void)make_extents(m, n, k);
        auto issues = fit_issues(family_from_name(name), blocks_from(bs, nbs), hierarchy_from(levels, nlevels));
        count = static_cast<int>(issues.size());
        for (const auto& v : issues)
            g_rules += v.rule + ":" + std::to_string(v.level) + ":" + std::to_string(v.lhs) + ":" + std::to_string(v.rhs) + "\n";
    });
    return rc == kOk ? count : -rc;
}

int tm_gpu_hierarchy(int tile, tm_level* levels, int cap, int* count) {
    return guard([&] {
        if (tile != 64 && tile != 128) fail_usage("tile must be 64 or 128");
        if (cap < 3) fail_usage("level buffer too small");
        int dev = 0, smem = 0, l2 = 0;
        cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
        cuda_check(cudaDeviceGetAttribute(&smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev), "smem attr");
        cuda_check(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev), "l2 attr");
        levels[0] = tm_level{static_cast<int64_t>(tile) * tile, 1, 0, 1, 1};
        levels[1] = tm_level{smem / 8, 1, 0, 1, 1};
        levels[2] = tm_level{l2 / 8, 1, 0, 1, 1};
        if (count) *count = 3;
    });
}

int tm_plan_create(const char* name, const tm_level* levels, int nlevels, int64_t m, int64_t n, int64_t k,
                   const tm_blocksize* bs, int nbs, tm_plan** plan) {
    return guard([&] {
        if (!plan) fail_usage("null plan out-pointer");
        auto p = std::make_unique<tm_plan>();
        p->hier = hierarchy_from(levels, nlevels);
        p->nest = build_nest(family_from_name(name), blocks_from(bs, nbs), p->hier, make_extents(m, n, k));
        *plan = p.release();
    });
}

void tm_plan_destroy(tm_plan* plan) { delete plan; }

int tm_plan_loops(const tm_plan* plan, tm_loop* loops, int cap, int* count) {
    return guard([&] {
        const auto& L = plan->nest.loops;
        if (count) *count = static_cast<int>(L.size());
        if (static_cast<int>(L.size()) > cap) fail_usage("loop buffer too small");
        for (std::size_t i = 0; i < L.size(); ++i)
            loops[i] = tm_loop{L[i].level, dim_char(L[i].dim), L[i].size, L[i].cap ? 1 : 0};
    });
}

int64_t tm_plan_cells(const tm_plan* plan) { return plan ? plan->nest.cells() : -1; }

int tm_plan_model(const tm_plan* plan, int64_t* out, int cap) {
    return guard([&] {
        if (!plan) fail_usage("null plan");
        IoModel r = level_io(plan->nest.family, plan->nest.blocks, plan->hier, plan->nest.ext);
        if (static_cast<int>(r.levels.size()) * 6 > cap) fail_usage("model buffer too small");
        for (const auto& lf : r.levels)
            for (int o = 0; o < 3; ++o) {
                out[(lf.level * 3 + o) * 2] = lf.op[static_cast<std::size_t>(o)].reads;
                out[(lf.level * 3 + o) * 2 + 1] = lf.op[static_cast<std::size_t>(o)].writes;
            }
    });
}

int tm_plan_levels(const tm_plan* plan) { return plan ? plan->hier.size() : -1; }

int tm_model(const char* name, int allow_non_c, const tm_level* levels, int nlevels, int64_t m, int64_t n, int64_t k,
             const tm_blocksize* bs, int nbs, int64_t* out, int cap) {
    return guard([&] {
        IoModel r = level_io(family_from_name(name, allow_non_c != 0), blocks_from(bs, nbs),
                             hierarchy_from(levels, nlevels), make_extents(m, n, k));
        if (static_cast<int>(r.levels.size()) * 6 > cap) fail_usage("model buffer too small");
        for (const auto& lf : r.levels)
            for (int o = 0; o < 3; ++o) {
                out[(lf.level * 3 + o) * 2] = lf.op[static_cast<std::size_t>(o)].reads;
                out[(lf.level * 3 + o) * 2 + 1] = lf.op[static_cast<std::size_t>(o)].writes;
            }
    });
}

int tm_io_lower_bound(int64_t m, int64_t n, int64_t k, int64_t M, int64_t* reads, int64_t* writes) {
    return guard([&] {
        Flow f = lower_bound_io(make_extents(m, n, k), M);
        *reads = f.reads;
        *writes = f.writes;
    });
}

int tm_resident_cost(char variant, int64_t m, int64_t n, int64_t k, int64_t b1, int64_t b2, int64_t* out) {
    return guard([&] {
        LevelFlow t = resident_io(opnd_of_char(variant), make_extents(m, n, k), b1, b2);
        for (int o = 0; o < 3; ++o) {
            out[o * 2] = t.op[static_cast<std::size_t>(o)].reads;
            out[o * 2 + 1] = t.op[static_cast<std::size_t>(o)].writes;
        }
    });
}

double tm_streaming_efficiency(char variant, int64_t b1, int64_t b2) {
    double r = -1;
    guard([&] { r = streaming_flops_per_element(opnd_of_char(variant), b1, b2); });
    return r;
}

double tm_goto_efficiency(int64_t k_c, int64_t n_c) {
    double r = -1;
    guard([&] { r = goto_flops_per_element(k_c, n_c); });
    return r;
}

double tm_roofline_bound(double intensity, double peak, double bandwidth) {
    double r = -1;
    guard([&] { r = roofline(intensity, peak, bandwidth); });
    return r;
}

int tm_execute(tm_plan* plan, const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
               const tm_exec_opts* opts, void* stream) {
    return guard([&] {
        if (!plan) fail_usage("null plan");
        run(plan, A, lda, B, ldb, C, ldc, opts, static_cast<cudaStream_t>(stream));
    });
}

int tm_execute_host(tm_plan* plan, const double* A, const double* B, double* C, const tm_exec_opts* opts) {
    return guard([&] {
        if (!plan) fail_usage("null plan");
        if (!A || !B || !C) fail_usage("null operand pointer");
        std::lock_guard<std::mutex> hold(plan->host_mu);
        const Extents& e = plan->nest.ext;
        const std::size_t na = static_cast<std::size_t>(e.m * e.k), nb = static_cast<std::size_t>(e.k * e.n),
                          nc = static_cast<std::size_t>(e.m * e.n);
        auto mkstream = [](cudaStream_t& s) {
            if (!s) cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
        };
        mkstream(plan->host_stream);
        if (!plan->dA) {
            cuda_check(cudaMalloc(&plan->dA, na * sizeof(double)), "cudaMalloc(A)");
            cuda_check(cudaMalloc(&plan->dB, nb * sizeof(double)), "cudaMalloc(B)");
            cuda_check(cudaMalloc(&plan->dC, nc * sizeof(double)), "cudaMalloc(C)");
        }
        cudaStream_t st = plan->host_stream;
        tm_exec_opts o{};
        if (opts) o = *opts;
        const bool pipelined = o.schedule == TM_SCHEDULE_FUSED && o.split_k <= 1 && (e.k >= 4096 || e.n >= 4096);
        if (!pipelined) {
            cuda_check(cudaMemcpyAsync(plan->dA, A, na * sizeof(double), cudaMemcpyHostToDevice, st), "H2D A");
            cuda_check(cudaMemcpyAsync(plan->dB, B, nb * sizeof(double), cudaMemcpyHostToDevice, st), "H2D B");
            cuda_check(cudaMemcpyAsync(plan->dC, C, nc * sizeof(double), cudaMemcpyHostToDevice, st), "H2D C");
            run(plan, plan->dA, e.m, plan->dB, e.k, plan->dC, e.m, opts, st);
            cuda_check(cudaMemcpyAsync(C, plan->dC, nc * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H C");
            cuda_check(cudaStreamSynchronize(st), "execute_host sync");
            return;
        }
        // Copy/compute pipeline over (C column block, k-chunk) units; every
        // C entry still sees its k chunks in ascending order (chunks are
        // multiples of the 32-deep slab), i.e. exactly the unpipelined
        // operation sequence. Preferred: one persistent launch fed by the
        // copy engine (run_pipe).
        mkstream(plan->copy_stream);
        mkstream(plan->d2h_stream);
        if (memops().write && memops().wait && !serialized_launches()) {
            run_pipe(plan, A, B, C, o);
            return;
        }
        // Fallback (driver without stream memory operations): one launch per
        // unit, units in wavefront order (b + q ascending), uploads on one
        // copy stream in first-need order, downloads on a third stream.
        const std::vector<i64> kcut = even_cuts(e.k, e.k >= 4096 ? static_cast<int>(std::min<i64>(8, e.k / 2048)) : 1, 32);
        const std::vector<i64> ncut = even_cuts(e.n, e.n >= 2048 ? static_cast<int>(std::min<i64>(16, e.n / 1024)) : 1, 128);
        const int nq = static_cast<int>(kcut.size()) - 1;
        const int nbk = static_cast<int>(ncut.size()) - 1;
        const std::size_t nev = static_cast<std::size_t>(nq + 2 * nbk + nbk * nq);
        while (plan->chunk_ready.size() < nev) {
            cudaEvent_t ev;
            cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
            plan->chunk_ready.push_back(ev);
        }
        cudaEvent_t* evA = plan->chunk_ready.data();
        cudaEvent_t* evC = evA + nq;
        cudaEvent_t* evDone = evC + nbk;
        cudaEvent_t* evB = evDone + nbk;
        auto sub = [&](i64 nn, i64 kk) -> tm_plan* {
            auto& slot = plan->chunk_plans[{nn, kk}];
            if (!slot) {
                slot = std::make_unique<tm_plan>();
                slot->nest = plan->nest;
                slot->nest.ext.n = nn;
                slot->nest.ext.k = kk;
                slot->hier = plan->hier;
            }
            return slot.get();
        };
        cudaStream_t cs = plan->copy_stream, ds = plan->d2h_stream;
        const std::size_t ld = static_cast<std::size_t>(e.k) * sizeof(double);
        int64_t tasks = 0;
        int32_t launches = 0, ctas = 0;
        auto d2h = [&](int b) {
            const i64 j0 = ncut[static_cast<std::size_t>(b)], w = ncut[static_cast<std::size_t>(b) + 1] - j0;
            cuda_check(cudaStreamWaitEvent(ds, evDone[b], 0), "wait block");
            cuda_check(cudaMemcpyAsync(C + j0 * e.m, plan->dC + j0 * e.m, static_cast<std::size_t>(w * e.m) * 8,
                                       cudaMemcpyDeviceToHost, ds),
                       "D2H C block");
        };
        std::vector<char> have_a(static_cast<std::size_t>(nq), 0);
        std::vector<int> finished;  // blocks whose D2H is issued one unit later (a pageable D2H blocks the host)
        std::vector<std::pair<int, int>> units;
        for (int wave = 0; wave < nbk + nq - 1; ++wave)
            for (int b = std::max(0, wave - nq + 1); b <= std::min(nbk - 1, wave); ++b) units.push_back({b, wave - b});
        {
            for (auto [b, q] : units) {
                const i64 j0 = ncut[static_cast<std::size_t>(b)], w = ncut[static_cast<std::size_t>(b) + 1] - j0;
                const i64 p0 = kcut[static_cast<std::size_t>(q)], kq = kcut[static_cast<std::size_t>(q) + 1] - p0;
                if (q == 0) {
                    cuda_check(cudaMemcpyAsync(plan->dC + j0 * e.m, C + j0 * e.m, static_cast<std::size_t>(w * e.m) * 8,
                                               cudaMemcpyHostToDevice, cs),
                               "H2D C block");
                    cuda_check(cudaEventRecord(evC[b], cs), "event");
                }
                if (!have_a[static_cast<std::size_t>(q)]) {
                    have_a[static_cast<std::size_t>(q)] = 1;
                    cuda_check(cudaMemcpyAsync(plan->dA + p0 * e.m, A + p0 * e.m,
                                               static_cast<std::size_t>(kq * e.m) * 8, cudaMemcpyHostToDevice, cs),
                               "H2D A chunk");
                    cuda_check(cudaEventRecord(evA[q], cs), "event");
                }
                cuda_check(cudaMemcpy2DAsync(plan->dB + p0 + j0 * e.k, ld, B + p0 + j0 * e.k, ld,
                                             static_cast<std::size_t>(kq) * 8, static_cast<std::size_t>(w),
                                             cudaMemcpyHostToDevice, cs),
                           "H2D B piece");
                cudaEvent_t eb = evB[b * nq + q];
                cuda_check(cudaEventRecord(eb, cs), "event");
                // issue the GEMM right away so pageable-memory copies (which
                // block the host while staging) still overlap device compute
                if (q == 0) cuda_check(cudaStreamWaitEvent(st, evC[b], 0), "wait C block");
                cuda_check(cudaStreamWaitEvent(st, evA[q], 0), "wait A chunk");
                cuda_check(cudaStreamWaitEvent(st, eb, 0), "wait B piece");
                tm_plan* pq = sub(w, kq);
                run(pq, plan->dA + p0 * e.m, e.m, plan->dB + p0 + j0 * e.k, e.k, plan->dC + j0 * e.m, e.m, &o, st);
                tasks += pq->last_tasks;
                launches += pq->last_launches;
                ctas = pq->last_ctas;
                for (int f : finished) d2h(f);
                finished.clear();
                if (q == nq - 1) {
                    cuda_check(cudaEventRecord(evDone[b], st), "event");
                    finished.push_back(b);
                }
            }
        }
        for (int f : finished) d2h(f);
        cuda_check(cudaStreamSynchronize(ds), "execute_host sync");
        cuda_check(cudaStreamSynchronize(st), "execute_host sync");
        plan->last_tasks = tasks;
        plan->last_launches = launches;
        plan->last_ctas = ctas;
    });
}

int tm_execute_tc(tm_plan* plan, int dtype, const void* A, int64_t lda, const void* B, int64_t ldb, float* C,
                  int64_t ldc, const tm_exec_opts* opts, void* stream) {
    return guard([&] {
        if (!plan) fail_usage("null plan");
        if (!A || !B || !C) fail_usage("null operand pointer");
        if (dtype != TM_DTYPE_BF16 && dtype != TM_DTYPE_TF32) fail_usage("dtype must be TM_DTYPE_BF16 or TM_DTYPE_TF32");
        const Extents& e = plan->nest.ext;
        if (lda < e.m || ldb < e.k || ldc < e.m) fail_usage("leading dimension smaller than the operand's row count");
        tm_exec_opts o{};
        if (opts) o = *opts;
        if (o.schedule != TM_SCHEDULE_FUSED) fail_usage("tensor-core path runs the fused schedule only");
        if (o.split_k > 1) fail_usage("tensor-core path does not split k");
        o.split_k = 1;
        if (o.tile != 0 && o.tile != 128 && o.tile != 256) fail_usage("tensor-core tile must be 128 (1 SM) or 256 (SM pair)");
        const bool pair = o.tile != 128;
        const gpu::Kernel kernel = dtype == TM_DTYPE_TF32 ? (pair ? gpu::kTc2Tf32 : gpu::kTcTf32)
                                                          : (pair ? gpu::kTc2Bf16 : gpu::kTcBf16);
        std::lock_guard<std::mutex> lk(plan->mu);
        Key key{o.schedule, kernel, 1, o.ctas, false};
        auto& slot = plan->schedules[key];
        int dev = 0;
        cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
        if (!slot || slot->device != dev) slot = lower(plan->nest, o, kernel, static_cast<cudaStream_t>(stream));
        Schedule& s = *slot;
        const int nt = static_cast<int>(s.host_tasks.size());
        cuda_check(pair ? gpu::launch_tc_pair(dtype == TM_DTYPE_TF32, A, lda, B, ldb, C, ldc, e.m, e.n, e.k, s.tasks,
                                              nt, s.grid, static_cast<cudaStream_t>(stream))
                        : gpu::launch_tc(dtype == TM_DTYPE_TF32, A, lda, B, ldb, C, ldc, e.m, e.n, e.k, s.tasks, nt,
                                         s.grid, static_cast<cudaStream_t>(stream)),
                   "tensor-core kernel launch (TMA needs 16-byte aligned bases and leading dimensions)");
        plan->last_tasks = static_cast<int64_t>(s.host_tasks.size());
        plan->last_launches = 1;
        plan->last_ctas = s.grid;
    });
}

int tm_round_inputs(int dtype, const double* x, void* y, int64_t count, void* stream) {
    return guard([&] {
        if (dtype != TM_DTYPE_BF16 && dtype != TM_DTYPE_TF32) fail_usage("dtype must be TM_DTYPE_BF16 or TM_DTYPE_TF32");
        cuda_check(gpu::launch_round(dtype == TM_DTYPE_TF32, x, y, count, static_cast<cudaStream_t>(stream)),
                   "round launch");
    });
}

// ------------------------------------------------------ prepacked layouts

namespace {

gpu::LayoutDev layout_dev(const Blocked& b) {
    if (static_cast<int>(b.cuts.size()) > gpu::LayoutDev::kMaxCuts) fail_usage("too many partition steps");
    gpu::LayoutDev L{};
    L.rows = b.rows;
    L.cols = b.cols;
    L.ncuts = static_cast<int32_t>(b.cuts.size());
    for (std::size_t s = 0; s < b.cuts.size(); ++s) {
        L.on_rows[s] = b.cuts[s].rows ? 1 : 0;
        L.size[s] = b.cuts[s].size;
    }
    return L;
}

}  // namespace

int tm_layout_address(int64_t rows, int64_t cols, const int32_t* on_rows, const int64_t* sizes, int ncuts, int64_t i,
                      int64_t j, int64_t* address) {
    return guard([&] {
        std::vector<Cut> cuts;
        for (int s = 0; s < ncuts; ++s) cuts.push_back(Cut{on_rows[s] != 0, sizes[s]});
        *address = make_blocked(rows, cols, std::move(cuts)).address(i, j);
    });
}

int tm_plan_layout(const tm_plan* plan, char operand, int32_t* on_rows, int64_t* sizes, int cap, int* ncuts) {
    return guard([&] {
        if (!plan) fail_usage("null plan");
        const Blocked b = layout_of(plan->nest, opnd_of_char(operand));
        if (ncuts) *ncuts = static_cast<int>(b.cuts.size());
        if (static_cast<int>(b.cuts.size()) > cap) fail_usage("cut buffer too small");
        for (std::size_t s = 0; s < b.cuts.size(); ++s) {
            on_rows[s] = b.cuts[s].rows ? 1 : 0;
            sizes[s] = b.cuts[s].size;
        }
    });
}

int tm_pack(const tm_plan* plan, char operand, const double* colmajor, double* packed, void* stream) {
    return guard([&] {
        if (!plan || !colmajor || !packed) fail_usage("null argument");
        cuda_check(gpu::launch_relayout(colmajor, packed, layout_dev(layout_of(plan->nest, opnd_of_char(operand))),
                                        true, static_cast<cudaStream_t>(stream)),
                   "pack launch");
    });
}

int tm_unpack(const tm_plan* plan, char operand, const double* packed, double* colmajor, void* stream) {
    return guard([&] {
        if (!plan || !colmajor || !packed) fail_usage("null argument");
        cuda_check(gpu::launch_relayout(packed, colmajor, layout_dev(layout_of(plan->nest, opnd_of_char(operand))),
                                        false, static_cast<cudaStream_t>(stream)),
                   "unpack launch");
    });
}

int tm_execute_packed(tm_plan* plan, const double* A, const double* B, double* C, const tm_exec_opts* opts,
                      void* stream) {
    return guard([&] {
        if (!plan) fail_usage("null plan");
        if (!A || !B || !C) fail_usage("null operand pointer");
        const Extents& e = plan->nest.ext;
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const std::size_t na = static_cast<std::size_t>(e.m * e.k), nb = static_cast<std::size_t>(e.k * e.n),
                          nc = static_cast<std::size_t>(e.m * e.n);
        if (!plan->dA) {
            cuda_check(cudaMalloc(&plan->dA, na * sizeof(double)), "cudaMalloc(A)");
            cuda_check(cudaMalloc(&plan->dB, nb * sizeof(double)), "cudaMalloc(B)");
            cuda_check(cudaMalloc(&plan->dC, nc * sizeof(double)), "cudaMalloc(C)");
        }
        // the kernels stage column-major k-slabs; prepacked operands are
        // relaid once per call (2 extra passes over A, B and C each)
        cuda_check(gpu::launch_relayout(A, plan->dA, layout_dev(layout_of(plan->nest, kA)), false, st), "unpack A");
        cuda_check(gpu::launch_relayout(B, plan->dB, layout_dev(layout_of(plan->nest, kB)), false, st), "unpack B");
        cuda_check(gpu::launch_relayout(C, plan->dC, layout_dev(layout_of(plan->nest, kC)), false, st), "unpack C");
        run(plan, plan->dA, e.m, plan->dB, e.k, plan->dC, e.m, opts, st);
        cuda_check(gpu::launch_relayout(plan->dC, C, layout_dev(layout_of(plan->nest, kC)), true, st), "pack C");
    });
}

int tm_plan_last_launch(const tm_plan* plan, int64_t* tasks, int32_t* launches, int32_t* ctas) {
    return guard([&] {
        if (tasks) *tasks = plan->last_tasks;
        if (launches) *launches = plan->last_launches;
        if (ctas) *ctas = plan->last_ctas;
    });
}

int tm_fill_seeded(uint64_t seed, double* a, int64_t na, double* b, int64_t nb, double* c, int64_t nc) {
    return guard([&] {
        if (!a && na > 0) fail_usage("null A buffer");
        fill_seeded(seed, a, na, b, nb, c, nc);
    });
}

int tm_measure_fp64_peak(int launches, double* tflops) {
    return guard([&] { cuda_check(gpu::measure_fp64_peak(launches < 1 ? 1 : launches, tflops), "fp64 peak probe"); });
}

int tm_fill_uniform_block(double* x, int64_t rows, int64_t cols, int64_t ld, uint64_t seed, int64_t row0,
                          int64_t col0, int64_t global_ld, void* stream) {
    return guard([&] {
        if (ld < rows) fail_usage("leading dimension smaller than the block's row count");
        cuda_check(gpu::launch_fill_block(x, rows, cols, ld, seed, row0, col0, global_ld,
                                          static_cast<cudaStream_t>(stream)),
                   "fill launch");
    });
}

int tm_fill_uniform_device(double* x, int64_t count, uint64_t seed, uint64_t offset, void* stream) {
    return guard([&] {
        cuda_check(gpu::launch_fill(x, count, seed, offset, static_cast<cudaStream_t>(stream)), "fill launch");
    });
}

}  // extern "C"

// ------------------------------------------------------- trace / simulator

struct tm_sim {
    CacheSim sim;
};

int64_t tm_trace_event_count(const tm_plan* plan) {
    int64_t r = -kUsage;
    guard([&] {
        if (plan == nullptr) fail_usage("null plan");
        r = access_count(plan->nest);
    });
    return r;
}

int tm_trace(const tm_plan* plan, int packed, int64_t cap, char* ops, int64_t* indices, uint8_t* writes,
             int64_t* count) {
    return guard([&] {
        if (plan == nullptr) fail_usage("null plan");
        if (cap > 0 && (ops == nullptr || indices == nullptr || writes == nullptr)) fail_usage("null event buffer");
        const TraceAddressing lay =
            packed ? TraceAddressing::packed(plan->nest) : TraceAddressing::column_major(plan->nest.ext);
        int64_t n = 0;
        for_each_access(plan->nest, lay, [&](const Access& a) {
            if (n < cap) {
                ops[n] = opnd_char(a.op);
                indices[n] = a.index;
                writes[n] = a.write ? 1 : 0;
            }
            ++n;
        });
        if (count) *count = n;
    });
}

int tm_sim_create(const tm_level* levels, int nlevels, int64_t m, int64_t n, int64_t k, int include_registers,
                  int flush_dirty_at_end, tm_sim** sim) {
    return guard([&] {
        if (sim == nullptr) fail_usage("null output");
        *sim = new tm_sim{CacheSim(hierarchy_from(levels, nlevels), make_extents(m, n, k),
                                   SimConfig{include_registers != 0, flush_dirty_at_end != 0})};
    });
}

void tm_sim_destroy(tm_sim* sim) { delete sim; }

int tm_sim_access(tm_sim* sim, const char* ops, const int64_t* indices, const uint8_t* writes, int64_t count) {
    return guard([&] {
        if (sim == nullptr) fail_usage("null simulator");
        if (count > 0 && (ops == nullptr || indices == nullptr)) fail_usage("null event buffer");
        for (int64_t e = 0; e < count; ++e) {
            const Opnd op = opnd_of_char(ops[e]);
            if (indices[e] < 0) fail_usage("negative element index");
            sim->sim.access(Access{op, indices[e], writes != nullptr && writes[e] != 0});
        }
    });
}

int tm_sim_replay(tm_sim* sim, const tm_plan* plan, int packed) {
    return guard([&] {
        if (sim == nullptr || plan == nullptr) fail_usage("null simulator or plan");
        const TraceAddressing lay =
            packed ? TraceAddressing::packed(plan->nest) : TraceAddressing::column_major(plan->nest.ext);
        for_each_access(plan->nest, lay, [&](const Access& a) { sim->sim.access(a); });
    });
}

int tm_sim_finish(tm_sim* sim, tm_sim_level* out, int cap, int* count, int64_t* events) {
    return guard([&] {
        if (sim == nullptr) fail_usage("null simulator");
        const auto st = sim->sim.finish();
        if (count) *count = static_cast<int>(st.size());
        if (events) *events = sim->sim.events();
        if (out == nullptr) return;
        if (static_cast<int>(st.size()) > cap) fail_usage("level buffer too small");
        for (std::size_t i = 0; i < st.size(); ++i) {
            const SimStats& s = st[i];
            tm_sim_level& o = out[i];
            o.level = s.level;
            o.capacity_lines = s.capacity_lines;
            o.granularity = s.granularity;
            o.hits = s.hits;
            o.read_misses = s.read_misses;
            o.write_misses = s.write_misses;
            o.fetched_lines = s.fetched_lines;
            o.passthrough_writes = s.passthrough_writes;
            o.writebacks = s.writebacks;
            for (int q = 0; q < 3; ++q) {
                o.per_operand_misses[q] = s.op_misses[static_cast<std::size_t>(q)];
                o.per_operand_writebacks[q] = s.op_writebacks[static_cast<std::size_t>(q)];
            }
        }
    });
}

int tm_sim_resident_lines(const tm_sim* sim, int position, int64_t* lines, int cap, int* count) {
    return guard([&] {
        if (sim == nullptr) fail_usage("null simulator");
        const auto r = sim->sim.resident(position);
        if (count) *count = static_cast<int>(r.size());
        if (lines == nullptr) return;
        if (static_cast<int>(r.size()) > cap) fail_usage("line buffer too small");
        std::copy(r.begin(), r.end(), lines);
    });
}
