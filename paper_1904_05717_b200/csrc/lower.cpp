// Lowering of a loop nest onto CTA tasks and its execution on device
// buffers (the blocked-loop driver, reference plan.hpp:61-84 +
// exec.hpp:94-138, re-targeted): a task is one C region x k range run by one
// CTA with its accumulators in registers. Two schedules:
//   fused    — every k loop of the nest is sunk below its m/n loops, so each
//              register-level C block is visited once, in the order of its
//              first appearance in the nest (the m/n loops above it become the
//              CTA raster: the L2-level plan sets which tiles share a wave).
//              Optional split-k, finished in a fixed slot order.
//   faithful — one task per nest cell, in nest order; cells of the same C
//              block run in ascending k (per-region progress counters), so
//              the C block round-trips to memory per cell exactly as the
//              reference's micro-kernel does.
// Either way every C entry is accumulated in ascending k from its incoming
// value, which is what makes the result independent of the schedule.
#include <algorithm>
#include <array>
#include <cstring>
#include <functional>
#include <tuple>
#include <unordered_map>

#include "engine.hpp"

namespace mmm {
namespace engine {

namespace {
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

// The nest walk (Nest::walk, plan.hpp:61-84) also reporting, per cell, the
// iteration index of loop `par` at the visit that produced it (0 if par < 0).
void walk_indexed_rec(const Nest& nest, std::size_t depth, int par, i64 widx, std::array<i64, 3> org,
                      std::array<i64, 3> ext, const std::function<void(const Cell&, i64)>& f) {
    if (depth == nest.loops.size()) {
        f(Cell{org[0], ext[0], org[1], ext[1], org[2], ext[2]}, widx);
        return;
    }
    const Loop& L = nest.loops[depth];
    const int d = L.dim;
    const i64 lo = org[d], hi = org[d] + ext[d];
    i64 it = 0;
    for (i64 s0 = lo; s0 < hi; s0 += L.size, ++it) {
        org[d] = s0;
        ext[d] = std::min(L.size, hi - s0);
        walk_indexed_rec(nest, depth + 1, par, static_cast<int>(depth) == par ? it : widx, org, ext, f);
    }
}
void walk_indexed(const Nest& nest, int par, const std::function<void(const Cell&, i64)>& f) {
    walk_indexed_rec(nest, 0, par, 0, {0, 0, 0}, {nest.ext.m, nest.ext.n, nest.ext.k}, f);
}

}  // namespace

int sm_count() {
    int dev = 0, sms = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "cudaDeviceGetAttribute");
    return sms;
}

gpu::Kernel pick_tc_kernel(int dtype, const tm_exec_opts& o) {
    const bool pair = o.tile != 128;
    // SM pairs default to 256 x 512 tiles: 25 % fewer L2->SMEM bytes per flop than 256 x 256, which
    // under the board power cap buys clock (config 4)
    const bool wide = pair && o.tile_n != 256;
    const bool tf32 = dtype == TM_DTYPE_TF32;
    return wide ? (tf32 ? gpu::kTc2wTf32 : gpu::kTc2wBf16)
                : pair ? (tf32 ? gpu::kTc2Tf32 : gpu::kTc2Bf16) : (tf32 ? gpu::kTcTf32 : gpu::kTcBf16);
}

gpu::Kernel pick_kernel(const Nest& nest, const tm_exec_opts& o, bool tma) {
    const bool small_tile = o.tile == 64 || (o.tile == 0 && (nest.m_r < 128 || nest.n_r < 128));
    if (o.tile != 0 && o.tile != 64 && o.tile != 128) fail_usage("tile must be 0, 64 or 128");
    const int tn = o.tile_n == 0 ? o.tile : o.tile_n;
    if (o.tile_n != 0 && !((o.tile == 128 && (tn == 64 || tn == 128)) || (o.tile == 64 && tn == 64)))
        fail_usage("tile x tile_n must be 128x128, 128x64 or 64x64");
    switch (o.numerics) {
        case TM_NUMERICS_DMMA:
            if (o.tile == 128 && tn == 64) return gpu::kDmma128x64;
            // short k: every task is mostly C load/store. With TMA staging the
            // 128 x 128 kernel's producer loads the next tile's first slabs
            // under this tile's C write-back (rank-k 16384^2 x 256: 87.3 % of
            // peak); with cp.async, two CTAs per SM (128 x 64 tiles) hide one
            // CTA's C traffic behind the other's DMMAs (84.1 %).
            if (o.tile == 0 && !small_tile && nest.ext.k <= 512 && o.schedule == TM_SCHEDULE_FUSED && !tma)
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
HostSchedule plan_tasks(const Nest& nest, const tm_exec_opts& o, gpu::Kernel kernel, int tile_m, int tile_n,
                        int slots) {
    HostSchedule hs;
    struct {
        int tile_m, tile_n;
    } info{tile_m, tile_n};
    const Extents& e = nest.ext;
    check_i32(e.m, "m");
    check_i32(e.n, "n");
    check_i32(e.k, "k");
    auto& T = hs.tasks;

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
        // Round 2: auto also takes stream-K whenever the tiles do not fill whole waves and the launch is
        // short (at most 4096 k-slabs per CTA: one TMA launch, no segments, which need whole rounds).
        // Measured back to back against the per-tile / tail splits (profiles/ab_r02_streamk_auto.json):
        // 512^2 x 131072 92.5 -> 95.2 %, 1024^2 x 65536 82.8 -> 96.1 %, rank-k 90.4 -> 91.5 %,
        // 65536 x 256 x 1024 92.5 -> 93.2 %.
        static const int sk_knob = [] {  // TILEMUL_STREAMK_AUTO=0: A/B knob
            const char* env = std::getenv("TILEMUL_STREAMK_AUTO");
            return env ? std::atoi(env) : 1;
        }();
        const i64 nks_all = cdiv(e.k, static_cast<i64>(32));
        const bool short_uneven = sk_knob && ntiles % slots != 0 && ntiles * nks_all <= int64_t{4096} * slots;
        if (dmma && (o.split_k == -1 || (o.split_k == 0 && ((ragged && e.k >= 2048) || short_uneven)))) {
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
            hs.blocked = true;
            hs.grid_fixed = G;
            hs.first = std::move(first);
            hs.fixup = fixk;
            hs.slots = next_slot;
            hs.counters = fixk ? ncounters : 0;
            if (!fixk) hs.red = std::move(red);
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
        hs.fixup = fix;
        hs.slots = next_slot;
        hs.counters = fix ? ncounters : 0;
        hs.red = std::move(red);
        }  // uniform / tail split
    } else if (o.schedule == TM_SCHEDULE_FAITHFUL) {
        const i64 cells = nest.cells();
        if (cells > 64LL * 1000 * 1000) fail_usage("faithful schedule limited to 64M cells; use the fused schedule");
        // The reference runs a chosen m/n loop's iterations on separate
        // workers, each walking its share in nest order (plan.hpp:49-84,
        // exec.hpp:106-131). Here every iteration of that loop is a worker and
        // the workers' task lists are interleaved, so the CTAs in flight hold
        // independent C regions; a region's cells keep their nest order
        // (progress counters), and every wait points at an earlier task.
        // Default: plain nest order (the CTAs take consecutive cells), which
        // reproduces the member's traffic (0.95-1.03x its model, DESIGN.md
        // 5.3). Naming an m/n loop splits its iterations into workers like the
        // reference's threads: an outer one (e.g. m1 of B2A1C0) runs several
        // resident blocks at once -- far more parallel, but their combined
        // working set no longer matches the member's model.
        const int nl = static_cast<int>(nest.loops.size());
        int par = o.parallel_loop - 1;
        if (o.parallel_loop == 0) {
            par = -1;
        } else {
            if (par < 0 || par >= nl) fail_usage("parallel loop index out of range");
            if (nest.loops[static_cast<std::size_t>(par)].dim == kK)
                fail_usage("cannot parallelize a k-dimension loop: workers would accumulate into shared C");
        }
        std::vector<std::vector<gpu::Task>> workers(1);
        std::unordered_map<i64, std::pair<int32_t, int32_t>> regions;  // key -> (id, next seq)
        walk_indexed(nest, par, [&](const Cell& c, i64 w) {
            if (static_cast<std::size_t>(w) >= workers.size()) workers.resize(static_cast<std::size_t>(w) + 1);
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
                workers[static_cast<std::size_t>(w)].push_back(tk);
            });
        });
        // merge by relative position so unequal workers (margins) advance in
        // proportion to their size: task r of a worker of n tasks sorts at
        // (r + 1/2) / n
        std::vector<std::tuple<double, std::size_t, std::size_t>> order;
        for (std::size_t w = 0; w < workers.size(); ++w)
            for (std::size_t r = 0; r < workers[w].size(); ++r)
                order.emplace_back((static_cast<double>(r) + 0.5) / static_cast<double>(workers[w].size()), w, r);
        std::sort(order.begin(), order.end());
        for (const auto& [key, w, r] : order) T.push_back(workers[w][r]);
        hs.regions = static_cast<int>(regions.size());
    } else {
        fail_usage("unknown schedule");
    }
    if (T.size() > static_cast<std::size_t>(INT32_MAX)) fail_usage("too many tasks");
    return hs;
}

gpu::KernelInfo kernel_tiles(gpu::Kernel kernel, bool query) {
    const bool wide = kernel == gpu::kTc2wBf16 || kernel == gpu::kTc2wTf32;
    const bool pair = kernel == gpu::kTc2Bf16 || kernel == gpu::kTc2Tf32 || wide;
    if (kernel == gpu::kTcBf16 || kernel == gpu::kTcTf32)
        return gpu::KernelInfo{128, 256, 256, query ? gpu::tc_smem_bytes(kernel == gpu::kTcTf32) : 0, 1};
    if (wide) return gpu::KernelInfo{256, 512, 384, query ? gpu::tc2_smem_bytes(kernel == gpu::kTc2wTf32, true) : 0, 1};
    if (pair) return gpu::KernelInfo{256, 256, 256, query ? gpu::tc2_smem_bytes(kernel == gpu::kTc2Tf32) : 0, 1};
    if (query) {
        gpu::KernelInfo info{};
        cuda_check(gpu::kernel_info(kernel, &info), "kernel_info");
        return info;
    }
    // the DMMA / SIMT tiles and their occupancy (gpu::kernel_info measures it on a device)
    switch (kernel) {
        case gpu::kDmma128: return gpu::KernelInfo{128, 128, 512, 0, 1};
        case gpu::kDmma128x64: return gpu::KernelInfo{128, 64, 128, 0, 2};
        case gpu::kFma128: return gpu::KernelInfo{128, 128, 256, 0, 1};
        default: return gpu::KernelInfo{64, 64, 128, 0, 1};
    }
}

std::unique_ptr<Schedule> lower(const Nest& nest, const tm_exec_opts& o, gpu::Kernel kernel, cudaStream_t stream,
                                bool upload) {
    auto s = std::make_unique<Schedule>();
    s->kernel = kernel;
    const gpu::KernelInfo info = kernel_tiles(kernel, true);
    const bool wide = kernel == gpu::kTc2wBf16 || kernel == gpu::kTc2wTf32;
    const bool pair = kernel == gpu::kTc2Bf16 || kernel == gpu::kTc2Tf32 || wide;
    const int slots = sm_count() * std::max(1, info.ctas_per_sm);
    HostSchedule hs = plan_tasks(nest, o, kernel, info.tile_m, info.tile_n, slots);
    s->host_tasks = std::move(hs.tasks);
    auto& T = s->host_tasks;
    if (!upload) return s;  // host task list only (callers that splice task lists)
    if (hs.blocked) {
        s->blocked = true;
        s->grid_fixed = hs.grid_fixed;
        cuda_check(cudaMalloc(&s->cta_first, sizeof(int32_t) * hs.first.size()), "cudaMalloc(cta ranges)");
        cuda_check(cudaMemcpyAsync(s->cta_first, hs.first.data(), sizeof(int32_t) * hs.first.size(),
                                   cudaMemcpyHostToDevice, stream),
                   "upload cta ranges");
    }
    if (hs.fixup) alloc_fixup(*s, info, hs.slots, hs.counters, stream);
    if (!hs.red.empty()) {
        s->slices = static_cast<int>(hs.red.size());
        s->work_ld = info.tile_m;
        s->work_slice = static_cast<i64>(info.tile_m) * info.tile_n;
        cuda_check(cudaMalloc(&s->work, sizeof(double) * static_cast<std::size_t>(s->work_slice) * hs.slots),
                   "cudaMalloc(split-k workspace)");
        cuda_check(cudaMalloc(&s->reduce, sizeof(gpu::ReduceTile) * hs.red.size()), "cudaMalloc(reduce list)");
        cuda_check(cudaMemcpyAsync(s->reduce, hs.red.data(), sizeof(gpu::ReduceTile) * hs.red.size(),
                                   cudaMemcpyHostToDevice, stream),
                   "upload reduce list");
    }
    if (hs.regions > 0) {
        s->regions = hs.regions;
        cuda_check(cudaMalloc(&s->progress, sizeof(int32_t) * static_cast<std::size_t>(s->regions)),
                   "cudaMalloc(progress)");
    }
    // Persistent grid: every CTA must be co-resident for the faithful
    // schedule's waits to make progress.
    int grid = o.ctas > 0 ? std::min(o.ctas, slots) : slots;
    s->grid = std::max(1, std::min<int>(grid, static_cast<int>(T.size())));
    if (pair) s->grid = 2 * std::max(1, std::min<int>(slots / 2, static_cast<int>(T.size())));  // clusters of 2
    // 256 x 512 pair tiles run one tile per cluster (not persistent): a fresh cluster starts each tile, so the
    // clusters in flight are always a window of consecutive raster tiles and share their A/B panels in L2
    // (16384^3 bf16: 8.9 GB of HBM reads per launch vs 18.3 GB persistent; the 512-column accumulator leaves
    // no second TMEM buffer to overlap an epilogue with anyway)
    if (wide) s->grid = 2 * std::max(1, static_cast<int>(T.size()));
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

int launch_tasks(Schedule& s, const gpu::Args& a, int64_t M, int64_t N, int64_t K, bool vec16, int32_t staging,
                 cudaStream_t stream, bool long_ok) {
    if (staging < TM_STAGING_AUTO || staging > TM_STAGING_TMA) fail_usage("staging must be 0 (auto), 1 (cp.async) or 2 (TMA)");
    const int bk = gpu::tma_bk(s.kernel);
    if (staging == TM_STAGING_TMA && bk == 0) fail_usage("TMA staging exists for the DMMA kernels only");
    if (bk > 0 && s.tma_ok < 0) {
        s.tma_ok = 1;
        int64_t slabs = 0;
        for (const auto& t : s.host_tasks) {
            if (t.k % bk != 0 && static_cast<int64_t>(t.p0) + t.k != K) s.tma_ok = 0;
            slabs += (t.k + bk - 1) / bk;
        }
        s.slabs_per_cta = slabs / std::max(1, s.grid);
    }
    // Auto takes TMA for the 128x128 kernel in launches in which a CTA
    // streams at most kTmaAutoMaxSlabs k-slabs (longer task lists: segments,
    // below). Measured on one B200 (DESIGN.md
    // 4.2): TMA is 0.4-1.7 points of FP64 peak faster than cp.async on every
    // config, but its CTAs drift apart over a long launch (the copies never
    // stall them), so the CTAs of a wave stop reading shared A/B panels
    // within L2's reach. HBM reads over cp.async's grow with the launch's
    // length in slabs per CTA: 1.2x at ~7k (8192^3, 1.32x the model), 1.6x at
    // ~14k, 2.2x at ~28k, 5.5x at ~56k (16384^3). A wave gate (CTAs of a
    // round wait for the round's average progress) restored the traffic but
    // cost 2-4 points, more than TMA gains (profiles/tma_l2_r01.json). The
    // 128x64 / 64x64 TMA variants trail cp.async by 0.5-4 points.
    // A long strided task list is launched in segments of whole rounds (task
    // r*G .. r*G+G-1 on CTA 0..G-1) of at most kTmaSegmentSlabs slabs per
    // CTA: each kernel boundary brings the wave back in step. 16384^3 in 14
    // segments of 4096 slabs: 54 GB of HBM reads per step (1.15x the model,
    // cp.async's traffic; 69 GB with 8192-slab segments, 283 GB as one
    // launch) at cp.async's 95.5 % of peak.
    constexpr int64_t kTmaAutoMaxSlabs = 4096;
    static const int64_t kTmaSegmentSlabs = [] {  // (TILEMUL_TMA_SEGMENT_SLABS: A/B knob)
        const char* env = std::getenv("TILEMUL_TMA_SEGMENT_SLABS");
        return env ? std::max<int64_t>(1, std::atoll(env)) : int64_t{4096};
    }();
    s.last_launches = 1;
    if (bk > 0 && staging == TM_STAGING_AUTO && s.kernel == gpu::kDmma128 && !long_ok && !s.blocked &&
        s.slabs_per_cta > kTmaAutoMaxSlabs && s.tma_ok == 1 && vec16) {
        if (s.segments.empty()) {
            const std::size_t G = static_cast<std::size_t>(std::max(1, s.grid)), nt = s.host_tasks.size();
            s.segments.push_back(0);
            int64_t acc = 0, longest = 0;
            for (std::size_t r0 = 0; r0 < nt; r0 += G) {
                const int64_t round = (s.host_tasks[r0].k + bk - 1) / bk;
                if (acc > 0 && acc + round > kTmaSegmentSlabs) {
                    s.segments.push_back(static_cast<int32_t>(r0));
                    acc = 0;
                }
                acc += round;
                longest = std::max(longest, acc);
            }
            s.segments.push_back(static_cast<int32_t>(nt));
            // rounds too long to cut (one task of > kTmaAutoMaxSlabs slabs per CTA): cp.async
            if (longest > kTmaAutoMaxSlabs) s.segments.assign({-1});
        }
        bool ok = s.segments.front() == 0;
        for (std::size_t q = 0; q + 1 < s.segments.size() && ok; ++q) {
            gpu::Args sa = a;
            sa.tasks = a.tasks + s.segments[q];
            sa.ntasks = s.segments[q + 1] - s.segments[q];
            static const int pdl_knob = [] {  // TILEMUL_TMA_PDL=0: A/B knob
                const char* env = std::getenv("TILEMUL_TMA_PDL");
                return env ? std::atoi(env) : 1;
            }();
            // segments after the first start their CTAs as the previous segment's CTAs retire (programmatic
            // dependent launch): the segments' tasks are distinct C tiles, and split parts straddling a
            // segment boundary synchronise through the fix-up counters, never through launch order
            const cudaError_t r = gpu::launch_tma(s.kernel, sa, M, N, K, std::min(s.grid, sa.ntasks), stream,
                                                  q > 0 && pdl_knob);
            if (r == cudaErrorNotSupported && q == 0) ok = false;  // (decided before any launch)
            else cuda_check(r, "task kernel launch (TMA segment)");
        }
        if (ok) {
            s.last_launches = static_cast<int>(s.segments.size()) - 1;
            return TM_STAGING_TMA;
        }
    }
    const bool want = staging == TM_STAGING_TMA ||
                      (staging == TM_STAGING_AUTO && s.kernel == gpu::kDmma128 &&
                       (long_ok || s.slabs_per_cta <= kTmaAutoMaxSlabs));
    if (bk > 0 && want) {
        // TMA boxes start on 16-byte boundaries of a column: the alignment the
        // 16-byte cp.async path needs too (even task origins, even ld, aligned bases)
        cudaError_t r = cudaErrorNotSupported;
        if (s.tma_ok == 1 && vec16) {
            r = gpu::launch_tma(s.kernel, a, M, N, K, s.grid, stream);
            if (r == cudaSuccess) return TM_STAGING_TMA;
            if (r != cudaErrorNotSupported) cuda_check(r, "task kernel launch (TMA)");
        }
        if (staging == TM_STAGING_TMA)
            fail_usage("TMA staging does not apply: A/B, their leading dimensions or the task origins are not "
                       "16-byte aligned, or a task's k range is not a whole number of slabs");
    }
    cuda_check(gpu::launch(s.kernel, vec16, a, s.grid, stream), "task kernel launch");
    return bk > 0 ? TM_STAGING_CPASYNC : 0;
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
    const bool tma_hint = o.staging != TM_STAGING_CPASYNC && lda % 2 == 0 && ldb % 2 == 0 &&
                          reinterpret_cast<uintptr_t>(A) % 16 == 0 && reinterpret_cast<uintptr_t>(B) % 16 == 0;
    const gpu::Kernel kernel = pick_kernel(plan->nest, o, tma_hint);
    std::lock_guard<std::mutex> lk(plan->mu);
    Key key{o.schedule, kernel, o.schedule == TM_SCHEDULE_FUSED ? o.split_k : 0, o.ctas, false,
            o.schedule == TM_SCHEDULE_FAITHFUL ? o.parallel_loop : 0};
    auto& slot = plan->schedules[key];
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    if (!slot || slot->device != dev) slot = lower(plan->nest, o, kernel, stream);
    Schedule& s = *slot;
    const bool vec16 = (lda % 2 == 0) && (ldb % 2 == 0) && (reinterpret_cast<uintptr_t>(A) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(B) % 16 == 0) && origins_even(s.host_tasks);
    // this plan's previous launch (any stream) is done with the shared scratch before this one starts
    if (!plan->order) cuda_check(cudaEventCreateWithFlags(&plan->order, cudaEventDisableTiming), "order event");
    else cuda_check(cudaStreamWaitEvent(stream, plan->order, 0), "order after the previous launch");
    if (s.regions > 0)
        cuda_check(cudaMemsetAsync(s.progress, 0, sizeof(int32_t) * static_cast<std::size_t>(s.regions), stream),
                   "reset progress");
    gpu::Args a{A, lda, B, ldb, C, ldc, s.tasks, static_cast<int32_t>(s.host_tasks.size()), s.progress, s.work,
                s.work_ld, s.work_slice, s.blocked ? s.cta_first : nullptr};
    plan->last_staging = launch_tasks(s, a, e.m, e.n, e.k, vec16, o.staging, stream);
    int launches = s.last_launches;
    if (s.slices > 0) {
        cuda_check(gpu::launch_reduce_tiles(C, ldc, s.work, s.work_ld, s.work_slice, s.reduce, s.slices, stream),
                   "split-k reduce launch");
        ++launches;
    }
    cuda_check(cudaEventRecord(plan->order, stream), "record launch order");
    plan->last_tasks = static_cast<int64_t>(s.host_tasks.size());
    plan->last_launches = launches;
    plan->last_ctas = s.grid;
}

}  // namespace engine
}  // namespace mmm
