// C ABI (include/tilemul_b200.h) over the host library (csrc/host), the
// lowering and execution engine (engine.hpp: lower.cpp, host_pipe.cpp) and
// the sm_100a kernels. Every entry converts C++ failures to status codes
// (guard) and keeps the message thread-local (tm_last_error).
//
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "engine.hpp"
#include "host/cachesim.hpp"

using namespace mmm;
using mmm::engine::cuda_check;

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

}  // namespace

using namespace mmm::engine;

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
    return guard([&] { execute_host(plan, A, B, C, opts); });
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
        if (o.tile_n != 0 && o.tile_n != 256 && o.tile_n != 512) fail_usage("tensor-core tile_n must be 256 or 512");
        const bool pair = o.tile != 128;
        if (!pair && o.tile_n == 512) fail_usage("512-column tiles run on SM pairs only");
        // SM pairs default to 256 x 512 tiles: 25 % fewer L2->SMEM bytes per flop than 256 x 256, which
        // under the board power cap buys clock (config 4)
        const bool wide = pair && o.tile_n != 256;
        const bool tf32 = dtype == TM_DTYPE_TF32;
        const gpu::Kernel kernel = wide   ? (tf32 ? gpu::kTc2wTf32 : gpu::kTc2wBf16)
                                   : pair ? (tf32 ? gpu::kTc2Tf32 : gpu::kTc2Bf16)
                                          : (tf32 ? gpu::kTcTf32 : gpu::kTcBf16);
        std::lock_guard<std::mutex> lk(plan->mu);
        Key key{o.schedule, kernel, 1, o.ctas, false};
        auto& slot = plan->schedules[key];
        int dev = 0;
        cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
        if (!slot || slot->device != dev) slot = lower(plan->nest, o, kernel, static_cast<cudaStream_t>(stream));
        Schedule& s = *slot;
        const int nt = static_cast<int>(s.host_tasks.size());
        cuda_check(pair ? gpu::launch_tc_pair(dtype == TM_DTYPE_TF32, A, lda, B, ldb, C, ldc, e.m, e.n, e.k, s.tasks,
                                              nt, s.grid, static_cast<cudaStream_t>(stream), wide)
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

int tm_plan_last_staging(const tm_plan* plan, int32_t* staging) {
    return guard([&] {
        if (staging) *staging = plan->last_staging;
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

int tm_measure_tc_peak(int dtype, int launches, int sustained, double* tflops) {
    return guard([&] {
        if (dtype != TM_DTYPE_BF16 && dtype != TM_DTYPE_TF32) fail_usage("dtype must be TM_DTYPE_BF16 or TM_DTYPE_TF32");
        if (!tflops) fail_usage("null output");
        cuda_check(gpu::measure_tc_peak(dtype == TM_DTYPE_TF32, launches < 1 ? 1 : launches, sustained != 0, tflops),
                   "tensor-core peak probe");
    });
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
