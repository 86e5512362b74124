// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim over the UNMODIFIED reference headers (tilemul, header-only
// C++20, /root/reference/proj/include). Built by oracle/Makefile into
// oracle/_ref/libtilemul_ref.so with the reference's own RelWithDebInfo flags
// (-O2 -g, no -march; /root/reference/proj/CMakeLists.txt:7-9), so the
// arithmetic is exactly what the reference ships: separate multiply and add,
// no FMA contraction (x86-64 baseline ISA).
//
// Used by tests/ (golden generation and live cross-checks in this
// container) and by bench.py's reference arm (the reference's own execute()
// on the GPU box's host cores). This file contains no reference source; it
// only calls the reference API.
#include <cstdint>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "tilemul/tilemul.hpp"

using namespace tilemul;

namespace {

void put_err(char* err, int errlen, const std::string& msg) {
    if (err == nullptr || errlen <= 0) return;
    std::snprintf(err, static_cast<std::size_t>(errlen), "%s", msg.c_str());
}

CacheHierarchy make_hier(const int64_t* caps, const int* inclusive, int nlev) {
    std::vector<CacheLevel> lv;
    for (int i = 0; i < nlev; ++i) lv.push_back({i, caps[i], 1, inclusive ? inclusive[i] != 0 : false, true, true});
    return CacheHierarchy(std::move(lv));
}

BlocksizeSet make_bs(const int* lvl, const char* dim, const int64_t* val, int n) {
    BlocksizeSet bs;
    for (int i = 0; i < n; ++i) bs.set(lvl[i], dim_from_char(dim[i]), val[i]);
    return bs;
}

// Runs f and maps the reference's exceptions onto the CLI exit-code
// convention (tools/tilemul_main.cpp:519-535): 1 validation/parse/infeasible,
// 2 anything else.
template <typename F>
int guarded(char* err, int errlen, F&& f) {
    try {
        f();
        return 0;
    } catch (const ValidationFailure& e) {
        std::string s;
        for (const auto& v : e.violations) s += v.rule + ":" + std::to_string(v.level) + ":" +
                                                std::to_string(v.lhs) + ":" + std::to_string(v.rhs) + "\n";
        put_err(err, errlen, s);
        return 1;
    } catch (const ParseError& e) {
        put_err(err, errlen, e.rule + "\n");
        return 1;
    } catch (const InfeasibleError& e) {
        put_err(err, errlen, std::string("infeasible: ") + e.what());
        return 1;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return 2;
    }
}

}  // namespace

extern "C" {

// Seeded inputs exactly as cmd_run / acceptance fill them
// (tools/tilemul_main.cpp:236-242): one mt19937_64 stream, uniform(-1,1),
// A then B then C (C only when c != nullptr).
void ref_fill_uniform(uint64_t seed, double* a, int64_t na, double* b, int64_t nb, double* c, int64_t nc) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    for (int64_t i = 0; i < na; ++i) a[i] = dist(rng);
    for (int64_t i = 0; i < nb; ++i) b[i] = dist(rng);
    if (c != nullptr)
        for (int64_t i = 0; i < nc; ++i) c[i] = dist(rng);
}

uint64_t ref_mt19937_64(uint64_t seed, int64_t skip) {
    std::mt19937_64 rng(seed);
    rng.discard(static_cast<unsigned long long>(skip));
    return rng();
}

int ref_parse(const char* name, int* level, char* resident, char* outer, char* inner, int* nplans, char* err,
              int errlen) {
    return guarded(err, errlen, [&] {
        AlgorithmDescriptor d = parse_name(name);
        *nplans = static_cast<int>(d.plans.size());
        for (std::size_t i = 0; i < d.plans.size(); ++i) {
            level[i] = d.plans[i].level;
            resident[i] = to_char(d.plans[i].resident);
            outer[i] = to_char(d.plans[i].outer_dim);
            inner[i] = to_char(d.plans[i].inner_dim);
        }
    });
}

int ref_derive(const char* name, const int64_t* caps, const int* inclusive, int nlev, int64_t m, int64_t n,
               int64_t k, double slack, int64_t mr, int64_t nr, double beta_a, double beta_b, double beta_c,
               const int* pin_level, const char* pin_dim, const int64_t* pin_val, int npin, int* out_level,
               char* out_dim, int64_t* out_val, int* nout, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        AlgorithmDescriptor d = parse_name(name);
        DeriveOptions opts;
        opts.slack = slack;
        opts.micro = MicroTile{mr, nr};
        BlocksizeSet bs = derive_blocksizes(d, make_hier(caps, inclusive, nlev), Shape(m, n, k),
                                            AccessCosts{beta_a, beta_b, beta_c}, opts,
                                            make_bs(pin_level, pin_dim, pin_val, npin));
        int i = 0;
        for (const auto& [key, value] : bs.entries()) {
            out_level[i] = key.level;
            out_dim[i] = to_char(key.dim);
            out_val[i] = value;
            ++i;
        }
        *nout = i;
    });
}

// Returns the number of violations (rules written to `err` one per line as
// rule:level:lhs:rhs), or -1 on a parse error.
int ref_validate(const char* name, const int64_t* caps, const int* inclusive, int nlev, int64_t m, int64_t n,
                 int64_t k, const int* lvl, const char* dim, const int64_t* val, int nbs, char* err, int errlen) {
    int count = -1;
    int rc = guarded(err, errlen, [&] {
        AlgorithmDescriptor d = parse_name(name);
        auto vs = validate_blocksizes(d, make_bs(lvl, dim, val, nbs), make_hier(caps, inclusive, nlev),
                                      Shape(m, n, k));
        std::string s;
        for (const auto& v : vs)
            s += v.rule + ":" + std::to_string(v.level) + ":" + std::to_string(v.lhs) + ":" +
                 std::to_string(v.rhs) + "\n";
        put_err(err, errlen, s);
        count = static_cast<int>(vs.size());
    });
    return rc == 0 ? count : -1;
}

// out: per level h, per operand (A,B,C): reads, writes -> out[(h*3+op)*2 + {0,1}]
int ref_cost(const char* name, const int64_t* caps, const int* inclusive, int nlev, int64_t m, int64_t n,
             int64_t k, const int* lvl, const char* dim, const int64_t* val, int nbs, int64_t* out, char* err,
             int errlen) {
    return guarded(err, errlen, [&] {
        AlgorithmDescriptor d = parse_name(name);
        CostReport rep = multilevel_cost(d, make_bs(lvl, dim, val, nbs), make_hier(caps, inclusive, nlev),
                                         Shape(m, n, k));
        for (const auto& lt : rep.levels)
            for (int op = 0; op < 3; ++op) {
                out[(lt.level * 3 + op) * 2 + 0] = lt.per_operand[static_cast<std::size_t>(op)].reads;
                out[(lt.level * 3 + op) * 2 + 1] = lt.per_operand[static_cast<std::size_t>(op)].writes;
            }
    });
}

int ref_nest(const char* name, const int64_t* caps, const int* inclusive, int nlev, int64_t m, int64_t n,
             int64_t k, const int* lvl, const char* dim, const int64_t* val, int nbs, int* out_level,
             char* out_dim, int64_t* out_bs, int* out_cap, int* nloops, int64_t* cells, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        LoopNest nest = build_plan(parse_name(name), make_bs(lvl, dim, val, nbs), make_hier(caps, inclusive, nlev),
                                   Shape(m, n, k));
        *nloops = static_cast<int>(nest.loops.size());
        for (std::size_t i = 0; i < nest.loops.size(); ++i) {
            out_level[i] = nest.loops[i].level;
            out_dim[i] = to_char(nest.loops[i].dim);
            out_bs[i] = nest.loops[i].blocksize;
            out_cap[i] = nest.loops[i].cap ? 1 : 0;
        }
        if (cells) *cells = nest.cell_count();
    });
}

// The hot path itself: build_plan + execute() on column-major buffers
// (packed=0) or on buffers prepacked in the nest's hierarchical layout
// (packed=1; pack/unpack outside, as cmd_run times only execute()).
// Returns elapsed seconds of execute() in *seconds.
int ref_execute(const char* name, const int64_t* caps, const int* inclusive, int nlev, int64_t m, int64_t n,
                int64_t k, const int* lvl, const char* dim, const int64_t* val, int nbs, const double* a,
                const double* b, double* c, int workers, int parallel_loop, int packed, double* seconds,
                char* err, int errlen) {
    return guarded(err, errlen, [&] {
        LoopNest nest = build_plan(parse_name(name), make_bs(lvl, dim, val, nbs), make_hier(caps, inclusive, nlev),
                                   Shape(m, n, k));
        MatrixBuffer A = MatrixBuffer::column_major(Operand::A, m, k);
        MatrixBuffer B = MatrixBuffer::column_major(Operand::B, k, n);
        MatrixBuffer C = MatrixBuffer::column_major(Operand::C, m, n);
        std::memcpy(A.data.data(), a, sizeof(double) * static_cast<std::size_t>(m * k));
        std::memcpy(B.data.data(), b, sizeof(double) * static_cast<std::size_t>(k * n));
        std::memcpy(C.data.data(), c, sizeof(double) * static_cast<std::size_t>(m * n));
        ExecOptions opts;
        opts.workers = workers;
        opts.parallel_loop = parallel_loop;
        double el = 0;
        if (packed) {
            MatrixBuffer Ap = pack(A, nest), Bp = pack(B, nest), Cp = pack(C, nest);
            auto t0 = std::chrono::steady_clock::now();
            execute(nest, Ap, Bp, Cp, opts);
            el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            C = unpack(Cp);
        } else {
            auto t0 = std::chrono::steady_clock::now();
            execute(nest, A, B, C, opts);
            el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
        if (seconds) *seconds = el;
        std::memcpy(c, C.data.data(), sizeof(double) * static_cast<std::size_t>(m * n));
    });
}

// Zero-copy variant for large timed samples: views the caller's arrays
// through MatrixBuffers that own copies only once per call setup.
void ref_reference_gemm(int64_t m, int64_t n, int64_t k, const double* a, const double* b, double* c) {
    MatrixBuffer A = MatrixBuffer::column_major(Operand::A, m, k);
    MatrixBuffer B = MatrixBuffer::column_major(Operand::B, k, n);
    MatrixBuffer C = MatrixBuffer::column_major(Operand::C, m, n);
    std::memcpy(A.data.data(), a, sizeof(double) * static_cast<std::size_t>(m * k));
    std::memcpy(B.data.data(), b, sizeof(double) * static_cast<std::size_t>(k * n));
    std::memcpy(C.data.data(), c, sizeof(double) * static_cast<std::size_t>(m * n));
    reference_gemm(A, B, C);
    std::memcpy(c, C.data.data(), sizeof(double) * static_cast<std::size_t>(m * n));
}

void ref_micro_kernel(const double* a, int64_t lda, const double* b, int64_t ldb, double* c, int64_t ldc,
                      int64_t mr, int64_t nr, int64_t kc) {
    std::vector<double> acc(static_cast<std::size_t>(mr * nr > 0 ? mr * nr : 1));
    micro_kernel(a, lda, b, ldb, c, ldc, mr, nr, kc, acc.data());
}

void ref_io_lower_bound(int64_t m, int64_t n, int64_t k, int64_t M, int64_t* reads, int64_t* writes) {
    OperandTraffic t = io_lower_bound(Shape(m, n, k), M);
    *reads = t.reads;
    *writes = t.writes;
}

// out[op*2 + {0,1}]
void ref_resident_cost(char variant, int64_t m, int64_t n, int64_t k, int64_t b1, int64_t b2, int64_t* out) {
    LevelTraffic t = resident_cost(operand_from_char(variant), Shape(m, n, k), b1, b2);
    for (int op = 0; op < 3; ++op) {
        out[op * 2] = t.per_operand[static_cast<std::size_t>(op)].reads;
        out[op * 2 + 1] = t.per_operand[static_cast<std::size_t>(op)].writes;
    }
}

double ref_streaming_efficiency(char variant, int64_t b1, int64_t b2) {
    return streaming_efficiency(operand_from_char(variant), b1, b2);
}

double ref_goto_efficiency(int64_t kc, int64_t nc) { return goto_efficiency(kc, nc); }

// pack(src, nest) for one operand (plan.hpp:122-124 / layout.hpp:122-135):
// column-major src -> dst in layout_for(nest, op).
int ref_pack(const char* name, const int64_t* caps, const int* inclusive, int nlev, int64_t m, int64_t n, int64_t k,
             const int* lvl, const char* dim, const int64_t* val, int nbs, char op, const double* src, double* dst,
             char* err, int errlen) {
    return guarded(err, errlen, [&] {
        LoopNest nest = build_plan(parse_name(name), make_bs(lvl, dim, val, nbs), make_hier(caps, inclusive, nlev),
                                   Shape(m, n, k));
        Operand o = operand_from_char(op);
        MatrixBuffer b = MatrixBuffer::column_major(o, nest.shape.rows(o), nest.shape.cols(o));
        std::memcpy(b.data.data(), src, sizeof(double) * b.data.size());
        MatrixBuffer p = pack(b, nest);
        std::memcpy(dst, p.data.data(), sizeof(double) * p.data.size());
    });
}

char ref_select(int64_t m, int64_t n, int64_t k, int64_t cap) { return to_char(select_algorithm(Shape(m, n, k), cap)); }

// --- trace generator and LRU simulator (trace.hpp, cachesim.hpp) ----------
// Hierarchy with every CacheLevel field: flags[3*i] = inclusive,
// [3*i+1] = write_allocate, [3*i+2] = write_back.
static CacheHierarchy make_hier_flags(const int64_t* caps, const int64_t* gran, const int* flags, int nlev) {
    std::vector<CacheLevel> lv;
    for (int i = 0; i < nlev; ++i)
        lv.push_back({i, caps[i], gran[i], flags[3 * i] != 0, flags[3 * i + 1] != 0, flags[3 * i + 2] != 0});
    return CacheHierarchy(std::move(lv));
}

// 15 values per simulated level: level, capacity_lines, granularity, hits,
// read_misses, write_misses, fetched_lines, passthrough_writes, writebacks,
// per_operand_misses[A,B,C], per_operand_writebacks[A,B,C].
static void put_stats(const SimResult& r, int64_t* out, int* nout, int64_t* events) {
    int i = 0;
    for (const auto& s : r.levels) {
        int64_t* o = out + 15 * i++;
        const int64_t v[9] = {s.level, s.capacity_lines, s.granularity, s.hits, s.read_misses, s.write_misses,
                              s.fetched_lines, s.passthrough_writes, s.writebacks};
        for (int q = 0; q < 9; ++q) o[q] = v[q];
        for (int q = 0; q < 3; ++q) {
            o[9 + q] = s.per_operand_misses[static_cast<std::size_t>(q)];
            o[12 + q] = s.per_operand_writebacks[static_cast<std::size_t>(q)];
        }
    }
    *nout = i;
    *events = r.events;
}

static Operand op_of(char c) { return c == 'A' ? Operand::A : c == 'B' ? Operand::B : Operand::C; }

// LruSimulator over an explicit event list.
int ref_sim_events(const int64_t* caps, const int64_t* gran, const int* flags, int nlev, int64_t m, int64_t n,
                   int64_t k, int include_registers, int flush, const char* ops, const int64_t* idx,
                   const uint8_t* writes, int64_t count, int64_t* out, int* nout, int64_t* events, char* err,
                   int errlen) {
    return guarded(err, errlen, [&] {
        SimOptions o;
        o.include_registers = include_registers != 0;
        o.flush_dirty_at_end = flush != 0;
        LruSimulator sim(make_hier_flags(caps, gran, flags, nlev), Shape(m, n, k), o);
        for (int64_t e = 0; e < count; ++e)
            sim.access({op_of(ops[e]), idx[e], writes[e] ? AccessKind::write : AccessKind::read});
        put_stats(sim.finish(), out, nout, events);
    });
}

// simulate(build_plan(name, plan hierarchy, shape, bs), layouts, sim hierarchy).
int ref_simulate(const char* name, const int64_t* caps, const int* inclusive, int nlev, int64_t m, int64_t n,
                 int64_t k, const int* bl, const char* bd, const int64_t* bv, int nb, const int64_t* scaps,
                 const int64_t* sgran, const int* sflags, int snlev, int packed, int include_registers, int flush,
                 int64_t* out, int* nout, int64_t* events, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        Shape shape(m, n, k);
        LoopNest nest = build_plan(parse_name(name), make_bs(bl, bd, bv, nb), make_hier(caps, inclusive, nlev), shape);
        SimOptions o;
        o.include_registers = include_registers != 0;
        o.flush_dirty_at_end = flush != 0;
        const TraceLayouts lay = packed ? TraceLayouts::packed(nest) : TraceLayouts::column_major(shape);
        put_stats(simulate(nest, lay, make_hier_flags(scaps, sgran, sflags, snlev), o), out, nout, events);
    });
}

// The first `cap` events of generate_trace; *count = trace_event_count.
int ref_trace(const char* name, const int64_t* caps, const int* inclusive, int nlev, int64_t m, int64_t n, int64_t k,
              const int* bl, const char* bd, const int64_t* bv, int nb, int packed, int64_t cap, char* ops,
              int64_t* idx, uint8_t* writes, int64_t* count, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        Shape shape(m, n, k);
        LoopNest nest = build_plan(parse_name(name), make_bs(bl, bd, bv, nb), make_hier(caps, inclusive, nlev), shape);
        const TraceLayouts lay = packed ? TraceLayouts::packed(nest) : TraceLayouts::column_major(shape);
        int64_t e = 0;
        generate_trace(nest, lay, [&](const TraceEvent& t) {
            if (e < cap) {
                ops[e] = to_char(t.op);
                idx[e] = t.index;
                writes[e] = t.kind == AccessKind::write ? 1 : 0;
            }
            ++e;
        });
        *count = trace_event_count(nest);
    });
}

// pareto_sweep (costmodel.hpp:299-328): 8 values per point, in ParetoPoint field order.
int ref_pareto(int64_t outer, const double* ratios, int nratios, int64_t m, int64_t n, int64_t k, double slack,
               int64_t mr, int64_t nr, double* out, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        DeriveOptions o;
        o.slack = slack;
        o.micro = MicroTile{mr, nr};
        const auto pts = pareto_sweep(outer, std::vector<double>(ratios, ratios + nratios), Shape(m, n, k), o);
        int i = 0;
        for (const auto& p : pts) {
            const double v[8] = {p.ratio, static_cast<double>(p.inner_capacity), static_cast<double>(p.outer_block_k),
                                 static_cast<double>(p.outer_block_n), static_cast<double>(p.inner_block_m),
                                 static_cast<double>(p.inner_block_k), p.eff_outer_flops_per_element,
                                 p.eff_inner_flops_per_element};
            for (int q = 0; q < 8; ++q) out[8 * i + q] = v[q];
            ++i;
        }
    });
}

}  // extern "C"
