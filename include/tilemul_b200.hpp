/* Header-only C++ shim: the reference's `tilemul::execute` signature over the
 * B200 C ABI (tilemul_b200.h), for a maintainer who swaps the call in place
 * (INTEGRATION.md §1).
 *
 * Include after the reference's own headers (it uses tilemul::LoopNest,
 * MatrixBuffer, CacheHierarchy and the exception types from
 * /root/reference/proj/include/tilemul/{plan,layout,cache,types}.hpp) and link
 * paper_1904_05717_b200/lib/libtilemul_b200.so.
 *
 *   reference                                  this shim
 *   execute(nest, A, B, C, opts)               tilemul::b200::execute(nest, A, B, C, opts)
 *     exec.hpp:94-95                             -- the same signature: the native plan is built from
 *                                                 the nest's own loops, m_r, n_r and shape
 *                                                 (tm_plan_create_loops) and cached per nest, so
 *                                                 repeated calls reuse its lowering and device buffers
 *   build_plan(d, bs, hier, shape)             b200::Plan(nest, hier): re-validated against `hier`
 *     plan.hpp:90-108                            with the reference's rules; carries the I/O model
 *   std::invalid_argument (exec.hpp:67-84,     status 2 (usage) / 3 (CUDA) -> std::invalid_argument /
 *     :99, :127-131)                             std::runtime_error
 *   ValidationFailure / ParseError /           status 1 -> the same types, violations rebuilt from
 *     InfeasibleError (types.hpp:148-174)        tm_last_rules() ("rule:level:lhs:rhs" lines)
 *
 * Buffers may be column-major or prepacked in the nest's layout (layout_for),
 * like the reference; checks on roles, extents and layouts are the
 * reference's own (detail::check_buffer), so the same inputs raise the same
 * errors. Numerics: Options::numerics = TM_NUMERICS_EXACT reproduces the
 * reference's execute() bit for bit (DMUL then DADD per step, ascending k
 * from C's incoming value); TM_NUMERICS_DMMA (default) is the FP64 tensor
 * pipe, within 4·k·u·(|A||B|)_ij of it. */
#pragma once

#include <list>
#include <memory>
#include <mutex>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "tilemul/exec.hpp"
#include "tilemul/layout.hpp"
#include "tilemul/plan.hpp"
#include "tilemul/types.hpp"
#include "tilemul_b200.h"

namespace tilemul::b200 {

struct Options {
    int numerics = TM_NUMERICS_DMMA;
    int schedule = TM_SCHEDULE_FUSED;
    int staging = TM_STAGING_AUTO;
};

/* Status code of a tm_* call -> the reference's exception for that failure. */
inline void throw_status(int rc) {
    if (rc == 0) return;
    const std::string msg = tm_last_error();
    if (rc == 1) {
        std::vector<Violation> vs;
        std::istringstream in(tm_last_rules());
        for (std::string ln; std::getline(in, ln);) {
            if (ln.empty()) continue;
            const auto a = ln.find(':'), b = ln.find(':', a + 1), c = ln.find(':', b + 1);
            if (a == std::string::npos || b == std::string::npos || c == std::string::npos) continue;
            Violation v;
            v.rule = ln.substr(0, a);
            v.level = std::stoi(ln.substr(a + 1, b - a - 1));
            v.lhs = std::stoll(ln.substr(b + 1, c - b - 1));
            v.rhs = std::stoll(ln.substr(c + 1));
            vs.push_back(std::move(v));
        }
        if (msg.rfind("validation failed", 0) == 0) throw ValidationFailure(std::move(vs));
        if (!vs.empty() && vs[0].rule == "infeasible") throw InfeasibleError(msg);
        const std::string rule = vs.empty() ? std::string() : vs[0].rule;
        const std::string prefix = rule + ": ";
        throw ParseError(rule, msg.rfind(prefix, 0) == 0 ? msg.substr(prefix.size()) : msg);
    }
    if (rc == 2) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

/* A B200 plan for a reference LoopNest. Owns the native plan: its lowered
 * task list and device buffers are reused across calls.
 *   Plan(nest)        -- from the nest's loops, m_r, n_r and shape, exactly
 *                        what execute() walks (plan.hpp:25-84); no model.
 *   Plan(nest, hier)  -- re-validated against the hierarchy with the
 *                        reference's rules (ValidationFailure on a misfit,
 *                        plan.hpp:90-108); carries the I/O model. */
class Plan {
  public:
    explicit Plan(const LoopNest& nest) : nest_(nest) {
        std::vector<tm_loop> lp;
        for (const auto& L : nest.loops) lp.push_back({L.level, to_char(L.dim), L.blocksize, L.cap ? 1 : 0});
        const std::string name = nest.descriptor.plans.empty() ? std::string() : format_name(nest.descriptor);
        throw_status(tm_plan_create_loops(name.empty() ? nullptr : name.c_str(), lp.data(),
                                          static_cast<int>(lp.size()), nest.m_r, nest.n_r, nest.shape.m,
                                          nest.shape.n, nest.shape.k, &plan_));
    }
    Plan(const LoopNest& nest, const CacheHierarchy& hier) : nest_(nest) {
        std::vector<tm_level> lv;
        for (const auto& l : hier.levels())
            lv.push_back({l.capacity_elements, l.granularity, l.inclusive ? 1 : 0, l.write_allocate ? 1 : 0,
                          l.write_back ? 1 : 0});
        std::vector<tm_blocksize> bs;
        for (const auto& [key, value] : nest.blocksizes.entries()) bs.push_back({key.level, to_char(key.dim), value});
        throw_status(tm_plan_create(format_name(nest.descriptor).c_str(), lv.data(), static_cast<int>(lv.size()),
                                    nest.shape.m, nest.shape.n, nest.shape.k, bs.data(),
                                    static_cast<int>(bs.size()), &plan_));
        // the native nest must walk the caller's cells: same loop order and register tile
        if (!loops_match(nest, plan_)) {
            tm_plan_destroy(plan_);
            throw std::invalid_argument("the nest's loops differ from build_plan(descriptor, blocksizes) on this "
                                        "hierarchy");
        }
    }
    ~Plan() { tm_plan_destroy(plan_); }
    Plan(const Plan&) = delete;
    Plan& operator=(const Plan&) = delete;

    tm_plan* get() const { return plan_; }
    const Shape& shape() const { return nest_.shape; }
    /* Whether this plan executes `nest`: same shape, loops and register tile. */
    bool matches(const LoopNest& nest) const { return same_nest(nest_, nest); }

    static bool same_nest(const LoopNest& a, const LoopNest& b) {
        if (a.shape.m != b.shape.m || a.shape.n != b.shape.n || a.shape.k != b.shape.k) return false;
        if (a.m_r != b.m_r || a.n_r != b.n_r || a.loops.size() != b.loops.size()) return false;
        for (std::size_t i = 0; i < a.loops.size(); ++i)
            if (a.loops[i].level != b.loops[i].level || a.loops[i].dim != b.loops[i].dim ||
                a.loops[i].blocksize != b.loops[i].blocksize || a.loops[i].cap != b.loops[i].cap)
                return false;
        return true;
    }

  private:
    static bool loops_match(const LoopNest& nest, tm_plan* p) {
        std::vector<tm_loop> got(64);
        int n = 0;
        if (tm_plan_loops(p, got.data(), static_cast<int>(got.size()), &n) != 0 ||
            n != static_cast<int>(nest.loops.size()))
            return false;
        for (int i = 0; i < n; ++i) {
            const auto& L = nest.loops[static_cast<std::size_t>(i)];
            if (got[i].level != L.level || got[i].dim != to_char(L.dim) || got[i].blocksize != L.blocksize ||
                (got[i].cap != 0) != L.cap)
                return false;
        }
        return true;
    }

    tm_plan* plan_ = nullptr;
    LoopNest nest_;
};

/* Same contract as tilemul::execute (exec.hpp:94-138): C += A·B in place,
 * every C entry accumulated in ascending k from its incoming value. The
 * reference's ExecOptions (workers, parallel_loop) are accepted and checked
 * the same way; the GPU grid replaces the host threads. */
inline void execute(Plan& plan, const LoopNest& nest, const MatrixBuffer& A, const MatrixBuffer& B, MatrixBuffer& C,
                    const ExecOptions& ropts = {}, const Options& o = {}) {
    if (!plan.matches(nest))
        throw std::invalid_argument("plan was built for another nest (shape, loops or register tile differ)");
    detail::check_buffer(A, Operand::A, nest);
    detail::check_buffer(B, Operand::B, nest);
    detail::check_buffer(C, Operand::C, nest);
    if (ropts.workers < 1) throw std::invalid_argument("worker count must be >= 1");
    if (ropts.workers > 1) {
        int par = ropts.parallel_loop;
        if (par < 0) par = static_cast<int>(nest.loops.size()) - 2;
        if (par < 0 || par >= static_cast<int>(nest.loops.size()))
            throw std::invalid_argument("parallel loop index out of range");
        if (nest.loops[static_cast<std::size_t>(par)].dim == Dim::k)
            throw std::invalid_argument(
                "cannot parallelize a k-dimension loop: workers would accumulate into shared C");
    }
    tm_exec_opts eo{};
    eo.numerics = o.numerics;
    eo.schedule = o.schedule;
    eo.split_k = o.numerics == TM_NUMERICS_DMMA ? 0 : 1;
    eo.staging = o.staging;
    // prepacked operands go through their column-major form (the device path
    // for packed data is tm_execute_packed on device buffers)
    const bool packed = A.layout.blocked() || B.layout.blocked() || C.layout.blocked();
    if (!packed) {
        throw_status(tm_execute_host(plan.get(), A.data.data(), B.data.data(), C.data.data(), &eo));
        return;
    }
    const MatrixBuffer a = A.layout.blocked() ? unpack(A) : A;
    const MatrixBuffer b = B.layout.blocked() ? unpack(B) : B;
    MatrixBuffer c = C.layout.blocked() ? unpack(C) : C;
    throw_status(tm_execute_host(plan.get(), a.data.data(), b.data.data(), c.data.data(), &eo));
    C = C.layout.blocked() ? tilemul::pack(c, C.layout) : std::move(c);
}

namespace detail_cache {
/* Plans of recently executed nests (most recent first), so the
 * signature-identical execute() below reuses a nest's lowering and device
 * buffers across calls instead of rebuilding them per call. */
struct Cache {
    std::mutex mu;
    std::list<std::shared_ptr<Plan>> plans;
    static constexpr std::size_t kMax = 4;
};
inline Cache& cache() {
    static Cache c;
    return c;
}
}  // namespace detail_cache

/* Frees the plans (and their device buffers) the cached execute() holds. */
inline void release_cached_plans() {
    auto& c = detail_cache::cache();
    std::lock_guard<std::mutex> lk(c.mu);
    c.plans.clear();
}

/* The reference's signature (exec.hpp:94-95): a drop-in for
 * tilemul::execute(nest, A, B, C, opts). */
inline void execute(const LoopNest& nest, const MatrixBuffer& A, const MatrixBuffer& B, MatrixBuffer& C,
                    const ExecOptions& ropts = {}, const Options& o = {}) {
    std::shared_ptr<Plan> plan;
    {
        auto& c = detail_cache::cache();
        std::lock_guard<std::mutex> lk(c.mu);
        for (auto it = c.plans.begin(); it != c.plans.end(); ++it)
            if ((*it)->matches(nest)) {
                plan = *it;
                c.plans.splice(c.plans.begin(), c.plans, it);
                break;
            }
        if (!plan) {
            plan = std::make_shared<Plan>(nest);
            c.plans.push_front(plan);
            if (c.plans.size() > detail_cache::Cache::kMax) c.plans.pop_back();
        }
    }
    execute(*plan, nest, A, B, C, ropts, o);
}

/* One-shot form against a hierarchy: re-validates, runs, frees the plan. */
inline void execute(const LoopNest& nest, const MatrixBuffer& A, const MatrixBuffer& B, MatrixBuffer& C,
                    const CacheHierarchy& hier, const ExecOptions& ropts = {}, const Options& o = {}) {
    Plan plan(nest, hier);
    execute(plan, nest, A, B, C, ropts, o);
}

}  // namespace tilemul::b200
