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
 *   execute(nest, A, B, C, opts)               tilemul::b200::execute(nest, A, B, C, hier, opts)
 *     exec.hpp:94-138                            (hier: the hierarchy the nest's blocksizes were
 *                                                 validated against, as in build_plan, plan.hpp:90-108)
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

/* A B200 plan for a reference LoopNest (same name, blocksizes, hierarchy,
 * shape). Owns the native plan: its lowered task list and device buffers
 * are reused across calls. */
class Plan {
  public:
    Plan(const LoopNest& nest, const CacheHierarchy& hier) : shape_(nest.shape) {
        std::vector<tm_level> lv;
        for (const auto& l : hier.levels())
            lv.push_back({l.capacity_elements, l.granularity, l.inclusive ? 1 : 0, l.write_allocate ? 1 : 0,
                          l.write_back ? 1 : 0});
        std::vector<tm_blocksize> bs;
        for (const auto& [key, value] : nest.blocksizes.entries()) bs.push_back({key.level, to_char(key.dim), value});
        throw_status(tm_plan_create(format_name(nest.descriptor).c_str(), lv.data(), static_cast<int>(lv.size()),
                                    nest.shape.m, nest.shape.n, nest.shape.k, bs.data(),
                                    static_cast<int>(bs.size()), &plan_));
    }
    ~Plan() { tm_plan_destroy(plan_); }
    Plan(const Plan&) = delete;
    Plan& operator=(const Plan&) = delete;

    tm_plan* get() const { return plan_; }
    const Shape& shape() const { return shape_; }

  private:
    tm_plan* plan_ = nullptr;
    Shape shape_;
};

/* Same contract as tilemul::execute (exec.hpp:94-138): C += A·B in place,
 * every C entry accumulated in ascending k from its incoming value. The
 * reference's ExecOptions (workers, parallel_loop) are accepted and checked
 * the same way; the GPU grid replaces the host threads. */
inline void execute(Plan& plan, const LoopNest& nest, const MatrixBuffer& A, const MatrixBuffer& B, MatrixBuffer& C,
                    const ExecOptions& ropts = {}, const Options& o = {}) {
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

/* One-shot form: builds the plan, runs, frees it. */
inline void execute(const LoopNest& nest, const MatrixBuffer& A, const MatrixBuffer& B, MatrixBuffer& C,
                    const CacheHierarchy& hier, const ExecOptions& ropts = {}, const Options& o = {}) {
    Plan plan(nest, hier);
    execute(plan, nest, A, B, C, ropts, o);
}

}  // namespace tilemul::b200
