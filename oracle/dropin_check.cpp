// TEST INFRASTRUCTURE (oracle/): the drop-in check. Compiled by oracle/Makefile
// against the reference's own headers (/root/reference/proj/include, unmodified)
// and include/tilemul_b200.hpp, linked to the product library; run on a GPU box
// by tests/test_gpu_dropin.py. It calls the reference's API exactly as its
// callers do (parse_name -> derive_blocksizes -> build_plan -> execute,
// exec.hpp:94-138; pack, plan.hpp:113-124) and swaps only the execute call for
// tilemul::b200::execute, then checks:
//   - numerics EXACT: C bit-identical to the reference's execute(), column-major
//     and prepacked operands, for each expressible family member;
//   - numerics DMMA: within 4(k+1)u(|C0| + |A||B|) of it;
//   - errors: the same exception types (and for ValidationFailure the same
//     rule ids, in order) as the reference for the same bad inputs.
// Prints one JSON line per check and exits 0 only if all pass.
#include <cmath>
#include <cstdio>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "tilemul/blocksizes.hpp"
#include "tilemul/descriptor.hpp"
#include "tilemul/exec.hpp"
#include "tilemul/plan.hpp"
#include "tilemul_b200.hpp"

using namespace tilemul;

namespace {

int g_fail = 0;

void report(const std::string& name, bool ok, const std::string& detail = "") {
    std::printf("{\"check\": \"%s\", \"ok\": %s%s%s}\n", name.c_str(), ok ? "true" : "false",
                detail.empty() ? "" : ", \"detail\": ", detail.empty() ? "" : ("\"" + detail + "\"").c_str());
    std::fflush(stdout);
    if (!ok) ++g_fail;
}

MatrixBuffer filled(Operand role, i64 rows, i64 cols, std::mt19937_64& rng) {
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    MatrixBuffer b = MatrixBuffer::column_major(role, rows, cols);
    for (auto& x : b.data) x = u(rng);
    return b;
}

CacheHierarchy gpu_like() {
    // {CTA C tile 128x128, SMEM per block, a quarter of L2} in FP64 elements (tm_gpu_hierarchy's shape)
    return CacheHierarchy({CacheLevel{0, 16384}, CacheLevel{1, 29056}, CacheLevel{2, 4145152}});
}

LoopNest plan_for(const std::string& name, const Shape& s, const CacheHierarchy& h) {
    const AlgorithmDescriptor d = parse_name(name);
    DeriveOptions o;
    o.micro = MicroTile{128, 128};
    // the CTA-row pin the repo's planner uses (level 1's m, else its n); unpinned last
    for (Dim pin : {Dim::m, Dim::n, Dim::k}) {
        BlocksizeSet pinned;
        if (pin != Dim::k) pinned.set(1, pin, 128);
        try {
            return build_plan(d, derive_blocksizes(d, h, s, {}, o, pinned), h, s);
        } catch (const std::exception&) {
            if (pin == Dim::k) throw;
        }
    }
    throw std::logic_error("unreachable");
}

template <typename E>
std::string thrown(const std::function<void()>& f) {
    try {
        f();
    } catch (const E& e) {
        return e.what();
    } catch (const std::exception& e) {
        return std::string("WRONG TYPE: ") + e.what();
    }
    return "NO THROW";
}

}  // namespace

int main() {
    const CacheHierarchy hier = gpu_like();
    const b200::Options exact{TM_NUMERICS_EXACT};
    // the 3-level members; the level-skipping A2C0 / B2C0 have no feasible derivation with
    // a 128x128 register tile on this hierarchy (blocksizes.hpp:243-425) and are not run
    const std::vector<std::string> members = {"C2A1C0", "B2A1C0", "A2B1C0", "C2B1C0"};
    const std::vector<Shape> shapes = {Shape(300, 200, 517), Shape(256, 384, 520), Shape(1000, 700, 300)};
    std::mt19937_64 rng(12345);
    int cases = 0, packed_cases = 0;
    for (const auto& name : members)
        for (const auto& s : shapes) {
            LoopNest nest;
            try {
                nest = plan_for(name, s, hier);
            } catch (const std::exception& e) {
                continue;  // not expressible at this shape on this hierarchy
            }
            ++cases;
            const std::string tag = name + " " + std::to_string(s.m) + "x" + std::to_string(s.n) + "x" +
                                    std::to_string(s.k);
            const MatrixBuffer A = filled(Operand::A, s.m, s.k, rng), B = filled(Operand::B, s.k, s.n, rng);
            const MatrixBuffer C0 = filled(Operand::C, s.m, s.n, rng);
            MatrixBuffer want = C0;
            execute(nest, A, B, want);  // the reference, on the host

            b200::Plan plan(nest, hier);
            MatrixBuffer got = C0;
            b200::execute(plan, nest, A, B, got, ExecOptions{}, exact);
            report("exact bitwise " + tag, got.data == want.data);

            // prepacked operands in the nest's own layout (plan.hpp:113-124), where the
            // reference can build it (same-axis blocksizes must divide, layout.hpp:31-39)
            bool packable = true;
            try {
                for (Operand op : {Operand::A, Operand::B, Operand::C}) (void)layout_for(nest, op);
            } catch (const std::invalid_argument&) {
                packable = false;
            }
            if (packable) {
                ++packed_cases;
                const MatrixBuffer Ap = pack(A, nest), Bp = pack(B, nest);
                MatrixBuffer wantp = pack(C0, nest), gotp = pack(C0, nest);
                execute(nest, Ap, Bp, wantp);
                b200::execute(plan, nest, Ap, Bp, gotp, ExecOptions{}, exact);
                report("exact bitwise prepacked " + tag, gotp.data == wantp.data && gotp.layout.blocked());
            }

            // the reference's own call, unchanged: tilemul::execute(nest, A, B, C, opts) (exec.hpp:94-95)
            // with only the namespace swapped (plan built from the nest's loops, cached per nest)
            MatrixBuffer same = C0;
            b200::execute(nest, A, B, same, ExecOptions{}, exact);
            report("signature-identical exact bitwise " + tag, same.data == want.data);

            MatrixBuffer dm = C0;
            b200::execute(nest, A, B, dm);  // default numerics: the DMMA fast path
            double worst = 0;
            const double u = std::ldexp(1.0, -53);
            for (i64 j = 0; j < s.n; ++j)
                for (i64 i = 0; i < s.m; ++i) {
                    double ab = 0;
                    for (i64 p = 0; p < s.k; ++p) ab += std::fabs(A.data[i + p * s.m]) * std::fabs(B.data[p + j * s.k]);
                    const std::size_t q = static_cast<std::size_t>(i + j * s.m);
                    const double bound = 4.0 * static_cast<double>(s.k + 1) * u * (std::fabs(C0.data[q]) + ab);
                    worst = std::max(worst, std::fabs(dm.data[q] - want.data[q]) / bound);
                }
            report("dmma within bound " + tag, worst <= 1.0, "worst/bound " + std::to_string(worst));
        }
    report("cases run", cases >= 12, std::to_string(cases) + " member x shape cases");
    {  // a shape whose blocksizes divide it: prepacked operands are exercised for certain
        const Shape s(512, 512, 512);
        BlocksizeSet bs;  // every same-axis blocksize divides the one above it (layout.hpp:31-39)
        bs.set(2, Dim::m, 256);
        bs.set(2, Dim::n, 256);
        bs.set(1, Dim::k, 64);
        bs.set(1, Dim::m, 128);
        bs.set(0, Dim::m, 128);
        bs.set(0, Dim::n, 128);
        const LoopNest nest = build_plan(parse_name("C2A1C0"), bs, hier, s);
        const MatrixBuffer A = filled(Operand::A, s.m, s.k, rng), B = filled(Operand::B, s.k, s.n, rng);
        const MatrixBuffer C0 = filled(Operand::C, s.m, s.n, rng);
        try {
            const MatrixBuffer Ap = pack(A, nest), Bp = pack(B, nest);
            MatrixBuffer wantp = pack(C0, nest), gotp = pack(C0, nest);
            execute(nest, Ap, Bp, wantp);
            b200::execute(nest, Ap, Bp, gotp, hier, ExecOptions{}, exact);
            ++packed_cases;
            report("exact bitwise prepacked C2A1C0 512x512x512", gotp.data == wantp.data && gotp.layout.blocked());
        } catch (const std::invalid_argument& e) {
            report("exact bitwise prepacked C2A1C0 512x512x512", false, e.what());
        }
    }
    report("prepacked cases run", packed_cases >= 1, std::to_string(packed_cases) + " cases");

    // ---- errors: same types as the reference for the same inputs
    const Shape s(300, 200, 517);
    const LoopNest nest = plan_for("C2A1C0", s, hier);
    const MatrixBuffer A = filled(Operand::A, s.m, s.k, rng), B = filled(Operand::B, s.k, s.n, rng);
    MatrixBuffer C = filled(Operand::C, s.m, s.n, rng);
    {  // role mismatch (exec.hpp:67)
        const std::string r = thrown<std::invalid_argument>([&] { execute(nest, B, B, C); });
        const std::string g = thrown<std::invalid_argument>([&] { b200::execute(nest, B, B, C); });
        report("role mismatch -> invalid_argument", r == g && r.rfind("WRONG", 0) != 0 && r != "NO THROW", g);
    }
    {  // parallel loop along k (exec.hpp:127-131)
        int kl = -1;
        for (std::size_t i = 0; i < nest.loops.size(); ++i)
            if (nest.loops[i].dim == Dim::k) kl = static_cast<int>(i);
        ExecOptions eo;
        eo.workers = 2;
        eo.parallel_loop = kl;
        const std::string r = thrown<std::invalid_argument>([&] { execute(nest, A, B, C, eo); });
        const std::string g = thrown<std::invalid_argument>([&] { b200::execute(nest, A, B, C, eo); });
        report("k-parallel -> invalid_argument", r == g && r.rfind("WRONG", 0) != 0 && r != "NO THROW", g);
    }
    {  // blocksizes that break the fit rules: ValidationFailure, same rule ids in order (blocksizes.hpp:125-235)
        LoopNest bad = nest;
        bad.blocksizes.set(1, Dim::k, 4000);
        const auto want = validate_blocksizes(bad.descriptor, bad.blocksizes, hier, bad.shape);
        std::vector<std::string> got;
        std::string what = "NO THROW";
        try {
            b200::Plan p(bad, hier);
        } catch (const ValidationFailure& e) {
            what = "ValidationFailure";
            for (const auto& v : e.violations) got.push_back(v.rule + "@" + std::to_string(v.level));
        } catch (const std::exception& e) {
            what = std::string("WRONG TYPE: ") + e.what();
        }
        std::vector<std::string> ref;
        for (const auto& v : want) ref.push_back(v.rule + "@" + std::to_string(v.level));
        std::string ids;
        for (const auto& x : got) ids += x + " ";
        report("bad blocksizes -> ValidationFailure with the reference's rules",
               what == "ValidationFailure" && !ref.empty() && got == ref, ids);
    }
    {  // a plan used with another nest (advisor r01): invalid_argument, never a silent out-of-bounds run
        const LoopNest other = plan_for("C2A1C0", Shape(256, 384, 520), hier);
        b200::Plan p(nest);
        MatrixBuffer Co = filled(Operand::C, 256, 384, rng);
        const MatrixBuffer Ao = filled(Operand::A, 256, 520, rng), Bo = filled(Operand::B, 520, 384, rng);
        const std::string g = thrown<std::invalid_argument>([&] { b200::execute(p, other, Ao, Bo, Co); });
        report("plan/nest mismatch -> invalid_argument", g.rfind("WRONG", 0) != 0 && g != "NO THROW", g);
    }
    {  // a nest assembled by hand (no build_plan, no descriptor): executed from its loops alone
        LoopNest hand;
        hand.shape = Shape(130, 70, 90);
        hand.loops = {NestStep{1, Dim::k, 32, false}, NestStep{1, Dim::n, 40, false}, NestStep{0, Dim::n, 20, false},
                      NestStep{0, Dim::m, 64, false}};
        hand.m_r = 64;
        hand.n_r = 20;
        const MatrixBuffer Ah = filled(Operand::A, 130, 90, rng), Bh = filled(Operand::B, 90, 70, rng);
        const MatrixBuffer Ch = filled(Operand::C, 130, 70, rng);
        MatrixBuffer want = Ch, got = Ch;
        execute(hand, Ah, Bh, want);
        b200::execute(hand, Ah, Bh, got, ExecOptions{}, exact);
        report("hand-built nest exact bitwise", got.data == want.data);
        LoopNest wide = hand;
        wide.m_r = 32;  // cells of 64 rows exceed the register tile the reference's scratch holds (exec.hpp:107)
        const std::string g = thrown<std::invalid_argument>([&] { b200::execute(wide, Ah, Bh, got); });
        report("cells larger than m_r x n_r -> invalid_argument", g.rfind("WRONG", 0) != 0 && g != "NO THROW", g);
    }
    std::printf("{\"summary\": true, \"failures\": %d}\n", g_fail);
    return g_fail == 0 ? 0 : 1;
}
