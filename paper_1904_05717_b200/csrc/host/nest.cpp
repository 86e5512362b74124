// The executable loop nest (plan.hpp:25-108) and the closed-form per-level
// I/O model (costmodel.hpp:67-284).
#include <algorithm>
#include <cmath>
#include <limits>

#include "mmm.hpp"

namespace mmm {

// ------------------------------------------------------------------- nest

namespace {

// Recursive blocked walk with margins: the trailing partition of each loop
// shrinks to what is left of the enclosing extent (plan.hpp:61-84).
void walk_rec(const Nest& nest, std::size_t depth, std::array<i64, 3> org, std::array<i64, 3> ext,
              const std::function<void(const Cell&)>& f) {
    if (depth == nest.loops.size()) {
        f(Cell{org[0], ext[0], org[1], ext[1], org[2], ext[2]});
        return;
    }
    const Loop& L = nest.loops[depth];
    const int d = L.dim;
    const i64 lo = org[d], hi = org[d] + ext[d];
    for (i64 s = lo; s < hi; s += L.size) {
        org[d] = s;
        ext[d] = std::min(L.size, hi - s);
        walk_rec(nest, depth + 1, org, ext, f);
    }
}

}  // namespace

void Nest::walk(const std::function<void(const Cell&)>& f) const {
    walk_rec(*this, 0, {0, 0, 0}, {ext.m, ext.n, ext.k}, f);
}

i64 Nest::cells() const {
    // Product over loops of partition counts is wrong with margins nested in
    // margins, so count the same way the walk enumerates, per dimension:
    // every dimension's partition tree is independent of the others.
    i64 total = 1;
    for (int d = 0; d < 3; ++d) {
        std::vector<std::pair<i64, i64>> sizes{{ext.of(static_cast<Dim>(d)), 1}};
        for (const auto& L : loops) {
            if (L.dim != d) continue;
            std::vector<std::pair<i64, i64>> next;
            for (auto [sz, cnt] : sizes) {
                if (sz / L.size > 0) next.emplace_back(L.size, cnt * (sz / L.size));
                if (sz % L.size > 0) next.emplace_back(sz % L.size, cnt);
            }
            sizes = std::move(next);
        }
        i64 parts = 0;
        for (auto [sz, cnt] : sizes) parts += cnt;
        total *= parts;
    }
    return total;
}

Nest build_nest(const Family& f, const Blocks& bs, const Hierarchy& h, const Extents& e, i64 min_c_tile) {
    auto issues = fit_issues(f, bs, h);
    if (!issues.empty()) fail_rules(std::move(issues));
    if (f.tiers.back().resident != kC) fail_usage("only C-resident register plans are executable");
    Nest nest;
    nest.ext = e;
    nest.family = f;
    nest.blocks = bs;
    nest.loops = loop_order(f, bs);
    nest.m_r = bs.get(0, kM);
    nest.n_r = bs.get(0, kN);
    if (min_c_tile > 0 && nest.m_r * nest.n_r < min_c_tile)
        fail_usage("register tile smaller than the configured latency floor of " + std::to_string(min_c_tile) +
                   " elements");
    return nest;
}

// --------------------------------------------------------------- I/O model

double IoModel::bytes(int h, const std::array<double, 3>& elem_bytes) const {
    for (const auto& lf : levels)
        if (lf.level == h) {
            double b = 0;
            for (int o = 0; o < 3; ++o)
                b += elem_bytes[static_cast<std::size_t>(o)] *
                     static_cast<double>(lf.op[static_cast<std::size_t>(o)].reads +
                                         lf.op[static_cast<std::size_t>(o)].writes);
            return b;
        }
    fail_usage("no traffic entry for level " + std::to_string(h));
}

Flow lower_bound_io(const Extents& e, i64 M) {  // costmodel.hpp:67-76
    if (M < 1) fail_usage("fast memory capacity must be >= 1");
    const long double raw = 2.0L * static_cast<long double>(e.m) * static_cast<long double>(e.n) *
                            static_cast<long double>(e.k) / std::sqrt(static_cast<long double>(M));
    Flow t;
    t.reads = std::max<i64>(0, static_cast<i64>(std::ceil(raw)) - 2 * M);
    t.writes = std::max<i64>(0, e.m * e.n - M);
    return t;
}

// The fundamental two-level algorithm with `variant` resident in blocks of
// (b1, b2) along spans(variant): the resident moves once (C also back once);
// each other operand is re-streamed once per partition of the resident along
// the dimension that operand lacks (costmodel.hpp:85-100).
LevelFlow resident_io(Opnd variant, const Extents& e, i64 b1, i64 b2) {
    if (b1 < 1 || b2 < 1) fail_usage("blocksizes must be >= 1");
    const auto sp = spans(variant);
    LevelFlow t;
    auto& r = t.op[variant];
    r.reads = e.size(variant);
    if (variant == kC) r.writes = r.reads;
    for (int y = 0; y < 3; ++y) {
        if (y == variant) continue;
        const Dim miss = untouched(static_cast<Opnd>(y));
        const i64 passes = cdiv(e.of(miss), miss == sp[0] ? b1 : b2);
        auto& s = t.op[static_cast<std::size_t>(y)];
        s.reads = e.size(static_cast<Opnd>(y)) * passes;
        if (y == kC) s.writes = s.reads;
    }
    return t;
}

namespace {

// Distinct chunk extents along one dimension with multiplicities
// (costmodel.hpp:105-130).
struct Chunks {
    std::vector<std::pair<i64, i64>> v;
    void cut(i64 b) {
        std::vector<std::pair<i64, i64>> next;
        auto add = [&](i64 sz, i64 cnt) {
            for (auto& x : next)
                if (x.first == sz) {
                    x.second += cnt;
                    return;
                }
            next.emplace_back(sz, cnt);
        };
        for (auto [sz, cnt] : v) {
            if (sz / b > 0) add(b, cnt * (sz / b));
            if (sz % b > 0) add(sz % b, cnt);
        }
        v = std::move(next);
    }
};

struct Subproblems {
    std::array<Chunks, 3> d;
    void cut(Dim dim, i64 b) { d[dim].cut(b); }
    template <typename F>
    void each(F&& f) const {
        for (auto [ms, mc] : d[0].v)
            for (auto [ns, nc] : d[1].v)
                for (auto [ks, kc] : d[2].v) f(Extents{ms, ns, ks}, mc * nc * kc);
    }
};

void add_scaled(LevelFlow& into, const LevelFlow& t, i64 count) {
    for (int o = 0; o < 3; ++o) {
        into.op[static_cast<std::size_t>(o)].reads += count * t.op[static_cast<std::size_t>(o)].reads;
        into.op[static_cast<std::size_t>(o)].writes += count * t.op[static_cast<std::size_t>(o)].writes;
    }
}

}  // namespace

// multilevel_cost (costmodel.hpp:163-229): a planned level sums the
// two-level cost over its enclosing subproblems; a skipped level is charged
// as if the enclosing guest panel were its resident.
IoModel level_io(const Family& f, const Blocks& bs, const Hierarchy& h, const Extents& e, int boundary) {
    auto issues = fit_issues(f, bs, h);
    if (!issues.empty()) fail_rules(std::move(issues));
    IoModel rep;
    rep.ext = e;
    rep.flops = e.flops();
    rep.boundary = boundary < 0 ? h.top() : boundary;

    Subproblems sub;
    sub.d[0].v = {{e.m, 1}};
    sub.d[1].v = {{e.n, 1}};
    sub.d[2].v = {{e.k, 1}};
    for (const auto& L : loop_order(f, bs))
        if (L.cap) sub.cut(L.dim, L.size);
    const Subproblems cap_scope = sub;
    std::vector<Subproblems> before(f.tiers.size()), after(f.tiers.size());
    for (std::size_t i = 0; i < f.tiers.size(); ++i) {
        const Tier& t = f.tiers[i];
        before[i] = sub;
        sub.cut(t.outer, bs.get(t.level, t.outer));
        sub.cut(t.inner, bs.get(t.level, t.inner));
        after[i] = sub;
    }

    for (int lvl = 0; lvl < h.size(); ++lvl) {
        LevelFlow lf;
        lf.level = lvl;
        if (const Tier* t = f.at(lvl)) {
            std::size_t i = 0;
            while (f.tiers[i].level != lvl) ++i;
            const auto sp = spans(t->resident);
            const i64 b1 = bs.get(lvl, sp[0]), b2 = bs.get(lvl, sp[1]);
            before[i].each([&](const Extents& s, i64 cnt) { add_scaled(lf, resident_io(t->resident, s, b1, b2), cnt); });
        } else {
            // Skipped: above the top plan the guest of memory, else the guest
            // panel of the enclosing planned level.
            const bool above = lvl > f.top();
            std::size_t i = 0;
            if (!above)
                while (i + 1 < f.tiers.size() && f.tiers[i + 1].level > lvl) ++i;
            const Tier& q = above ? f.tiers.front() : f.tiers[i + 1];
            const Subproblems& scope = above ? cap_scope : after[i];
            const Opnd g = guest_of(q);
            const auto sp = spans(g);
            scope.each([&](const Extents& s, i64 cnt) {
                auto blk = [&](Dim d) { return d == q.outer ? bs.get(q.level, q.outer) : s.of(d); };
                add_scaled(lf, resident_io(g, s, blk(sp[0]), blk(sp[1])), cnt);
            });
        }
        rep.levels.push_back(lf);
    }
    return rep;
}

double flops_per_element(const IoModel& r, int level, double write_weight) {  // efficiency(), :238-247
    const int want = level < 0 ? r.boundary : level;
    for (const auto& lf : r.levels)
        if (lf.level == want) {
            const double el = static_cast<double>(lf.reads()) + write_weight * static_cast<double>(lf.writes());
            if (el <= 0) return std::numeric_limits<double>::infinity();
            return static_cast<double>(r.flops) / el;
        }
    fail_usage("no traffic entry for level " + std::to_string(want));
}

double streaming_flops_per_element(Opnd variant, i64 b1, i64 b2) {  // :252-263
    if (b1 < 1 || b2 < 1) fail_usage("blocksizes must be >= 1");
    const auto sp = spans(variant);
    double den = 0;
    for (int y = 0; y < 3; ++y) {
        if (y == variant) continue;
        const Dim miss = untouched(static_cast<Opnd>(y));
        den += (y == kC ? 2.0 : 1.0) / static_cast<double>(miss == sp[0] ? b1 : b2);
    }
    return 2.0 / den;
}

double goto_flops_per_element(i64 k_c, i64 n_c) {  // :267-270
    if (k_c < 1 || n_c < 1) fail_usage("blocksizes must be >= 1");
    return 1.0 / (1.0 / static_cast<double>(k_c) + 1.0 / (2.0 * static_cast<double>(n_c)));
}

double roofline(double intensity, double peak, double bandwidth) {  // :278-284
    if (!(peak > 0) || !(bandwidth > 0)) fail_usage("roofline parameters must be strictly positive");
    if (intensity < 0) fail_usage("intensity must be >= 0");
    return std::min(peak, intensity * bandwidth);
}

}  // namespace mmm
