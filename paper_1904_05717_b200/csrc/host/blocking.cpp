// Blocksizes: the (level, dim) table, the capacity-fit rules, the
// innermost-out derivation under those rules, and the loop order a family +
// blocksizes produce. Follows /root/reference/proj/include/tilemul/
// blocksizes.hpp (validate_blocksizes :125-235, derive_blocksizes :243-425,
// nest_steps :438-453); the floating-point expressions of the derivation are
// kept in the reference's evaluation order so derived sizes agree exactly.
#include <algorithm>
#include <cmath>
#include <tuple>

#include "mmm.hpp"

namespace mmm {

i64 Blocks::get(int h, Dim d) const {
    if (!has(h, d))
        fail_usage(std::string("no blocksize for level ") + std::to_string(h) + " dim " + dim_char(d));
    return v[h][d];
}

void Blocks::put(int h, Dim d, i64 value) {
    if (value < 1) fail_usage("blocksize must be >= 1");
    if (h < 0 || h >= kMaxLevels) fail_usage("blocksize level out of range");
    v[h][d] = value;
}

int Blocks::count() const {
    int c = 0;
    for (const auto& row : v)
        for (i64 x : row) c += x > 0;
    return c;
}

std::vector<std::tuple<int, Dim, i64>> Blocks::entries() const {
    std::vector<std::tuple<int, Dim, i64>> out;
    for (int h = 0; h < kMaxLevels; ++h)
        for (int d = 0; d < 3; ++d)
            if (v[h][d] > 0) out.emplace_back(h, static_cast<Dim>(d), v[h][d]);
    return out;
}

namespace {

i64 block_area(const Tier& t, const Blocks& bs) { return bs.get(t.level, t.outer) * bs.get(t.level, t.inner); }

// Guest panel held beside `up`'s resident: (below's outer block) x (up's block
// along the dimension the guest shares with up's resident).
i64 guest_area(const Tier& up, const Tier& below, const Blocks& bs) {
    return bs.get(below.level, below.outer) * bs.get(up.level, common(guest_of(below), up.resident));
}

// Largest (outer, inner) with outer = ratio*inner and
// outer*inner + lo*outer + li*inner <= budget (blocksizes.hpp:106-112).
std::pair<double, double> quad_fit(double budget, double ratio, double lo, double li) {
    if (budget <= 0 || ratio <= 0) return {0.0, 0.0};
    const double p = lo * ratio + li;
    const double t = (-p + std::sqrt(p * p + 4.0 * ratio * budget)) / (2.0 * ratio);
    return {ratio * t, t};
}

}  // namespace

std::vector<Issue> fit_issues(const Family& f, const Blocks& bs, const Hierarchy& h) {
    std::vector<Issue> out = structure_issues(f);
    if (!out.empty()) return out;

    // Entries must sit on a planned loop, or be the single cap entry on a
    // skipped level above the top plan along its resident's long dimension.
    const Dim cap_dim = untouched(f.tiers.front().resident);
    int caps = 0;
    for (const auto& [level, dim, value] : bs.entries()) {
        if (const Tier* t = f.at(level)) {
            if (dim != t->outer && dim != t->inner)
                out.push_back({"unexpected_blocksize_entry", level, value, 0,
                               std::string("dimension '") + dim_char(dim) + "' is not looped at this level"});
        } else if (level <= f.top() || dim != cap_dim) {
            out.push_back({"unexpected_blocksize_entry", level, value, 0,
                           "only a skipped level above the outermost plan may carry a cap entry, "
                           "along the top resident's long dimension"});
        } else if (++caps > 1) {
            out.push_back({"multiple_cap_blocksizes", level, value, 0, "at most one cap entry is supported"});
        }
    }

    for (std::size_t i = 0; i < f.tiers.size(); ++i) {
        const Tier& up = f.tiers[i];
        if (!h.has(up.level)) {
            out.push_back({"level_not_in_hierarchy", up.level, 0, h.size() - 1, "no such cache level"});
            continue;
        }
        bool missing = false;
        for (Dim d : {up.outer, up.inner})
            if (!bs.has(up.level, d)) {
                out.push_back({"blocksize_missing", up.level, 0, 0,
                               std::string("no blocksize for dimension '") + dim_char(d) + "'"});
                missing = true;
            }
        if (missing) continue;
        const i64 cap = h.cap(up.level);
        const i64 resident = block_area(up, bs);
        const bool incl = h.lv[static_cast<std::size_t>(up.level)].inclusive;

        if (i + 1 == f.tiers.size()) {  // register tier: the tile itself must fit
            if (resident > cap)
                out.push_back({"resident_guest_exceed_capacity", up.level, resident, cap,
                               "register tile exceeds the register capacity"});
            continue;
        }
        const Tier& dn = f.tiers[i + 1];
        if (!bs.has(dn.level, dn.outer) || !bs.has(dn.level, dn.inner)) continue;
        const i64 guest = guest_area(up, dn, bs);
        const i64 lower = block_area(dn, bs);
        if (resident + guest > cap)  // rule (a)
            out.push_back({"resident_guest_exceed_capacity", up.level, resident + guest, cap,
                           "resident block plus guest panel exceed the level's capacity"});
        if (incl && resident + guest + lower > cap)  // rule (b)
            out.push_back({"inclusive_lower_resident_exceed", up.level, resident + guest + lower, cap,
                           "inclusive level must also hold the next plan's resident block"});
        if (incl) {  // rule (c)
            const i64 exposed = resident + bs.get(dn.level, dn.outer) *
                                               (bs.get(up.level, up.outer) + bs.get(up.level, up.inner));
            if (exposed > cap)
                out.push_back({"inclusive_lru_working_set_exceed", up.level, exposed, cap,
                               "partitions exposed by the next plan's outer loop exceed capacity"});
        }
        for (int s = dn.level + 1; s < up.level; ++s) {  // skipped levels in between
            if (!h.has(s)) continue;
            const i64 cap_s = h.cap(s);
            if (guest > cap_s)
                out.push_back({"skip_guest_exceed", s, guest, cap_s,
                               "guest panel of the enclosing level does not fit the skipped level"});
            const i64 panel = bs.get(dn.level, dn.inner) * bs.get(up.level, partner(up.resident, dn.inner));
            if (guest + panel > cap_s)
                out.push_back({"skip_lru_panel_exceed", s, guest + panel, cap_s,
                               "guest panel plus a panel of the enclosing resident exceed the skipped LRU level"});
            if (h.lv[static_cast<std::size_t>(s)].inclusive && guest + panel + lower > cap_s)
                out.push_back({"skip_inclusive_resident_exceed", s, guest + panel + lower, cap_s,
                               "inclusive skipped level must also hold the inner resident block"});
        }
    }

    // A capped skipped level above the top plan must hold the capped panel.
    const Tier& top = f.tiers.front();
    for (int s = top.level + 1; s < h.size(); ++s) {
        if (!bs.has(s, cap_dim) || !bs.has(top.level, top.outer)) continue;
        const i64 panel = bs.get(top.level, top.outer) * bs.get(s, cap_dim);
        if (panel > h.cap(s))
            out.push_back({"skip_guest_exceed", s, panel, h.cap(s), "capped panel does not fit the skipped level"});
    }
    return out;
}

Blocks derive(const Family& f, const Hierarchy& h, const Extents& e, const Weights& w, const DeriveOpts& o,
              const Blocks& pinned) {
    if (!(w.a > 0 && w.b > 0 && w.c > 0)) fail_usage("access cost weights must be strictly positive");
    if (o.slack < 0 || o.slack >= 1) fail_usage("slack must lie in [0, 1)");
    auto structural = structure_issues(f);
    if (!structural.empty()) fail_rules(std::move(structural));
    for (const auto& t : f.tiers)
        if (!h.has(t.level)) fail_rules({{"level_not_in_hierarchy", t.level, 0, h.size() - 1, ""}});

    Blocks bs = pinned;
    const double keep = 1.0 - o.slack;
    const std::size_t ntiers = f.tiers.size();

    // Rounding granule: the nearest lower tier that loops the same dim.
    auto granule = [&](std::size_t i, Dim d) -> i64 {
        for (std::size_t j = i + 1; j < ntiers; ++j)
            if (f.tiers[j].outer == d || f.tiers[j].inner == d) return bs.get(f.tiers[j].level, d);
        return 0;
    };
    auto no_fit = [&](int level, Dim d) {
        fail_infeasible("no feasible blocksize at level " + std::to_string(level) + " in dimension '" + dim_char(d) +
                        "'; consider skipping this level");
    };
    auto settle = [&](std::size_t i, Dim d, double value) -> i64 {
        i64 v = static_cast<i64>(std::floor(value));
        if (v >= e.of(d)) return e.of(d);  // one partition covers the extent
        const i64 q = granule(i, d);
        if (q > 0) {
            v = (v / q) * q;
            if (v < q) no_fit(f.tiers[i].level, d);
        }
        if (v < 1) no_fit(f.tiers[i].level, d);
        return v;
    };

    // Register tile: pins or the micro-tile default (C only).
    const Tier& reg = f.tiers.back();
    for (Dim d : {reg.outer, reg.inner}) {
        if (bs.has(reg.level, d)) continue;
        if (reg.resident != kC) fail_infeasible("register tile for a non-C resident must be pinned explicitly");
        bs.put(reg.level, d, d == kM ? o.m_r : o.n_r);
    }
    if (block_area(reg, bs) > h.cap(reg.level))
        fail_infeasible("register tile of " + std::to_string(block_area(reg, bs)) +
                        " elements exceeds the register capacity M_0 = " + std::to_string(h.cap(reg.level)));

    for (std::size_t ii = ntiers - 1; ii-- > 0;) {
        const Tier& up = f.tiers[ii];
        const Tier& dn = f.tiers[ii + 1];
        const bool pin_o = bs.has(up.level, up.outer), pin_i = bs.has(up.level, up.inner);
        if (pin_o && pin_i) continue;

        const double ratio = w.of(lacking(up.outer)) / w.of(lacking(up.inner));
        const i64 c = bs.get(dn.level, dn.outer);
        const i64 lower = block_area(dn, bs);
        const Dim gdim = common(guest_of(dn), up.resident);
        const bool incl = h.lv[static_cast<std::size_t>(up.level)].inclusive;

        const double budget =
            keep * static_cast<double>(h.cap(up.level)) - (incl ? static_cast<double>(lower) : 0.0);
        if (budget <= 0)
            fail_infeasible("level " + std::to_string(up.level) +
                            " cannot hold the inner resident block; consider skipping a level");

        // Rule (c) when inclusive (implies (a)); else rule (a) with the guest
        // panel's linear term along the shared dimension.
        double lo = 0, li = 0;
        if (incl) {
            lo = li = static_cast<double>(c);
        } else if (gdim == up.outer) {
            lo = static_cast<double>(c);
        } else {
            li = static_cast<double>(c);
        }

        double bo, bi;
        if (pin_o || pin_i) {
            const double fixed = static_cast<double>(bs.get(up.level, pin_o ? up.outer : up.inner));
            const double lin_fixed = pin_o ? lo : li;
            const double lin_free = pin_o ? li : lo;
            const double free_val = (budget - lin_fixed * fixed) / (fixed + lin_free);
            bo = pin_o ? fixed : free_val;
            bi = pin_o ? free_val : fixed;
        } else {
            std::tie(bo, bi) = quad_fit(budget, ratio, lo, li);
        }

        // Shrink to co*bo + ci*bi + quad*bo*bi <= limit, keeping the aspect
        // ratio unless one side is pinned.
        auto shrink = [&](double co, double ci, double quad, double limit) {
            const double lhs = co * bo + ci * bi + quad * bo * bi;
            if (lhs <= limit) return;
            auto pinned_violation = [&] {
                fail_infeasible("pinned blocksize at level " + std::to_string(up.level) +
                                " violates a fit constraint");
            };
            if (pin_o) {
                const double den = ci + quad * bo;
                if (den <= 0) pinned_violation();
                bi = (limit - co * bo) / den;
            } else if (pin_i) {
                const double den = co + quad * bi;
                if (den <= 0) pinned_violation();
                bo = (limit - ci * bi) / den;
            } else {
                const double r = bo / bi;
                double o2, i2;
                if (quad > 0) {
                    std::tie(o2, i2) = quad_fit(limit / quad, r, co / quad, ci / quad);
                } else {
                    const double t = limit / (co * r + ci);
                    o2 = r * t;
                    i2 = t;
                }
                if (i2 < bi) {
                    bo = o2;
                    bi = i2;
                }
            }
        };

        for (int s = dn.level + 1; s < up.level; ++s) {  // skipped levels bound the guest (+ LRU panel)
            if (!h.has(s)) continue;
            const double budget_s = keep * static_cast<double>(h.cap(s)) -
                                    (h.lv[static_cast<std::size_t>(s)].inclusive ? static_cast<double>(lower) : 0.0);
            if (budget_s <= 0)
                fail_infeasible("skipped level " + std::to_string(s) + " cannot hold the inner resident block");
            const double p_in = static_cast<double>(bs.get(dn.level, dn.inner));
            const Dim pdim = partner(up.resident, dn.inner);
            const double co = (gdim == up.outer ? c : 0.0) + (pdim == up.outer ? p_in : 0.0);
            const double ci = (gdim == up.inner ? c : 0.0) + (pdim == up.inner ? p_in : 0.0);
            shrink(co, ci, 0.0, budget_s);
        }
        if (ii == 0) {  // a capped skipped level above the top holds the guest-of-memory panel
            for (int s = up.level + 1; s < h.size(); ++s) {
                if (!bs.has(s, untouched(up.resident))) continue;
                shrink(static_cast<double>(bs.get(s, untouched(up.resident))), 0.0, 0.0,
                       keep * static_cast<double>(h.cap(s)));
            }
        }
        if (!pin_o) bs.put(up.level, up.outer, settle(ii, up.outer, bo));
        if (!pin_i) bs.put(up.level, up.inner, settle(ii, up.inner, bi));
    }

    auto issues = fit_issues(f, bs, h);
    if (!issues.empty()) fail_rules(std::move(issues));
    return bs;
}

std::vector<Loop> loop_order(const Family& f, const Blocks& bs) {
    std::vector<Loop> loops;
    if (f.tiers.empty()) return loops;
    const Dim cap_dim = untouched(f.tiers.front().resident);
    for (const auto& [level, dim, value] : bs.entries())
        if (level > f.top() && dim == cap_dim && f.at(level) == nullptr) loops.push_back({level, cap_dim, value, true});
    std::stable_sort(loops.begin(), loops.end(), [](const Loop& a, const Loop& b) { return a.level > b.level; });
    for (const auto& t : f.tiers) {
        loops.push_back({t.level, t.outer, bs.get(t.level, t.outer), false});
        loops.push_back({t.level, t.inner, bs.get(t.level, t.inner), false});
    }
    return loops;
}

}  // namespace mmm
