// Algebra, errors, memory hierarchy and the algorithm family (descriptor
// grammar, composition rules, validation, level skipping, outer-resident
// choice). Behaviour follows /root/reference/proj/include/tilemul/types.hpp,
// cache.hpp and descriptor.hpp (cited per function).
#include <cctype>
#include <cmath>

#include "mmm.hpp"

namespace mmm {

char dim_char(Dim d) { return "mnk"[d]; }
char opnd_char(Opnd o) { return "ABC"[o]; }

Dim dim_of_char(char c) {  // types.hpp:40-47
    if (c == 'm') return kM;
    if (c == 'n') return kN;
    if (c == 'k') return kK;
    fail_usage(std::string("unknown dimension '") + c + "'");
}

Opnd opnd_of_char(char c) {  // types.hpp:49-56
    if (c == 'A') return kA;
    if (c == 'B') return kB;
    if (c == 'C') return kC;
    fail_usage(std::string("unknown operand '") + c + "'");
}

Extents make_extents(i64 m, i64 n, i64 k) {  // types.hpp:107-111
    if (m < 1 || n < 1 || k < 1) fail_usage("shape extents must be >= 1");
    return Extents{m, n, k};
}

std::string describe(const Issue& v) {  // types.hpp:140-145
    std::string s = v.rule;
    if (v.level >= 0) s += " (level " + std::to_string(v.level) + ")";
    if (!v.detail.empty()) s += ": " + v.detail;
    return s;
}

void fail_parse(const std::string& rule, const std::string& msg) {
    throw Failure(kRuleBroken, rule, rule + ": " + msg);
}

void fail_rules(std::vector<Issue> issues) {
    std::string s = "validation failed:";
    for (const auto& v : issues) s += "\n  - " + describe(v);
    throw Failure(kRuleBroken, "", s, std::move(issues));
}

void fail_infeasible(const std::string& msg) { throw Failure(kRuleBroken, "infeasible", msg); }
void fail_usage(const std::string& msg) { throw Failure(kUsage, "", msg); }

// ---------------------------------------------------------------- hierarchy

Hierarchy make_hierarchy(std::vector<MemLevel> levels) {  // cache.hpp:27-38
    if (levels.empty()) fail_usage("hierarchy needs at least one level");
    for (std::size_t i = 0; i < levels.size(); ++i) {
        if (levels[i].capacity < 1) fail_usage("cache capacity must be >= 1");
        if (levels[i].line < 1) fail_usage("cache granularity must be >= 1");
        if (i > 0 && levels[i].capacity <= levels[i - 1].capacity)
            fail_usage("cache capacities must strictly increase with level");
    }
    if (levels.size() > static_cast<std::size_t>(Blocks::kMaxLevels)) fail_usage("too many hierarchy levels");
    return Hierarchy{std::move(levels)};
}

// ------------------------------------------------------------------ family

const Tier* Family::at(int level) const {
    for (const auto& t : tiers)
        if (t.level == level) return &t;
    return nullptr;
}

// The loop pair a lone plan runs when no lower resident forces it
// (descriptor.hpp:54-60).
static void lone_tier_loops(Tier& t) {
    if (t.resident == kC) {
        t.outer = kN;
        t.inner = kM;
    } else if (t.resident == kA) {
        t.outer = kK;
        t.inner = kM;
    } else {
        t.outer = kN;
        t.inner = kK;
    }
}

// make_descriptor (descriptor.hpp:68-107): the outermost tier's inner loop
// runs the dimension it shares with the next resident; every lower tier's
// outer loop runs the enclosing resident's untouched dimension.
Family compose(const std::vector<std::pair<int, Opnd>>& residents, bool free_registers) {
    if (residents.empty()) fail_parse("empty_descriptor", "descriptor needs at least one level");
    Family f;
    f.free_registers = free_registers;
    for (std::size_t i = 0; i < residents.size(); ++i) {
        const int level = residents[i].first;
        const Opnd res = residents[i].second;
        if (i > 0 && level >= residents[i - 1].first)
            fail_parse("levels_not_strictly_decreasing", "cache levels must strictly decrease outermost to innermost");
        if (i > 0 && res == residents[i - 1].second)
            fail_parse("consecutive_resident_equal",
                       std::string("operand ") + opnd_char(res) + " resident at two consecutive levels");
        Tier t;
        t.level = level;
        t.resident = res;
        if (i == 0 && residents.size() == 1) {
            lone_tier_loops(t);
        } else if (i == 0) {
            t.inner = common(res, residents[1].second);
            t.outer = partner(res, t.inner);
        } else {
            t.outer = untouched(residents[i - 1].second);
            t.inner = partner(res, t.outer);
        }
        f.tiers.push_back(t);
    }
    if (f.tiers.back().level != 0) fail_parse("missing_register_level", "descriptor must end at the register level (0)");
    if (f.tiers.back().resident != kC && !free_registers)
        fail_parse("registers_not_resident_c", "register level must hold C (set allow_non_c_registers to override)");
    return f;
}

// parse_name (descriptor.hpp:111-125): <letter><digit> tokens.
Family family_from_name(const std::string& text, bool free_registers) {
    if (text.empty() || text.size() % 2 != 0)
        fail_parse("name_grammar", "expected one or more <operand letter><level digit> tokens");
    std::vector<std::pair<int, Opnd>> residents;
    for (std::size_t i = 0; i < text.size(); i += 2) {
        const char letter = text[i], digit = text[i + 1];
        if (letter != 'A' && letter != 'B' && letter != 'C')
            fail_parse("name_grammar", std::string("operand letter expected, got '") + letter + "'");
        if (!std::isdigit(static_cast<unsigned char>(digit)))
            fail_parse("name_grammar", std::string("level digit expected, got '") + digit + "'");
        residents.emplace_back(digit - '0', opnd_of_char(letter));
    }
    return compose(residents, free_registers);
}

std::string family_name(const Family& f) {  // format_name, descriptor.hpp:128-136
    std::string s;
    for (const auto& t : f.tiers) {
        if (t.level > 9) fail_usage("names only cover cache levels 0..9");
        s += opnd_char(t.resident);
        s += static_cast<char>('0' + t.level);
    }
    return s;
}

// validate_structure (descriptor.hpp:140-173): every violated rule, in order.
std::vector<Issue> structure_issues(const Family& f) {
    std::vector<Issue> out;
    if (f.tiers.empty()) {
        out.push_back({"empty_descriptor", -1, 0, 0, "no level plans"});
        return out;
    }
    for (std::size_t i = 0; i < f.tiers.size(); ++i) {
        const Tier& t = f.tiers[i];
        if (t.outer == t.inner)
            out.push_back({"loop_dims_equal", t.level, 0, 0, "outer and inner loop share a dimension"});
        else if (!touches(t.resident, t.outer) || !touches(t.resident, t.inner))
            out.push_back({"loops_not_resident_dims", t.level, 0, 0,
                           "loop dimensions must be exactly the resident's dimensions"});
        if (i == 0) continue;
        const Tier& up = f.tiers[i - 1];
        if (t.level >= up.level) out.push_back({"levels_not_strictly_decreasing", t.level, t.level, up.level, ""});
        if (t.resident == up.resident)
            out.push_back({"consecutive_resident_equal", t.level, 0, 0,
                           std::string("operand ") + opnd_char(t.resident) + " repeats"});
        else if (t.outer != untouched(up.resident))
            out.push_back({"outer_not_long_dim", t.level, 0, 0,
                           std::string("outer loop must run along '") + dim_char(untouched(up.resident)) +
                               "', the enclosing resident's long dimension"});
    }
    const Tier& last = f.tiers.back();
    if (last.level != 0)
        out.push_back({"missing_register_level", last.level, 0, 0, "innermost plan must sit at the register level (0)"});
    if (last.resident != kC && !f.free_registers)
        out.push_back({"registers_not_resident_c", last.level, 0, 0,
                       "register level must hold C unless explicitly overridden"});
    return out;
}

// skip_level (descriptor.hpp:177-195).
Family without_level(const Family& f, int h) {
    if (h == 0) fail_usage("cannot skip the register level");
    std::vector<std::pair<int, Opnd>> residents;
    bool found = false;
    for (const auto& t : f.tiers) {
        if (t.level == h) {
            found = true;
        } else {
            residents.emplace_back(t.level, t.resident);
        }
    }
    if (found) return compose(residents, f.free_registers);
    if (f.tiers.empty() || h > f.tiers.front().level || h < 0)
        fail_usage("level " + std::to_string(h) + " is not inside the descriptor's level range");
    return f;
}

// select_algorithm (descriptor.hpp:206-218).
Opnd outer_resident_for(const Extents& e, i64 outer_capacity, double near, double large) {
    if (outer_capacity < 1) fail_usage("cache capacity must be >= 1");
    const double root = std::sqrt(static_cast<double>(outer_capacity));
    auto is_near = [&](i64 x) {
        const double v = static_cast<double>(x);
        return v >= root / near && v <= root * near;
    };
    auto is_large = [&](i64 x) { return static_cast<double>(x) >= root * large; };
    if (is_near(e.m) && is_near(e.k) && is_large(e.n)) return kA;
    if (is_near(e.n) && is_near(e.k) && is_large(e.m)) return kB;
    return kC;
}

}  // namespace mmm
