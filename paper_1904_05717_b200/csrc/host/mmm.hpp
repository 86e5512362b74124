// Host-side vocabulary of the MOMMS family on B200: operand/dimension algebra,
// algorithm families (resident operand per memory level), blocksizes and their
// fit rules, the executable loop nest, and the per-level I/O model.
//
// This restates the semantics of the reference toolkit (tilemul,
// /root/reference/proj/include/tilemul/*.hpp) as a compiled library behind
// the C ABI in include/tilemul_b200.h. File:line citations point at the
// reference behaviour each piece follows; rule names (Violation.rule) are the
// reference's, so callers can match on them.
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace mmm {

using i64 = std::int64_t;

// ---------------------------------------------------------------- algebra
// types.hpp:14-100. Dims index the problem C(m x n) += A(m x k) B(k x n).
enum Dim : int { kM = 0, kN = 1, kK = 2 };
enum Opnd : int { kA = 0, kB = 1, kC = 2 };

char dim_char(Dim d);
char opnd_char(Opnd o);
Dim dim_of_char(char c);     // throws Usage on anything but m/n/k
Opnd opnd_of_char(char c);   // throws Usage on anything but A/B/C

// (row dim, column dim) of an operand's storage.
constexpr std::array<Dim, 2> spans(Opnd o) {
    return o == kA ? std::array<Dim, 2>{kM, kK} : o == kB ? std::array<Dim, 2>{kK, kN} : std::array<Dim, 2>{kM, kN};
}
constexpr bool touches(Opnd o, Dim d) { return spans(o)[0] == d || spans(o)[1] == d; }
// The dimension an operand does not touch ("long dim", types.hpp:70-77).
constexpr Dim untouched(Opnd o) { return o == kA ? kN : o == kB ? kM : kK; }
// The operand that does not touch d (types.hpp:80-86).
constexpr Opnd lacking(Dim d) { return d == kN ? kA : d == kM ? kB : kC; }
// The operand's other dimension (types.hpp:89-92).
constexpr Dim partner(Opnd o, Dim d) { return spans(o)[0] == d ? spans(o)[1] : spans(o)[0]; }
// Dimension shared by two distinct operands (types.hpp:95-98).
constexpr Dim common(Opnd x, Opnd y) { return touches(y, spans(x)[0]) ? spans(x)[0] : spans(x)[1]; }

struct Extents {
    i64 m = 1, n = 1, k = 1;
    i64 of(Dim d) const { return d == kM ? m : d == kN ? n : k; }
    i64& of(Dim d) { return d == kM ? m : d == kN ? n : k; }
    i64 flops() const { return 2 * m * n * k; }
    i64 rows(Opnd o) const { return of(spans(o)[0]); }
    i64 cols(Opnd o) const { return of(spans(o)[1]); }
    i64 size(Opnd o) const { return rows(o) * cols(o); }
};
Extents make_extents(i64 m, i64 n, i64 k);  // throws Usage unless all >= 1

inline i64 cdiv(i64 a, i64 b) { return (a + b - 1) / b; }

// ----------------------------------------------------------------- errors
// Status codes of the C ABI; the classes mirror the reference's exception
// taxonomy (types.hpp:148-174) and the CLI's exit codes
// (tools/tilemul_main.cpp:519-535).
enum Status : int { kOk = 0, kRuleBroken = 1, kUsage = 2, kDevice = 3 };

struct Issue {  // types.hpp:132-138 (Violation)
    std::string rule;
    int level = -1;
    i64 lhs = 0, rhs = 0;
    std::string detail;
};
std::string describe(const Issue& v);

struct Failure : std::runtime_error {
    Status status;
    std::string rule;             // ParseError rule, or "" (empty for infeasible/usage)
    std::vector<Issue> issues;    // ValidationFailure list
    Failure(Status s, std::string r, const std::string& msg, std::vector<Issue> is = {})
        : std::runtime_error(msg), status(s), rule(std::move(r)), issues(std::move(is)) {}
};
[[noreturn]] void fail_parse(const std::string& rule, const std::string& msg);
[[noreturn]] void fail_rules(std::vector<Issue> issues);
[[noreturn]] void fail_infeasible(const std::string& msg);
[[noreturn]] void fail_usage(const std::string& msg);

// -------------------------------------------------------------- hierarchy
// cache.hpp:12-49. Level 0 = registers; capacities in elements.
struct MemLevel {
    i64 capacity = 1;
    i64 line = 1;
    bool inclusive = false;
    bool write_allocate = true;
    bool write_back = true;
};
struct Hierarchy {
    std::vector<MemLevel> lv;
    int size() const { return static_cast<int>(lv.size()); }
    bool has(int h) const { return h >= 0 && h < size(); }
    i64 cap(int h) const { return lv.at(static_cast<std::size_t>(h)).capacity; }
    int top() const { return size() - 1; }
};
Hierarchy make_hierarchy(std::vector<MemLevel> levels);  // checks contiguity + strictly rising capacity

// ----------------------------------------------------------------- family
// descriptor.hpp:18-43. One tier per planned level, outermost first.
struct Tier {
    int level = 0;
    Opnd resident = kC;
    Dim outer = kN, inner = kM;
    bool operator==(const Tier& o) const {
        return level == o.level && resident == o.resident && outer == o.outer && inner == o.inner;
    }
};
struct Family {
    std::vector<Tier> tiers;
    bool free_registers = false;  // allow_non_c_registers
    const Tier* at(int level) const;
    int top() const { return tiers.empty() ? -1 : tiers.front().level; }
};
// Guest panel owner of the level enclosing `below` (descriptor.hpp:47).
inline Opnd guest_of(const Tier& below) { return lacking(below.inner); }

Family compose(const std::vector<std::pair<int, Opnd>>& residents, bool free_registers = false);
Family family_from_name(const std::string& text, bool free_registers = false);
std::string family_name(const Family& f);
std::vector<Issue> structure_issues(const Family& f);
Family without_level(const Family& f, int h);                  // skip_level
Opnd outer_resident_for(const Extents& e, i64 outer_capacity,  // select_algorithm
                        double near = 2.0, double large = 4.0);

// ------------------------------------------------------------- blocksizes
// blocksizes.hpp:22-56 as a dense (level x dim) table; 0 = unset.
struct Blocks {
    static constexpr int kMaxLevels = 16;
    std::array<std::array<i64, 3>, kMaxLevels> v{};
    bool has(int h, Dim d) const { return h >= 0 && h < kMaxLevels && v[h][d] > 0; }
    i64 get(int h, Dim d) const;  // throws Usage if unset
    void put(int h, Dim d, i64 value);
    int count() const;
    // Entries in (level, dim) ascending order, as std::map<Key,...> iterates.
    std::vector<std::tuple<int, Dim, i64>> entries() const;
};

struct Weights {  // AccessCosts, blocksizes.hpp:59-76
    double a = 1, b = 1, c = 1;
    double of(Opnd o) const { return o == kA ? a : o == kB ? b : c; }
};
struct DeriveOpts {  // DeriveOptions + MicroTile, blocksizes.hpp:79-87
    double slack = 1.0 / 16.0;
    i64 m_r = 4, n_r = 12;
};

std::vector<Issue> fit_issues(const Family& f, const Blocks& bs, const Hierarchy& h);  // validate_blocksizes
Blocks derive(const Family& f, const Hierarchy& h, const Extents& e, const Weights& w = {},
              const DeriveOpts& o = {}, const Blocks& pinned = {});

struct Loop {  // NestStep, blocksizes.hpp:428-434
    int level = 0;
    Dim dim = kM;
    i64 size = 1;
    bool cap = false;
};
std::vector<Loop> loop_order(const Family& f, const Blocks& bs);  // nest_steps

// ------------------------------------------------------------------- nest
// plan.hpp:25-108.
struct Cell {
    i64 i0, m, j0, n, p0, k;
};
struct Nest {
    Extents ext;
    Family family;
    Blocks blocks;
    std::vector<Loop> loops;
    i64 m_r = 1, n_r = 1;
    // Visits cells in nest order. Returning false from f stops the walk.
    void walk(const std::function<void(const Cell&)>& f) const;
    i64 cells() const;
};
Nest build_nest(const Family& f, const Blocks& bs, const Hierarchy& h, const Extents& e, i64 min_c_tile = 0);

// -------------------------------------------------------------- I/O model
// costmodel.hpp:15-229. Element transfers into each level, per operand.
struct Flow {
    i64 reads = 0, writes = 0;
};
struct LevelFlow {
    int level = 0;
    std::array<Flow, 3> op{};
    i64 reads() const { return op[0].reads + op[1].reads + op[2].reads; }
    i64 writes() const { return op[0].writes + op[1].writes + op[2].writes; }
};
struct IoModel {
    Extents ext;
    i64 flops = 0;
    std::vector<LevelFlow> levels;  // ascending level
    int boundary = 0;
    // Bytes into level h with per-operand element sizes (the reference fixes
    // 8 B per element, costmodel.hpp:41; BF16/TF32 inputs need 2/4).
    double bytes(int h, const std::array<double, 3>& elem_bytes = {8, 8, 8}) const;
};
Flow lower_bound_io(const Extents& e, i64 M);                          // io_lower_bound
LevelFlow resident_io(Opnd variant, const Extents& e, i64 b1, i64 b2);  // resident_cost
IoModel level_io(const Family& f, const Blocks& bs, const Hierarchy& h, const Extents& e, int boundary = -1);
double flops_per_element(const IoModel& r, int level = -1, double write_weight = 1.0);
double streaming_flops_per_element(Opnd variant, i64 b1, i64 b2);
double goto_flops_per_element(i64 k_c, i64 n_c);
double roofline(double intensity, double peak, double bandwidth);

// Seeded inputs of the reference's `run` command (host/seeded.cpp).
void fill_seeded(uint64_t seed, double* a, int64_t na, double* b, int64_t nb, double* c, int64_t nc);

}  // namespace mmm

// ----------------------------------------------------------------- layouts
// layout.hpp:17-98, plan.hpp:113-119: a hierarchical ("prepacked") storage
// layout as a chain of partition steps, outermost first; each step cuts the
// current block along rows or columns; blocks of a cut are stored
// contiguously in partition order; the innermost block is column-major.
namespace mmm {

struct Cut {
    bool rows = true;
    i64 size = 1;
};

struct Blocked {
    i64 rows = 1, cols = 1;
    std::vector<Cut> cuts;
    bool blocked() const { return !cuts.empty(); }
    i64 address(i64 i, i64 j) const;  // bijection onto [0, rows*cols)
    // address(i, j) plus the row extent of the column-major leaf block
    // holding (i, j): inside one leaf, (i+1, j) is +1 and (i, j+1) is +rows.
    std::pair<i64, i64> locate(i64 i, i64 j) const;
};
Blocked make_blocked(i64 rows, i64 cols, std::vector<Cut> cuts);  // same-axis cuts must divide
Blocked layout_of(const Nest& nest, Opnd op);                      // layout_for

}  // namespace mmm
