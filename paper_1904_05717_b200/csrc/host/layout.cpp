// Hierarchical ("prepacked") operand layouts: layout.hpp:17-98 (BlockLayout,
// element_address) and plan.hpp:113-119 (layout_for).
#include <algorithm>

#include "mmm.hpp"

namespace mmm {

Blocked make_blocked(i64 rows, i64 cols, std::vector<Cut> cuts) {
    if (rows < 1 || cols < 1) fail_usage("layout extents must be >= 1");
    i64 last_row = 0, last_col = 0;  // 0: no enclosing cut on that axis yet
    for (const auto& c : cuts) {
        if (c.size < 1) fail_usage("partition blocksize must be >= 1");
        i64& last = c.rows ? last_row : last_col;
        if (last != 0 && last % c.size != 0)
            fail_usage("partition blocksize must divide the enclosing partition of the same dimension");
        last = c.size;
    }
    return Blocked{rows, cols, std::move(cuts)};
}

// Walk the cuts outermost-first: each cut selects the block containing
// (i, j) and adds the elements of all blocks before it.
i64 Blocked::address(i64 i, i64 j) const { return locate(i, j).first; }

std::pair<i64, i64> Blocked::locate(i64 i, i64 j) const {
    if (i < 0 || i >= rows || j < 0 || j >= cols) fail_usage("element index outside matrix");
    i64 base = 0, r0 = 0, r1 = rows, c0 = 0, c1 = cols;
    for (const auto& c : cuts) {
        if (c.rows) {
            const i64 q = (i - r0) / c.size;
            base += q * c.size * (c1 - c0);
            r0 += q * c.size;
            r1 = std::min(r0 + c.size, r1);
        } else {
            const i64 q = (j - c0) / c.size;
            base += q * c.size * (r1 - r0);
            c0 += q * c.size;
            c1 = std::min(c0 + c.size, c1);
        }
    }
    return {base + (i - r0) + (j - c0) * (r1 - r0), r1 - r0};
}

Blocked layout_of(const Nest& nest, Opnd op) {
    std::vector<Cut> cuts;
    const Dim row_dim = spans(op)[0];
    for (const auto& L : nest.loops)
        if (touches(op, L.dim)) cuts.push_back(Cut{L.dim == row_dim, L.size});
    return make_blocked(nest.ext.rows(op), nest.ext.cols(op), std::move(cuts));
}

}  // namespace mmm
