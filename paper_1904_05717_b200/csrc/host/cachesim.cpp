// Multilevel LRU replay of a nest's element accesses; see cachesim.hpp.
// Semantics follow the reference simulator (cachesim.hpp:61-354):
//   * lookups go inward-out; every level that misses counts the miss, the
//     first level holding the line counts a hit and refreshes its recency;
//   * the missed levels allocate (reads always, writes per write_allocate;
//     an inclusive level allocates whenever a faster level does), outermost
//     first, each allocation counting one fetched line;
//   * a write marks the innermost write-back level holding the line dirty;
//     every level it passes on the way there forwards it (passthrough);
//   * an evicted inclusive line removes its footprint from faster levels,
//     merging their dirt; a dirty line leaving a write-back level crosses
//     each boundary outward until a write-back level holding it absorbs it.
#include "cachesim.hpp"

#include <algorithm>
#include <numeric>

namespace mmm {

TraceAddressing TraceAddressing::column_major(const Extents& e) {
    return {make_blocked(e.m, e.k, {}), make_blocked(e.k, e.n, {}), make_blocked(e.m, e.n, {})};
}

TraceAddressing TraceAddressing::packed(const Nest& nest) {
    return {layout_of(nest, kA), layout_of(nest, kB), layout_of(nest, kC)};
}

i64 access_count(const Nest& nest) {
    i64 total = 0;
    nest.walk([&](const Cell& c) { total += 2 * c.m * c.n + c.k * (c.m + c.n); });
    return total;
}

// ------------------------------------------------------------ one store

void CacheSim::Store::detach(std::int32_t s) {
    const Slot& x = slot[static_cast<std::size_t>(s)];
    if (x.newer >= 0) slot[static_cast<std::size_t>(x.newer)].older = x.older; else mru = x.older;
    if (x.older >= 0) slot[static_cast<std::size_t>(x.older)].newer = x.newer; else lru = x.newer;
}

void CacheSim::Store::attach_front(std::int32_t s) {
    Slot& x = slot[static_cast<std::size_t>(s)];
    x.newer = -1;
    x.older = mru;
    if (mru >= 0) slot[static_cast<std::size_t>(mru)].newer = s;
    mru = s;
    if (lru < 0) lru = s;
}

std::int32_t CacheSim::Store::grab() {
    if (!spare.empty()) {
        const std::int32_t s = spare.back();
        spare.pop_back();
        return s;
    }
    return used++;
}

void CacheSim::Store::drop(std::int32_t s) {
    slot_of[static_cast<std::size_t>(slot[static_cast<std::size_t>(s)].line)] = -1;
    detach(s);
    slot[static_cast<std::size_t>(s)].line = -1;
    spare.push_back(s);
}

// ------------------------------------------------------------- simulator

CacheSim::CacheSim(const Hierarchy& h, const Extents& e, SimConfig cfg) : cfg_(cfg) {
    i64 align = 1;
    for (const auto& l : h.lv) align = std::lcm(align, l.line);
    const auto up = [&](i64 v) { return cdiv(v, align) * align; };
    base_[kA] = 0;
    base_[kB] = up(e.size(kA));
    base_[kC] = base_[kB] + up(e.size(kB));
    const i64 space = base_[kC] + up(e.size(kC));
    // the line table is dense over the address space (4 bytes per line)
    if (space > (i64{1} << 31)) fail_usage("trace address space too large to simulate");
    for (int idx = 0; idx < h.size(); ++idx) {
        if (idx == 0 && !cfg.include_registers) continue;
        Store s;
        s.cfg = h.lv[static_cast<std::size_t>(idx)];
        s.lines = std::max<i64>(1, s.cfg.capacity / s.cfg.line);
        s.st.level = idx;
        s.st.capacity_lines = s.lines;
        s.st.granularity = s.cfg.line;
        s.slot_of.assign(static_cast<std::size_t>(cdiv(space, s.cfg.line)), -1);
        s.slot.assign(static_cast<std::size_t>(s.lines), Slot{});
        lv_.push_back(std::move(s));
    }
    if (lv_.empty()) fail_usage("nothing to simulate");
    if (lv_.size() > 16) fail_usage("too many cache levels to simulate");
}

void CacheSim::access(const Access& a) {
    ++events_;
    const i64 addr = base_[a.op] + a.index;
    const int L = levels();
    int hit_at = L;  // L: served by memory
    for (int li = 0; li < L; ++li) {
        Store& s = lv_[static_cast<std::size_t>(li)];
        const std::int32_t slot = s.find(addr);
        if (slot >= 0) {
            if (s.mru != slot) {
                s.detach(slot);
                s.attach_front(slot);
            }
            ++s.st.hits;
            hit_at = li;
            break;
        }
        ++(a.write ? s.st.write_misses : s.st.read_misses);
        ++s.st.op_misses[a.op];
    }
    // which missed levels allocate
    std::array<bool, 16> take{};
    bool inner_takes = false;
    for (int li = 0; li < hit_at; ++li) {
        const MemLevel& c = lv_[static_cast<std::size_t>(li)].cfg;
        bool t = !a.write || c.write_allocate;
        if (!t && inner_takes && c.inclusive) t = true;
        inner_takes = inner_takes || t;
        take[static_cast<std::size_t>(li)] = t;
    }
    for (int li = hit_at - 1; li >= 0; --li) {
        if (!take[static_cast<std::size_t>(li)]) continue;
        ++lv_[static_cast<std::size_t>(li)].st.fetched_lines;
        install(li, addr, a.op);
    }
    if (!a.write) return;
    for (int li = 0; li < L; ++li) {
        Store& s = lv_[static_cast<std::size_t>(li)];
        const std::int32_t slot = s.find(addr);
        if (slot >= 0 && s.cfg.write_back) {
            s.slot[static_cast<std::size_t>(slot)].dirty = 1;
            return;
        }
        ++s.st.passthrough_writes;
    }
}

void CacheSim::install(int li, i64 addr, Opnd op) {
    Store& s = lv_[static_cast<std::size_t>(li)];
    if (s.full()) evict(li, s.lru);
    const std::int32_t slot = s.grab();
    Slot& x = s.slot[static_cast<std::size_t>(slot)];
    const i64 ln = addr / s.cfg.line;
    x.line = ln;
    x.dirty = 0;
    x.owner = static_cast<std::uint8_t>(op);
    s.slot_of[static_cast<std::size_t>(ln)] = slot;
    s.attach_front(slot);
}

void CacheSim::evict(int li, std::int32_t slot) {
    Store& s = lv_[static_cast<std::size_t>(li)];
    const Slot x = s.slot[static_cast<std::size_t>(slot)];
    const i64 ln = x.line;
    bool dirty = x.dirty != 0;
    const Opnd op = static_cast<Opnd>(x.owner);
    s.drop(slot);
    if (s.cfg.inclusive && purge_inner(li, ln)) dirty = true;
    if (dirty && s.cfg.write_back) write_out(li, ln * s.cfg.line, op);
}

bool CacheSim::purge_inner(int li, i64 ln) {
    const i64 g = lv_[static_cast<std::size_t>(li)].cfg.line;
    const i64 lo = ln * g, hi = lo + g;
    bool merged = false;
    for (int f = 0; f < li; ++f) {
        Store& in = lv_[static_cast<std::size_t>(f)];
        for (i64 a = lo; a < hi; a += in.cfg.line) {
            const std::int32_t slot = in.find(a);
            if (slot < 0) continue;
            if (in.slot[static_cast<std::size_t>(slot)].dirty) {
                merged = true;
                const Opnd op = static_cast<Opnd>(in.slot[static_cast<std::size_t>(slot)].owner);
                // the inner copy's data crosses every boundary up to the evicting level
                for (int j = f; j < li; ++j) {
                    ++lv_[static_cast<std::size_t>(j)].st.writebacks;
                    ++lv_[static_cast<std::size_t>(j)].st.op_writebacks[op];
                }
            }
            in.drop(slot);
        }
    }
    return merged;
}

void CacheSim::write_out(int li, i64 addr, Opnd op) {
    const int L = levels();
    for (int o = li; o < L; ++o) {
        Store& s = lv_[static_cast<std::size_t>(o)];
        ++s.st.writebacks;
        ++s.st.op_writebacks[op];
        if (o + 1 == L) return;
        Store& next = lv_[static_cast<std::size_t>(o + 1)];
        const std::int32_t slot = next.find(addr);
        if (slot >= 0 && next.cfg.write_back) {
            next.slot[static_cast<std::size_t>(slot)].dirty = 1;
            return;
        }
    }
}

std::vector<SimStats> CacheSim::finish() {
    if (cfg_.flush_at_end && !flushed_) {
        flushed_ = true;
        for (int li = 0; li < levels(); ++li) {
            Store& s = lv_[static_cast<std::size_t>(li)];
            for (std::int32_t slot = 0; slot < s.used; ++slot) {
                Slot& x = s.slot[static_cast<std::size_t>(slot)];
                if (x.line < 0 || !x.dirty) continue;
                x.dirty = 0;
                write_out(li, x.line * s.cfg.line, static_cast<Opnd>(x.owner));
            }
        }
    }
    std::vector<SimStats> out;
    for (const auto& s : lv_) out.push_back(s.st);
    return out;
}

std::vector<i64> CacheSim::resident(int position) const {
    if (position < 0 || position >= levels()) fail_usage("no such simulated level");
    const Store& s = lv_[static_cast<std::size_t>(position)];
    std::vector<i64> out;
    for (std::int32_t slot = 0; slot < s.used; ++slot)
        if (s.slot[static_cast<std::size_t>(slot)].line >= 0) out.push_back(s.slot[static_cast<std::size_t>(slot)].line);
    return out;
}

}  // namespace mmm
