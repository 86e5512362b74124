// Trace-driven check of the I/O model: the element
// access stream a loop nest implies, replayed through a multilevel, fully
// associative LRU hierarchy. Restates the reference's trace generator
// (trace.hpp:51-71) and simulator (cachesim.hpp:61-354): the per-level
// counts (hits, misses, fetched lines, forwarded writes, writebacks) are the
// reference's, so compare_model() reads the same against multilevel_cost.
#pragma once

#include <array>
#include <cstdint>
#include <vector>

#include "mmm.hpp"

namespace mmm {

// One element access in program order (trace.hpp:17-21).
struct Access {
    Opnd op;
    i64 index;  // flat element index under the operand's layout
    bool write;
};

// Addressing of the three operands: column-major or the nest's packed
// (hierarchical) layouts (trace.hpp:27-46).
struct TraceAddressing {
    Blocked a, b, c;
    static TraceAddressing column_major(const Extents& e);
    static TraceAddressing packed(const Nest& nest);
    const Blocked& of(Opnd o) const { return o == kA ? a : o == kB ? b : c; }
};

// Per cell in nest order: C tile read (column by column), then per k step the
// A column fragment and the B row fragment, then the C tile written back.
// A cell never straddles a leaf block of any operand's layout (the packed
// layouts cut along exactly the nest's loops), so each fragment is one
// address plus a fixed stride: +1 down a column, +leaf rows along a row.
template <typename Sink>
void for_each_access(const Nest& nest, const TraceAddressing& lay, Sink&& sink) {
    nest.walk([&](const Cell& c) {
        for (int pass = 0; pass < 2; ++pass) {
            if (pass == 1) {
                for (i64 p = 0; p < c.k; ++p) {
                    const i64 a0 = lay.a.locate(c.i0, c.p0 + p).first;
                    for (i64 i = 0; i < c.m; ++i) sink(Access{kA, a0 + i, false});
                    const auto [b0, bstride] = lay.b.locate(c.p0 + p, c.j0);
                    for (i64 j = 0; j < c.n; ++j) sink(Access{kB, b0 + j * bstride, false});
                }
            }
            const bool write = pass == 1;
            for (i64 j = 0; j < c.n; ++j) {
                const i64 c0 = lay.c.locate(c.i0, c.j0 + j).first;
                for (i64 i = 0; i < c.m; ++i) sink(Access{kC, c0 + i, write});
            }
        }
    });
}
i64 access_count(const Nest& nest);  // 2mn + k(m+n) per cell

struct SimStats {  // cachesim.hpp:18-38
    int level = 0;
    i64 capacity_lines = 0, granularity = 1;
    i64 hits = 0, read_misses = 0, write_misses = 0;
    i64 fetched_lines = 0;       // read misses + allocating write misses
    i64 passthrough_writes = 0;  // writes forwarded outward without allocation
    i64 writebacks = 0;          // dirty lines crossing the boundary above this level
    std::array<i64, 3> op_misses{}, op_writebacks{};
    i64 misses() const { return read_misses + write_misses; }
    i64 transferred() const { return granularity * (fetched_lines + writebacks) + passthrough_writes; }
};

struct SimConfig {  // SimOptions, cachesim.hpp:52-55
    bool include_registers = false;
    bool flush_at_end = true;
};

class CacheSim {
  public:
    CacheSim(const Hierarchy& h, const Extents& e, SimConfig cfg = {});
    void access(const Access& a);
    // Drains dirty lines (when configured) and returns the per-level counts,
    // innermost simulated level first.
    std::vector<SimStats> finish();
    i64 events() const { return events_; }
    int levels() const { return static_cast<int>(lv_.size()); }
    std::vector<i64> resident(int position) const;

  private:
    // One fully associative LRU array: line -> slot table plus an intrusive
    // recency list over slots (mru .. lru).
    struct Slot {  // one cache line's state: a recency update touches one host cache line
        i64 line = -1;  // -1: free
        std::int32_t newer = -1, older = -1;
        std::uint8_t dirty = 0, owner = 0;
    };
    struct Store {
        MemLevel cfg;
        i64 lines = 1;
        SimStats st;
        std::vector<std::int32_t> slot_of;  // line -> slot, -1 absent
        std::vector<Slot> slot;
        std::vector<std::int32_t> spare;
        std::int32_t mru = -1, lru = -1, used = 0;

        std::int32_t find(i64 addr) const { return slot_of[static_cast<std::size_t>(addr / cfg.line)]; }
        void detach(std::int32_t s);
        void attach_front(std::int32_t s);
        bool full() const { return spare.empty() && used == static_cast<std::int32_t>(lines); }
        std::int32_t grab();
        void drop(std::int32_t s);  // forget the slot's line (no accounting)
    };

    void install(int li, i64 addr, Opnd op);
    void evict(int li, std::int32_t s);
    bool purge_inner(int li, i64 line);
    void write_out(int li, i64 addr, Opnd op);

    SimConfig cfg_;
    std::vector<Store> lv_;
    std::array<i64, 3> base_{};
    i64 events_ = 0;
    bool flushed_ = false;
};

}  // namespace mmm
