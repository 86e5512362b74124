// GPU-mode I/O model of a lowered schedule (SURVEY.md §7.1 "FIFO-SMEM mode",
// §8(a15)/(f2); the reference's model is costmodel.hpp:163-229).
//
// The reference charges each level with a resident block that stays put
// while the guest and the streamed panels pass through it, and charges a
// skipped level as if the enclosing guest panel were resident
// (costmodel.hpp:212-225). On the GPU neither holds as is:
//   * SMEM is a FIFO of k-slabs: a CTA task streams its A rows and B columns
//     through a 3-stage ring, and C lives in registers for the task's whole k
//     range. Into the SMEM level: A m_t k_t + B k_t n_t per task and the C
//     tile once in, once out (plus split-k partials) -- for the fused
//     schedule without splits exactly mk*ceil(n/n_r) + kn*ceil(m/m_r) + 2mn.
//     A block the reference keeps resident in SMEM across an inner spatial
//     loop is, on the GPU, re-staged by every CTA that runs an iteration of
//     that loop: its traffic is multiplied by that replication factor
//     (faithful schedule: the A k1-slab of C2A1C0 once per n0 iteration).
//   * The L2-level resident block of the fused schedule is the wave of
//     co-resident CTAs (their C tiles in the register files); L2 holds the
//     A/B slabs the wave streams. The model runs the schedule's own task
//     list in lockstep (one k-slab per CTA per step; strided rounds or
//     stream-K ranges exactly as the kernel takes them) through an LRU of
//     the L2's byte capacity at slab granularity, with C tiles and split-k
//     partials write-back.
// Both are computed from the host half of the lowering (plan_tasks), so the
// model describes exactly the schedule the kernel runs, and needs no GPU.
#include <algorithm>
#include <cstdlib>
#include <list>
#include <unordered_map>

#include "engine.hpp"

namespace mmm {
namespace engine {

namespace {

struct UnitKey {
    int64_t a, b;
    bool operator==(const UnitKey& o) const { return a == o.a && b == o.b; }
};
struct UnitHash {
    std::size_t operator()(const UnitKey& k) const {
        return std::hash<int64_t>()(k.a * 0x9E3779B97F4A7C15LL ^ (k.b + 0x632BE59BD9B4E019LL));
    }
};

// Write-back cache over variable-size units (bytes), counting the bytes it
// fetches from and writes back to memory per operand (0 A, 1 B, 2 C).
// policy 0: LRU; policy 1: random replacement (seeded, reproducible).
class UnitCache {
  public:
    UnitCache(int64_t capacity, int policy) : cap_(capacity), policy_(policy) {}
    void access(int op, UnitKey key, int64_t bytes, bool write) {
        auto it = map_.find(key);
        if (it != map_.end()) {
            Entry& e = ents_[it->second];
            if (policy_ == 0) touch(it->second);
            if (write) e.dirty = true;
            return;
        }
        if (!write) fetched[op] += bytes;  // a write allocates without reading (whole tiles are written)
        while (used_ + bytes > cap_ && !ents_.empty()) evict(victim());
        const int64_t slot = static_cast<int64_t>(ents_.size());
        ents_.push_back(Entry{key, bytes, write, op, -1, -1});
        map_[key] = slot;
        used_ += bytes;
        if (policy_ == 0) link_front(slot);
    }
    void flush() {
        while (!ents_.empty()) evict(static_cast<int64_t>(ents_.size()) - 1);
    }
    int64_t fetched[3] = {0, 0, 0}, written[3] = {0, 0, 0};

  private:
    struct Entry {
        UnitKey key;
        int64_t bytes;
        bool dirty;
        int op;
        int64_t prev, next;  // LRU list (policy 0), by slot
    };
    int64_t victim() {
        if (policy_ == 0) return tail_;
        rng_ = rng_ * 6364136223846793005ULL + 1442695040888963407ULL;
        return static_cast<int64_t>((rng_ >> 33) % ents_.size());
    }
    void unlink(int64_t s) {
        Entry& e = ents_[s];
        if (e.prev >= 0) ents_[e.prev].next = e.next; else head_ = e.next;
        if (e.next >= 0) ents_[e.next].prev = e.prev; else tail_ = e.prev;
        e.prev = e.next = -1;
    }
    void link_front(int64_t s) {
        Entry& e = ents_[s];
        e.prev = -1;
        e.next = head_;
        if (head_ >= 0) ents_[head_].prev = s;
        head_ = s;
        if (tail_ < 0) tail_ = s;
    }
    void touch(int64_t s) {
        if (head_ == s) return;
        unlink(s);
        link_front(s);
    }
    void evict(int64_t s) {
        Entry& e = ents_[s];
        if (e.dirty) written[e.op] += e.bytes;
        used_ -= e.bytes;
        map_.erase(e.key);
        if (policy_ == 0) unlink(s);
        const int64_t last = static_cast<int64_t>(ents_.size()) - 1;
        if (s != last) {  // move the last slot into the hole
            if (policy_ == 0) {
                const int64_t p = ents_[last].prev, n = ents_[last].next;
                ents_[s] = ents_[last];
                if (p >= 0) ents_[p].next = s; else head_ = s;
                if (n >= 0) ents_[n].prev = s; else tail_ = s;
            } else {
                ents_[s] = ents_[last];
            }
            map_[ents_[s].key] = s;
        }
        ents_.pop_back();
    }
    int64_t cap_, used_ = 0;
    int policy_;
    int64_t head_ = -1, tail_ = -1;
    uint64_t rng_ = 0x853c49e6748fea9bULL;
    std::vector<Entry> ents_;
    std::unordered_map<UnitKey, int64_t, UnitHash> map_;
};

}  // namespace

GpuIo gpu_io(const Nest& nest, const tm_exec_opts& o, int sms, int64_t l2_bytes, const double elem_bytes[3],
             int policy, int kernel_override) {
    const bool stagger = kernel_override == gpu::kTc2wBf16 || kernel_override == gpu::kTc2wTf32;
    if (sms < 1) fail_usage("SM count must be >= 1");
    if (l2_bytes < 1) fail_usage("L2 capacity must be >= 1 byte");
    const bool tma = o.staging != TM_STAGING_CPASYNC;
    const gpu::Kernel kernel = kernel_override >= 0 ? static_cast<gpu::Kernel>(kernel_override) : pick_kernel(nest, o, tma);
    const gpu::KernelInfo info = kernel_tiles(kernel, false);
    const bool pair = kernel == gpu::kTc2Bf16 || kernel == gpu::kTc2Tf32 || kernel == gpu::kTc2wBf16 ||
                      kernel == gpu::kTc2wTf32;
    // SM-pair kernels: a task is one cluster's tile, sms / 2 clusters in flight
    const int slots = pair ? std::max(1, sms / 2) : sms * std::max(1, info.ctas_per_sm);
    const HostSchedule hs = plan_tasks(nest, o, kernel, info.tile_m, info.tile_n, slots);
    const auto& T = hs.tasks;
    const i64 bk = kernel >= gpu::kTcBf16 ? 64 : 32;  // k-slab depth of the kernel's SMEM ring
    GpuIo r;
    r.kernel = kernel;
    r.tile_m = info.tile_m;
    r.tile_n = info.tile_n;
    r.tasks = static_cast<i64>(T.size());
    int G = o.ctas > 0 ? std::min(o.ctas, slots) : slots;
    G = std::max(1, std::min<int>(G, static_cast<int>(T.size())));
    if (hs.blocked) G = hs.grid_fixed;
    r.grid = G;

    // ---- into SMEM (L2 <-> SM): exact per task
    auto& sm = r.smem.op;
    for (const auto& t : T) {
        const i64 mn = static_cast<i64>(t.m) * t.n;
        sm[0].reads += static_cast<i64>(t.m) * t.k;
        sm[1].reads += static_cast<i64>(t.k) * t.n;
        if (t.fixup == 1) {          // contributor: partial to its slot
            sm[2].writes += mn;
        } else if (t.fixup == 2) {   // owner: C in, the seq partials in, C out
            sm[2].reads += mn * (1 + t.seq);
            sm[2].writes += mn;
        } else if (t.slice >= 0) {   // reduce-launch part: partial out (the head part starts from C)
            sm[2].reads += t.from_c ? mn : 0;
            sm[2].writes += mn;
        } else {
            sm[2].reads += mn;
            sm[2].writes += mn;
        }
    }
    for (const auto& rt : hs.red) {  // the fixed-order reduce launch
        const i64 mn = static_cast<i64>(rt.m) * rt.n;
        sm[2].reads += mn * (rt.nslots + 1);
        sm[2].writes += mn;
    }

    // ---- into L2 (the HBM boundary): lockstep waves through an LRU of the L2
    std::vector<std::vector<int32_t>> seq(static_cast<std::size_t>(G));
    if (hs.blocked) {
        for (int c = 0; c < G; ++c)
            for (int32_t q = hs.first[static_cast<std::size_t>(c)]; q < hs.first[static_cast<std::size_t>(c) + 1]; ++q)
                seq[static_cast<std::size_t>(c)].push_back(q);
    } else {
        for (std::size_t q = 0; q < T.size(); ++q) seq[q % static_cast<std::size_t>(G)].push_back(static_cast<int32_t>(q));
    }
    UnitCache lru(l2_bytes, policy);
    const double ea = elem_bytes[0], eb = elem_bytes[1], ec = elem_bytes[2];
    const i64 M = nest.ext.m, N = nest.ext.n;
    std::vector<std::size_t> pos(static_cast<std::size_t>(G), 0);
    std::vector<i64> slab(static_cast<std::size_t>(G), -1);  // next slab of the current task (-1: task not started)
    // One fresh cluster per tile (the 256 x 512 tcgen05 kernel): a tile starts when any earlier one ends, so in
    // steady state the tiles in flight are spread evenly over a tile's k range rather than in lockstep. Modelled
    // by starting slot c c/G of a task later (steps of idle) -- a property of dynamic launch order, no fit.
    std::vector<i64> delay(static_cast<std::size_t>(G), 0);
    if (stagger && !T.empty()) {
        const i64 ns = cdiv(static_cast<i64>(T[0].k), bk);
        for (int c = 0; c < G; ++c) delay[static_cast<std::size_t>(c)] = (ns * c) / G;
    }
    i64 active = G, steps = 0;
    auto c_key = [&](const gpu::Task& t) { return UnitKey{2 + 4 * (static_cast<int64_t>(t.i0) + M * t.j0), 0}; };
    auto w_key = [&](int32_t s) { return UnitKey{3 + 4 * static_cast<int64_t>(s), 0}; };
    while (active > 0) {
        active = 0;
        for (int c = 0; c < G; ++c) {
            auto& sq = seq[static_cast<std::size_t>(c)];
            std::size_t& p = pos[static_cast<std::size_t>(c)];
            i64& s = slab[static_cast<std::size_t>(c)];
            if (p >= sq.size()) continue;
            ++active;
            if (delay[static_cast<std::size_t>(c)] > 0) {
                --delay[static_cast<std::size_t>(c)];
                continue;
            }
            const gpu::Task& t = T[static_cast<std::size_t>(sq[p])];
            const i64 mn = static_cast<i64>(t.m) * t.n;
            if (s < 0) {  // task start: C in, unless the part starts from zero (split-k contributors)
                if (t.fixup == 2 || (t.fixup == 0 && (t.slice < 0 || t.from_c)))
                    lru.access(2, c_key(t), static_cast<int64_t>(mn * ec), false);
                s = 0;
            }
            const i64 nslabs = cdiv(static_cast<i64>(t.k), bk);
            if (s < nslabs) {
                const i64 p0 = t.p0 + s * bk, kk = std::min<i64>(bk, t.p0 + t.k - p0);
                lru.access(0, UnitKey{4 * (static_cast<int64_t>(t.i0) + M * p0), 0},
                           static_cast<int64_t>(static_cast<double>(t.m) * kk * ea), false);
                lru.access(1, UnitKey{1 + 4 * (p0 + nest.ext.k * static_cast<int64_t>(t.j0)), 0},
                           static_cast<int64_t>(static_cast<double>(kk) * t.n * eb), false);
                ++s;
            }
            if (s >= nslabs) {  // task end: C out / partial out / owner fold
                if (t.fixup == 1) {
                    lru.access(2, w_key(t.slice), static_cast<int64_t>(mn * ec), true);
                } else if (t.fixup == 2) {
                    for (int32_t q = 0; q < t.seq; ++q) lru.access(2, w_key(t.slice + q), static_cast<int64_t>(mn * ec), false);
                    lru.access(2, c_key(t), static_cast<int64_t>(mn * ec), true);
                } else if (t.slice >= 0) {
                    lru.access(2, w_key(t.slice), static_cast<int64_t>(mn * ec), true);
                } else {
                    lru.access(2, c_key(t), static_cast<int64_t>(mn * ec), true);
                }
                ++p;
                s = -1;
            }
        }
        ++steps;
    }
    for (const auto& rt : hs.red) {  // reduce launch after the task kernel
        const i64 mn = static_cast<i64>(rt.m) * rt.n;
        gpu::Task t{};
        t.i0 = rt.i0;
        t.j0 = rt.j0;
        for (int32_t q = 0; q < rt.nslots; ++q) lru.access(2, w_key(rt.slot0 + q), static_cast<int64_t>(mn * ec), false);
        lru.access(2, c_key(t), static_cast<int64_t>(mn * ec), false);
        lru.access(2, c_key(t), static_cast<int64_t>(mn * ec), true);
    }
    lru.flush();
    r.lockstep_slabs = steps;
    for (int q = 0; q < 3; ++q) {
        r.hbm_read_bytes[q] = lru.fetched[q];
        r.hbm_write_bytes[q] = lru.written[q];
    }
    (void)N;
    return r;
}

}  // namespace engine
}  // namespace mmm
