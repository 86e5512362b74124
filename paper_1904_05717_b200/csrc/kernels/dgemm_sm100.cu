// FP64 C += A·B task kernels for sm_100a (B200).
//
// A launch processes a list of CTA tasks (gpu.hpp) with a persistent grid.
// Every task is one C region accumulated in ascending k from its incoming
// value — the reference's micro-kernel cell (exec.hpp:35-46) at CTA
// granularity. A and B k-slabs are staged global->shared through a
// multi-stage cp.async ring (the SMEM level of the family member); the C
// region lives in registers for the whole task (the register level).
//
// Numerics variants:
//   k_dmma  — FP64 tensor pipe (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4),
//             the fast path (B200: 64 FP64 FMA/clk/SM on either pipe; the
//             DMMA path leaves the issue slots free for the staging loads).
//   k_simt<FMA>   — one DFMA per (entry, k): bit-exact against a sequential
//                   fma restatement of the reference cell.
//   k_simt<EXACT> — DMUL then DADD per (entry, k): bit-exact against the
//                   reference's own execute() (built -O2, no FMA contraction).
//
// Staging variants of the DMMA kernel:
//   k_dmma      — every thread issues 16-byte cp.async chunks of the slabs
//                 into padded [k][m] / [n][k] stages;
//   k_dmma_tma  — one thread (of a producer warpgroup in the 128x128 kernel)
//                 issues TMA tensor copies (cp.async.bulk.tensor) of the
//                 slabs into 128B-swizzled stages and runs ahead across task
//                 boundaries (the next task's first slabs land under this
//                 task's epilogue).
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "gpu.hpp"

namespace mmm {
namespace gpu {
namespace {

constexpr int kBK = 16;  // k-slab depth per pipeline stage

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp16(double* dst, const double* src, int bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_addr(dst)), "l"(src), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void cp8(double* dst, const double* src, int bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_addr(dst)), "l"(src), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }

// ---- mbarriers (shared::cta) for the warp-decoupled cp.async ring ----
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "MBAR_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra MBAR_WAIT_%=;\n}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_addr(bar)) : "memory");
}
// The same with an address operand `dep` (always 0) added: the instruction then waits for whatever produced dep.
__device__ __forceinline__ void mbar_arrive_after(uint64_t* bar, uint32_t dep) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_addr(bar) + dep) : "memory");
}
// Warp-uniform wait: lane 0 polls, __syncwarp hands its acquire to the
// other lanes. (Every lane polling lets a warp split on the loop branch; the
// lanes then issue their half of a coalesced cp.async separately, and the
// duplicated partial sector requests doubled the kernel's HBM reads.)
__device__ __forceinline__ void mbar_wait_warp(uint64_t* bar, uint32_t parity) {
    if ((threadIdx.x & 31) == 0) mbar_wait(bar, parity);
    __syncwarp();
}
// Arrives on the barrier once every cp.async this thread issued so far has landed.
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_addr(bar)) : "memory");
}
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ---- per-CTA timeline probe (experiment builds only: -DTM_TRACE) ----
// Thread 0 stamps (globaltimer, clock64, event | task << 8) at task-boundary
// events of k_dmma_tma; tm_trace_read copies them out. Off in the product build.
#ifdef TM_TRACE
constexpr int kTraceCtas = 160, kTraceEv = 1024;
__device__ unsigned long long g_trace[kTraceCtas * kTraceEv * 3];
__device__ int g_trace_n[kTraceCtas];
__device__ __forceinline__ void trace_ev(int ev, int ti) {
    if (threadIdx.x != 0 || blockIdx.x >= kTraceCtas) return;
    const int i = g_trace_n[blockIdx.x]++;
    if (i >= kTraceEv) return;
    unsigned long long gt, ck;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(ck));
    unsigned long long* p = g_trace + (static_cast<size_t>(blockIdx.x) * kTraceEv + i) * 3;
    p[0] = gt;
    p[1] = ck;
    p[2] = static_cast<unsigned long long>(ev) | (static_cast<unsigned long long>(ti) << 8);
}
#define TM_TRACE_EV(ev, ti) trace_ev(ev, ti)
#else
#define TM_TRACE_EV(ev, ti) ((void)0)
#endif

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

// Barrier over the CTA's task-running threads: all of them (__syncthreads), or, in kernels with an extra
// producer warp behind them, the first NC threads (named barrier 1).
template <int NC>
__device__ __forceinline__ void cta_sync() {
    if constexpr (NC == 0) __syncthreads();
    else asm volatile("bar.sync 1, %0;\n" ::"n"(NC) : "memory");
}

// ---- ordering between tasks on the same C region (faithful schedule) ----
// (fix-up tasks carry tile = -2 - counter, so this protocol skips them)
template <int NC = 0>
__device__ __forceinline__ void wait_turn(const Args& a, const Task& t) {
    if (t.tile < 0 || t.seq <= 0) return;
    if (threadIdx.x == 0) {
        int v;
        for (;;) {
            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(a.progress + t.tile) : "memory");
            if (v >= t.seq) break;
            __nanosleep(100);
        }
    }
    cta_sync<NC>();
}

template <int NC = 0>
__device__ __forceinline__ void signal_done(const Args& a, const Task& t, int ti) {
    if (t.tile < 0) return;
    cta_sync<NC>();
    if (threadIdx.x == 0) {
        __threadfence();
        asm volatile("st.release.gpu.global.s32 [%0], %1;\n" ::"l"(a.progress + t.tile), "r"(t.seq + 1) : "memory");
        if (a.done) {  // pipeline: count the block's finished tiles (the D2H copy waits on it)
            const int dn = a.tasks[ti].done;
            if (dn > 0) asm volatile("red.release.gpu.global.add.s32 [%0], 1;\n" ::"l"(a.done + dn - 1) : "memory");
        }
    }
}

// Copy-engine-fed pipeline: the task's inputs are in HBM once the copy stream
// has written its flag (cuStreamWriteValue32 after the copies, in order).
template <int NC = 0>
__device__ __forceinline__ void wait_ready(const Args& a, const Task& t) {
    if (t.ready == 0) return;
    if (threadIdx.x == 0) {
        const int32_t* f = a.ready + t.ready - 1;
        int v;
        for (;;) {
            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(f) : "memory");
            if (v != 0) break;
            __nanosleep(256);
        }
    }
    cta_sync<NC>();
}

// Split-k fix-up inside the task kernel (Task::fixup). Contributors publish
// their partial with a release increment of the tile's counter; the owner
// acquires the count, then adds the partials in slot order -- the same sums
// in the same order as k_reduce_tiles, one launch and one C round trip less.
template <int NC = 0>
__device__ __forceinline__ void signal_partial(const Args& a, const Task& t) {
    cta_sync<NC>();
    if (threadIdx.x == 0) {
        __threadfence();
        asm volatile("red.release.gpu.global.add.s32 [%0], 1;\n" ::"l"(a.progress + (-2 - t.tile)) : "memory");
    }
}

// Row and column of a lane's C pair (rows r, r+1 of column c) in DMMA
// group (mi, ni). SWZ: the TMA kernel's m and n orders. A 64-bit shared load
// is served per half-warp (16 lanes = 128 B). In the 128B-swizzled stages
// (16-byte unit ^ row%8) the lanes of a half-warp read 4 k rows (A) or 4 n
// rows (B); with consecutive m or n they would pair rows r and r^1 on the
// same units (2-way conflict). Lane g of group mi takes m = (g&1) +
// 8((g>>1)&1) + 2(g>>2) + 4(mi&1) of chunk mi/2 (units {x, x^4} per
// half-warp) and lane g of group ni takes n = 2(g&3) + (g>>2) (even n rows in
// one half-warp, odd in the other): one wavefront per half-warp. The orders
// only permute which lane holds which C entry; every entry sees the same
// DMMA groups in the same k order as in the cp.async kernel.
template <bool SWZ>
__device__ __forceinline__ int c_row(int wm0, int mi, int tq) {
    if constexpr (SWZ)
        return wm0 + (mi >> 1) * 16 + (mi & 1) * 4 + 8 * (tq & 1) + 2 * (tq >> 1);
    else
        return wm0 + mi * 8 + 2 * tq;
}
template <bool SWZ>
__device__ __forceinline__ int c_col(int wn0, int ni, int g) {
    if constexpr (SWZ)
        return wn0 + ni * 8 + 2 * (g & 3) + (g >> 2);
    else
        return wn0 + ni * 8 + g;
}

template <int FM, int FN, bool SWZ = false, int NC = 0>
__device__ __forceinline__ void fold_partials(const Args& a, const Task& t, double (&acc)[FM][FN][2], int wm0,
                                              int wn0, int g, int tq) {
    if (threadIdx.x == 0) {
        int32_t* ctr = a.progress + (-2 - t.tile);
        int v;
        for (;;) {
            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(ctr) : "memory");
            if (v >= t.seq) break;
            __nanosleep(64);
        }
        *ctr = 0;  // every contribution is in: ready for the next launch
    }
    cta_sync<NC>();
    for (int q = 0; q < t.seq; ++q) {
        const double* w = a.work + static_cast<int64_t>(t.slice + q) * a.work_slice;
#pragma unroll
        for (int mi = 0; mi < FM; ++mi)
#pragma unroll
            for (int ni = 0; ni < FN; ++ni) {
                const int r = c_row<SWZ>(wm0, mi, tq), c = c_col<SWZ>(wn0, ni, g);
                // slots are tile-shaped (work_ld = tile rows, even) and 16-byte aligned
                const double2 v = __ldcg(reinterpret_cast<const double2*>(w + r + static_cast<int64_t>(c) * a.work_ld));
                acc[mi][ni][0] = __dadd_rn(acc[mi][ni][0], v.x);
                acc[mi][ni][1] = __dadd_rn(acc[mi][ni][1], v.y);
            }
    }
}

// Where a task reads its starting value and writes its result.
struct Dest {
    const double* src;  // nullptr: start from zero
    double* dst;
    int64_t ld_src, ld_dst;
    int64_t oi, oj;     // destination coordinates of the task's (0, 0)
};
__device__ __forceinline__ Dest resolve(const Args& a, const Task& t) {
    Dest d;
    if (t.fixup == 1) {  // contributor: partial from zero into its slot
        d.src = nullptr;
        d.ld_src = a.ldc;
        d.dst = a.work + static_cast<int64_t>(t.slice) * a.work_slice;
        d.ld_dst = a.work_ld;
        d.oi = 0;
        d.oj = 0;
    } else if (t.slice < 0 || t.fixup == 2) {
        d.src = a.C;
        d.dst = a.C;
        d.ld_src = d.ld_dst = a.ldc;
        d.oi = t.i0;
        d.oj = t.j0;
    } else {  // a k-part of a split tile: partial into its compact slot
        d.src = t.from_c ? a.C : nullptr;
        d.ld_src = a.ldc;
        d.dst = a.work + static_cast<int64_t>(t.slice) * a.work_slice;
        d.ld_dst = a.work_ld;
        d.oi = 0;
        d.oj = 0;
    }
    return d;
}

// ---- shared-memory geometry ----
// As[k][m] (row stride BM+4 doubles: the 4-double pad puts the four k rows a
// DMMA A-fragment touches 8 banks apart -> 2 wavefronts per 64-bit load, the
// minimum). Bs[n][k] (stride BK+4, same argument for the B-fragment).
// The SIMT kernels keep B transposed, Bt[k][n], so a thread's n-run is
// contiguous.
template <int BM, int BN, bool BT>
struct Geo {
    static constexpr int LDA = BM + 4;
    static constexpr int LDB = BT ? BN + 4 : kBK + 4;
    static constexpr int A_ELEMS = kBK * LDA;
    static constexpr int B_ELEMS = BT ? kBK * LDB : BN * LDB;
    static constexpr int STAGE = A_ELEMS + B_ELEMS;
};

// One k-slab [p, p+BK) of the task's A rows and B columns into one stage;
// out-of-range elements are zero-filled (cp.async src-size < cp-size).
template <int BM, int BN, int NT, bool V16, bool BT>
__device__ __forceinline__ void load_slab(double* As, double* Bs, const Args& a, const Task& t, int p) {
    using G = Geo<BM, BN, BT>;
    const int tid = threadIdx.x;
    const int klim = t.p0 + t.k - p;
    const double* Ab = a.A + static_cast<int64_t>(t.i0) + static_cast<int64_t>(p) * a.lda;
    const double* Bb = a.B + static_cast<int64_t>(p) + static_cast<int64_t>(t.j0) * a.ldb;
    if constexpr (V16) {
#pragma unroll
        for (int q = tid; q < BM * kBK / 2; q += NT) {
            const int c = q / (BM / 2), r = (q % (BM / 2)) * 2;
            const int v = c < klim ? min(max(t.m - r, 0), 2) : 0;
            cp16(As + c * G::LDA + r, v ? Ab + r + static_cast<int64_t>(c) * a.lda : a.A, v * 8);
        }
    } else {
#pragma unroll 4
        for (int q = tid; q < BM * kBK; q += NT) {
            const int c = q / BM, r = q % BM;
            const bool v = c < klim && r < t.m;
            cp8(As + c * G::LDA + r, v ? Ab + r + static_cast<int64_t>(c) * a.lda : a.A, v ? 8 : 0);
        }
    }
    if constexpr (BT) {
        // Bt[k][n]: consecutive threads walk k down one B column (coalesced).
#pragma unroll 4
        for (int q = tid; q < BN * kBK; q += NT) {
            const int n = q / kBK, c = q % kBK;
            const bool v = c < klim && n < t.n;
            cp8(Bs + c * G::LDB + n, v ? Bb + c + static_cast<int64_t>(n) * a.ldb : a.B, v ? 8 : 0);
        }
    } else if constexpr (V16) {
#pragma unroll
        for (int q = tid; q < BN * kBK / 2; q += NT) {
            const int n = q / (kBK / 2), c = (q % (kBK / 2)) * 2;
            const int v = n < t.n ? min(max(klim - c, 0), 2) : 0;
            cp16(Bs + n * G::LDB + c, v ? Bb + c + static_cast<int64_t>(n) * a.ldb : a.B, v * 8);
        }
    } else {
#pragma unroll 4
        for (int q = tid; q < BN * kBK; q += NT) {
            const int n = q / kBK, c = q % kBK;
            const bool v = c < klim && n < t.n;
            cp8(Bs + n * G::LDB + c, v ? Bb + c + static_cast<int64_t>(n) * a.ldb : a.B, v ? 8 : 0);
        }
    }
}


// Element-granular staging (any alignment, any origin) for the DMMA kernel's
// non-16B path: As[k][m] (stride BM+4), Bs[n][k] (stride BK+4).
template <int BM, int BN, int BK, int NT>
__device__ __forceinline__ void load_slab_generic(double* As, double* Bs, const Args& a, const Task& t, int p) {
    constexpr int LDA = BM + 4, LDB = BK + 4;
    const int tid = threadIdx.x;
    const int klim = t.p0 + t.k - p;
    const double* Ab = a.A + static_cast<int64_t>(t.i0) + static_cast<int64_t>(p) * a.lda;
    const double* Bb = a.B + static_cast<int64_t>(p) + static_cast<int64_t>(t.j0) * a.ldb;
#pragma unroll 4
    for (int q = tid; q < BM * BK; q += NT) {
        const int c = q / BM, r = q % BM;
        const bool v = c < klim && r < t.m;
        cp8(As + c * LDA + r, v ? Ab + r + static_cast<int64_t>(c) * a.lda : a.A, v ? 8 : 0);
    }
#pragma unroll 4
    for (int q = tid; q < BN * BK; q += NT) {
        const int n = q / BK, c = q % BK;
        const bool v = c < klim && n < t.n;
        cp8(Bs + n * LDB + c, v ? Bb + c + static_cast<int64_t>(n) * a.ldb : a.B, v ? 8 : 0);
    }
}

// ============================== DMMA kernel ==============================
// Per-task staging state for the 16-byte path: every thread owns a fixed set
// of 16B chunks of the A and B slabs, so source pointers, shared-memory
// offsets and row/column validity are computed once per task; per slab only
// the k validity (last slab) changes. The chunks are issued between the DMMA
// groups of the current slab so the staging instructions fill issue slots
// the FP64 pipe leaves idle.
template <int BM, int BN, int BK, int NT>
struct Stager {
    static constexpr int LDA = BM + 4, LDB = BK + 4;
    static constexpr int A_ELEMS = BK * LDA, STAGE = A_ELEMS + BN * LDB;
    static constexpr int A_PER_COL = BM / 2, B_PER_COL = BK / 2;
    static constexpr int A_CH = BM * BK / 2 / NT, B_CH = BN * BK / 2 / NT;
    static constexpr int A_CSTEP = NT / A_PER_COL, B_NSTEP = NT / B_PER_COL;
    static_assert(NT % A_PER_COL == 0 && NT % B_PER_COL == 0, "thread count must tile the slab");
    const double* a;  // A(i0 + ar, p0 + ac0)
    const double* b;  // B(p0 + bc, j0 + bn0)
    int64_t a_ld, b_ld;
    int ac0, bc;      // k offsets of this thread's chunks within a slab
    int a_bytes;      // 16/8/0: rows ar, ar+1 inside the task
    uint32_t b_nvalid;  // bit it: column bn0 + it*B_NSTEP inside the task
    uint32_t a_dst, b_dst;  // shared byte addresses in stage 0
    const double* a_any;
    const double* b_any;

    __device__ __forceinline__ void init(const Args& g, const Task& t, const double* smem) {
        const int tid = threadIdx.x;
        const int ar = (tid % A_PER_COL) * 2;
        ac0 = tid / A_PER_COL;
        bc = (tid % B_PER_COL) * 2;
        const int bn0 = tid / B_PER_COL;
        a_ld = g.lda;
        b_ld = g.ldb;
        a = g.A + static_cast<int64_t>(t.i0) + ar + static_cast<int64_t>(t.p0 + ac0) * g.lda;
        b = g.B + static_cast<int64_t>(t.p0) + bc + static_cast<int64_t>(t.j0 + bn0) * g.ldb;
        a_bytes = min(max(t.m - ar, 0), 2) * 8;
        b_nvalid = 0;
#pragma unroll
        for (int it = 0; it < B_CH; ++it) b_nvalid |= (bn0 + it * B_NSTEP < t.n ? 1u : 0u) << it;
        a_dst = smem_addr(smem + ac0 * LDA + ar);
        b_dst = smem_addr(smem + A_ELEMS + bn0 * LDB + bc);
        a_any = g.A;
        b_any = g.B;
    }
    // klim = valid k columns from this slab's start (>= BK for interior slabs)
    __device__ __forceinline__ void issue_a(int slab, int stage, int klim) const {
        const double* src = a + static_cast<int64_t>(slab) * BK * a_ld;
        const uint32_t dst = a_dst + stage * STAGE * 8;
#pragma unroll
        for (int it = 0; it < A_CH; ++it) {
            const int bytes = (ac0 + it * A_CSTEP < klim) ? a_bytes : 0;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst + it * A_CSTEP * LDA * 8),
                         "l"(bytes ? src + static_cast<int64_t>(it) * A_CSTEP * a_ld : a_any), "r"(bytes)
                         : "memory");
        }
    }
    __device__ __forceinline__ void issue_b(int slab, int stage, int klim) const {
        const double* src = b + static_cast<int64_t>(slab) * BK;
        const uint32_t dst = b_dst + stage * STAGE * 8;
        const int kb = min(max(klim - bc, 0), 2) * 8;
#pragma unroll
        for (int it = 0; it < B_CH; ++it) {
            const int bytes = ((b_nvalid >> it) & 1u) ? kb : 0;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst + it * B_NSTEP * LDB * 8),
                         "l"(bytes ? src + static_cast<int64_t>(it) * B_NSTEP * b_ld : b_any), "r"(bytes)
                         : "memory");
        }
    }
};

// The slab ring is synchronised by mbarriers, not a CTA barrier per slab:
// full[stage] completes when every thread's cp.async for the slab has landed
// (cp.async.mbarrier.arrive.noinc), empty[stage] when every warp has
// finished reading it. A warp waits (warp-uniformly) only for the slab it
// consumes and, two k steps into a slab, for the previous slab's stage to be
// free before refilling it -- so the FP64 pipe does not drain at every slab
// boundary. Measured at 16384^3 against the __syncthreads ring: 94.7 ->
// 95.4 % of peak, HBM reads 63 -> 62 GB. Refilling at a slab's last k step
// was faster still (95.8 %) but doubled the HBM reads, as did per-lane
// polling of the barriers (tools/l2_ab.sh).
// FIX: compile the in-kernel split-k fix-up (Task::fixup) into this variant.
template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool V16, bool FIX = true>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32, 1) k_dmma(Args a) {
    constexpr int NWM = BM / WM, NT = (BM / WM) * (BN / WN) * 32;
    constexpr int FM = WM / 8, FN = WN / 8, KK = BK / 4;
    constexpr int PD = STAGES - 1;                 // slabs in flight ahead of the one being consumed
    constexpr int ISSUE_KK = 2 < KK ? 2 : KK - 1;  // k step of a slab at which the refill is issued
    using S = Stager<BM, BN, BK, NT>;
    extern __shared__ __align__(128) double smem[];
    __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < STAGES; ++q) {
            mbar_init(&full[q], NT);
            mbar_init(&empty[q], NT / 32);
        }
    }
    __syncthreads();
    uint32_t n_issue = 0, n_use = 0;  // slabs issued / consumed by this CTA so far (ring position and phase)

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, tq = lane & 3;
    const int wm0 = (warp % NWM) * WM, wn0 = (warp / NWM) * WN;

    const int t_hi = a.cta_first ? a.cta_first[blockIdx.x + 1] : a.ntasks;
    const int t_step = a.cta_first ? 1 : static_cast<int>(gridDim.x);
    int ti = a.cta_first ? a.cta_first[blockIdx.x] : static_cast<int>(blockIdx.x);
    for (; ti < t_hi; ti += t_step) {
        const Task t = a.tasks[ti];
        wait_ready(a, t);
        wait_turn(a, t);
        const int nk = (t.k + BK - 1) / BK;
        S st;
        if constexpr (V16) st.init(a, t, smem);
        // issue slab x of this task into the next ring stage
        auto produce = [&](int x) {
            const uint32_t stage = n_issue % STAGES;
            if (n_issue >= STAGES) mbar_wait_warp(&empty[stage], ((n_issue / STAGES) - 1) & 1);
            if constexpr (V16) {
                st.issue_a(x, stage, t.k - x * BK);
                st.issue_b(x, stage, t.k - x * BK);
            } else {
                double* sp = smem + stage * S::STAGE;
                load_slab_generic<BM, BN, BK, NT>(sp, sp + S::A_ELEMS, a, t, t.p0 + x * BK);
            }
            cp_async_arrive(&full[stage]);
            ++n_issue;
        };
        for (int s = 0; s < PD && s < nk; ++s) produce(s);

        const Dest d = resolve(a, t);
        // The MMA computes the transposed tile (D' = B^T A^T, operands
        // swapped): lane (g, tq) then holds C rows wm0+mi*8+2tq+{0,1} of
        // column wn0+ni*8+g — two consecutive column-major elements, so the C
        // tile moves with one 16-byte access per pair instead of two 8-byte
        // ones (same products, same k order).
        double acc[FM][FN][2];
        const bool src_vec = d.src != nullptr && ((reinterpret_cast<uintptr_t>(d.src) & 15) | (d.ld_src & 1) |
                                                  (static_cast<int64_t>(t.i0) & 1)) == 0;
#pragma unroll
        for (int mi = 0; mi < FM; ++mi)
#pragma unroll
            for (int ni = 0; ni < FN; ++ni) {
                const int r = wm0 + mi * 8 + 2 * tq, c = wn0 + ni * 8 + g;
                const double* p = d.src + (t.i0 + r) + static_cast<int64_t>(t.j0 + c) * d.ld_src;
                if (src_vec && r + 1 < t.m && c < t.n) {
                    const double2 v = __ldcg(reinterpret_cast<const double2*>(p));
                    acc[mi][ni][0] = v.x;
                    acc[mi][ni][1] = v.y;
                } else {
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        acc[mi][ni][e] = (d.src && r + e < t.m && c < t.n) ? __ldcg(p + e) : 0.0;
                }
            }

        for (int s = 0; s < nk; ++s) {
            const uint32_t stage = n_use % STAGES;
            mbar_wait_warp(&full[stage], (n_use / STAGES) & 1);
            const int nx = s + PD;
            const double* As = smem + stage * S::STAGE;
            const double* Bs = As + S::A_ELEMS;
#pragma unroll
            for (int kk = 0; kk < KK; ++kk) {
                double af[FM], bf[FN];
#pragma unroll
                for (int mi = 0; mi < FM; ++mi) af[mi] = As[(kk * 4 + tq) * S::LDA + wm0 + mi * 8 + g];
#pragma unroll
                for (int ni = 0; ni < FN; ++ni) bf[ni] = Bs[(wn0 + ni * 8 + g) * S::LDB + kk * 4 + tq];
#pragma unroll
                for (int mi = 0; mi < FM; ++mi)
#pragma unroll
                    for (int ni = 0; ni < FN; ++ni) dmma884(acc[mi][ni], bf[ni], af[mi]);
                // refill the stage of the previous slab a few k steps into this one
                if (kk == ISSUE_KK && nx < nk) produce(nx);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stage]);
            ++n_use;
        }
        if constexpr (FIX) {
            if (t.fixup == 2) fold_partials<FM, FN>(a, t, acc, wm0, wn0, g, tq);
        }

        const int64_t di = d.oi, dj = d.oj;
        const bool dst_vec = ((reinterpret_cast<uintptr_t>(d.dst) & 15) | (d.ld_dst & 1) | (di & 1)) == 0;
#pragma unroll
        for (int mi = 0; mi < FM; ++mi)
#pragma unroll
            for (int ni = 0; ni < FN; ++ni) {
                const int r = wm0 + mi * 8 + 2 * tq, c = wn0 + ni * 8 + g;
                double* p = d.dst + (di + r) + (dj + c) * d.ld_dst;
                if (dst_vec && r + 1 < t.m && c < t.n) {
                    *reinterpret_cast<double2*>(p) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
                } else {
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        if (r + e < t.m && c < t.n) p[e] = acc[mi][ni][e];
                }
            }
        if (FIX && t.fixup == 1) signal_partial(a, t);
        else signal_done(a, t, ti);
    }
}

// ========================== DMMA kernel, TMA-fed ==========================
// The SMEM level of the family member as a TMA ring: A's slab (BM rows x BK
// columns of the column-major A) lands as BM/16 boxes of 16 x BK doubles
// ([k][16 m] rows of 128 B), B's slab (BK x BN) as BK/16 boxes of 16 x BN
// ([n][16 k] rows), both with the 128-byte swizzle, so no padding and no
// per-thread address arithmetic. One thread is the producer. In the 128x128
// kernel it is lane 0 of a warp of its own (the producer warpgroup, PW; see
// TM_PRODUCER_WARP below): it keeps every stage filled, held back only by
// the stages' empty barriers, following the CTA's task list across task
// boundaries, so the next task's first slabs arrive while this task's C
// tile is written back; entering a task it also warms L2 with that task's C
// tile (one bulk tensor prefetch), so the C load at the task's start hits
// L2; a task's copy-engine data flag (Task::ready) it polls itself.
// In the 128x64 / 64x64 variants (PW = false) the producer is lane 0 of DMMA
// warp 0: it keeps STAGES-1 slabs in flight ahead of the slab being consumed
// and issues the refill of a stage at k step TM_TMA_ISSUE_KK of the slab
// after it (measured: step 2 beats steps 1 and 5 by 0.3-2 points); it does
// not run ahead into a task whose data flag it has not seen.
// full[s] completes on the TMA byte count; empty[s] on one arrive per warp.
#ifndef TM_TMA_ISSUE_KK
#define TM_TMA_ISSUE_KK 2
#endif
// Experiment knobs (tools/build_variant.sh; the product build leaves them at their defaults): the k-slab depth
// and stage count of the 128x128 TMA kernel, and a start-up stagger of its warp groups (warps w, w+4, w+8,
// w+12 share an SM sub-partition; group w/4 starts (NW/4-1 - w/4) * TM_STAGGER cycles late, so the groups reach
// the task boundaries' C exchange one after the other). All measured and rejected:
// profiles/ab_r02_fp64_slab_depth_stagger.json.
#ifndef TM_TMA_BK128
#define TM_TMA_BK128 32
#endif
#ifndef TM_TMA_ST128
#define TM_TMA_ST128 3
#endif
#ifndef TM_STAGGER
#define TM_STAGGER 0
#endif
// TM_PRODUCER_WARP (default 1; 0 = the round-1/2 arrangement, an A/B knob): the 128x128 TMA kernel runs a
// fifth warpgroup whose first lane only issues the TMA copies, instead of warp 0's lane 0 issuing them between
// its own DMMAs (that warp then trailed the other fifteen, and every slab waited for it). The register file
// is per SM sub-partition (16384 registers), so five warps there start at 96 registers each; the producer
// warps then drop to 24 (setmaxnreg.dec) and the DMMA warps grow to 112: the pool setmaxnreg draws on is what
// the CTA's own warps released (16 x 112 + 4 x 24 <= 20 x 96; 120 would wait forever).
// Measured (profiles/ab_r02_fp64_producer_warpgroup.json): 16384^3 96.6 -> 98.2 % of the DMMA peak, rank-k
// 90.7 -> 95.6 %, inner product 94.5 -> 96.3 %, panel-panel 91.6 -> 94.2 %, 2048^3 87-88.5 -> 89.5 %.
#ifndef TM_PRODUCER_WARP
#define TM_PRODUCER_WARP 1
#endif
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_addr(bar)), "r"(c0), "r"(c1)
        : "memory");
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool FIX = true, bool PW = false>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32 + (PW ? 128 : 0), 1)
    k_dmma_tma(Args a, const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const __grid_constant__ CUtensorMap tmC) {
    constexpr int NWM = BM / WM, NW = (BM / WM) * (BN / WN);
    constexpr int NC = PW ? NW * 32 : 0;  // threads behind the task-boundary barriers (cta_sync)
    constexpr int FM = WM / 8, FN = WN / 8, KK = BK / 4;
    constexpr int PD = STAGES - 1;
    constexpr int ISSUE_KK = TM_TMA_ISSUE_KK < KK - 1 ? TM_TMA_ISSUE_KK : KK - 1;  // k step of the refill
    constexpr uint32_t A_CHUNK = BK * 128, B_CHUNK = BN * 128;  // bytes of one 16-wide box
    constexpr uint32_t A_BYTES = BM * BK * 8, STAGE_BYTES = A_BYTES + BN * BK * 8;
    static_assert(BM % 16 == 0 && BK % 16 == 0 && WM % 16 == 0 && WN % 8 == 0, "16-wide swizzle atoms");
    static_assert(A_CHUNK % 1024 == 0 && B_CHUNK % 1024 == 0, "boxes must start on 1024-byte swizzle periods");
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
    const uint32_t raw = smem_addr(smem_raw);
    const uint32_t sbase = (raw + 1023u) & ~1023u;
    const unsigned char* sgen = smem_raw + (sbase - raw);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < STAGES; ++q) {
            mbar_init(&full[q], 1);
            mbar_init(&empty[q], NW);
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    }
    __syncthreads();

    const int g = lane >> 2, tq = lane & 3;
    const int wm0 = (warp % NWM) * WM, wn0 = (warp / NWM) * WN;
    // Fragment byte offsets inside a stage. A element (k, m) of a slab sits
    // at box m/16 | row k | unit ((m%16)/2) ^ (k%8) | half m%2 -- disjoint bit
    // fields (box * A_CHUNK, k << 7, unit << 4, half << 3); B element (k, n)
    // at box k/16 | row n | unit ((k%16)/2) ^ (n%8) | half k%2. With k =
    // 4kk + tq and the SWZ orders the (mi&1, kk&1) / (kk&3) dependence of the
    // unit is a bit flip of a per-lane base, the rest an immediate.
    const int nn = 2 * (g & 3) + (g >> 2);  // n % 8 of this lane's B rows
    const uint32_t aoff = (wm0 >> 4) * A_CHUNK + tq * 128 + (((4 * ((g >> 1) & 1) + (g >> 2)) ^ tq) << 4) + (g & 1) * 8;
    const uint32_t boff = A_BYTES + (wn0 + nn) * 128 + (((tq >> 1) ^ nn) << 4) + (tq & 1) * 8;

    const int t_hi = a.cta_first ? a.cta_first[blockIdx.x + 1] : a.ntasks;
    const int t_step = a.cta_first ? 1 : static_cast<int>(gridDim.x);
    int ti = a.cta_first ? a.cta_first[blockIdx.x] : static_cast<int>(blockIdx.x);

    // Producer cursor, kept in shared memory (only warp 0 touches it, so it
    // costs the consumers no registers): next slab to issue = slab `slab` of
    // task `ti`; `issued` counts slabs issued by this CTA.
    __shared__ struct {
        int ti, slab, nk, i0, j0, p0, ready;
        uint32_t issued;
    } pc;
    uint32_t n_use = 0;
    auto p_load = [&](int from) {  // lane 0
        int x = from;
        for (; x < t_hi; x += t_step) {
            const Task pt = a.tasks[x];
            if (pt.k <= 0) continue;
            pc.nk = (pt.k + BK - 1) / BK;
            pc.i0 = pt.i0;
            pc.j0 = pt.j0;
            pc.p0 = pt.p0;
            pc.ready = pt.ready;
            if (a.prefetch_c && pt.slice < 0 && pt.ready == 0 && pc.issued > 0) {  // (not the CTA's first task)
                // the tile's C is read at the task's start, about two slabs from now: warm L2 with it
                asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];\n" ::"l"(
                                 reinterpret_cast<uint64_t>(&tmC)),
                             "r"(pt.i0), "r"(pt.j0)
                             : "memory");
            }
            break;
        }
        pc.ti = x;
        pc.slab = 0;
    };
    // warp 0: issue slabs until `limit` have been issued in total (lane 0 works, the warp waits)
    auto top_up = [&](uint32_t limit, int cur) {
        if (lane == 0) {
            while (pc.issued < limit && pc.ti < t_hi) {
                if (pc.slab == 0 && pc.ti != cur && pc.ready != 0) break;  // its data flag is awaited at its start
                const uint32_t n = pc.issued, stage = n % STAGES;
                if (n >= STAGES) mbar_wait(&empty[stage], ((n / STAGES) - 1) & 1);
                mbar_expect_tx(&full[stage], STAGE_BYTES);
                const uint32_t sa = sbase + stage * STAGE_BYTES;
                const int kc = pc.p0 + pc.slab * BK, i0 = pc.i0, j0 = pc.j0;
#pragma unroll
                for (int c = 0; c < BM / 16; ++c) tma_2d(sa + c * A_CHUNK, &tmA, &full[stage], i0 + 16 * c, kc);
#pragma unroll
                for (int c = 0; c < BK / 16; ++c)
                    tma_2d(sa + A_BYTES + c * B_CHUNK, &tmB, &full[stage], kc + 16 * c, j0);
                pc.issued = n + 1;
                if (++pc.slab == pc.nk) p_load(pc.ti + t_step);
            }
        }
        __syncwarp();
    };
    if constexpr (PW) {
        // The producer warp: lane 0 walks the CTA's task list and keeps every stage of the ring filled, held
        // back only by the stages' empty barriers (and a task's copy-engine data flag); then the warp exits.
        if (warp >= NW) {
            asm volatile("setmaxnreg.dec.sync.aligned.u32 24;\n");
            if (warp == NW && lane == 0) {
                uint32_t n = 0;
                for (int x = ti; x < t_hi; x += t_step) {
                    const Task pt = a.tasks[x];
                    if (pt.k <= 0) continue;
                    if (pt.ready != 0) {
                        const int32_t* f = a.ready + pt.ready - 1;
                        int v;
                        for (;;) {
                            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(f) : "memory");
                            if (v != 0) break;
                            __nanosleep(256);
                        }
                    }
                    if (a.prefetch_c && pt.slice < 0 && pt.ready == 0 && n > 0)
                        asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];\n" ::"l"(
                                         reinterpret_cast<uint64_t>(&tmC)),
                                     "r"(pt.i0), "r"(pt.j0)
                                     : "memory");
                    const int pnk = (pt.k + BK - 1) / BK;
                    for (int sl = 0; sl < pnk; ++sl, ++n) {
                        const uint32_t stage = n % STAGES;
                        if (n >= STAGES) mbar_wait(&empty[stage], ((n / STAGES) - 1) & 1);
                        mbar_expect_tx(&full[stage], STAGE_BYTES);
                        const uint32_t sa = sbase + stage * STAGE_BYTES;
                        const int kc = pt.p0 + sl * BK;
#pragma unroll
                        for (int c = 0; c < BM / 16; ++c) tma_2d(sa + c * A_CHUNK, &tmA, &full[stage], pt.i0 + 16 * c, kc);
#pragma unroll
                        for (int c = 0; c < BK / 16; ++c)
                            tma_2d(sa + A_BYTES + c * B_CHUNK, &tmB, &full[stage], kc + 16 * c, pt.j0);
                    }
                }
            }
            return;
        }
        asm volatile("setmaxnreg.inc.sync.aligned.u32 112;\n");
    } else {
        if (threadIdx.x == 0) {
            pc.issued = 0;
            p_load(ti);
        }
        __syncwarp();
    }
    TM_TRACE_EV(0, 0);
    [[maybe_unused]] bool restagger = true;

    for (; ti < t_hi; ti += t_step) {
        const Task t = a.tasks[ti];
        // last task of this CTA: let a programmatically dependent launch (the next segment of the task list)
        // start its CTAs as this launch's CTAs retire, instead of after the slowest one
        if (a.pdl_trigger && ti + t_step >= t_hi) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
        wait_ready<NC>(a, t);
        wait_turn<NC>(a, t);
        TM_TRACE_EV(1, ti);
        const int nk = (t.k + BK - 1) / BK;
        if constexpr (!PW) {
            if (warp == 0) top_up(n_use + PD, ti);
        }
        if constexpr (TM_STAGGER > 0 && NW >= 8) {
            if (restagger) {  // (again after a task whose fix-up brought the CTA's warps back in step)
                const long long t0 = clock64(), wait = static_cast<long long>(NW / 4 - 1 - (warp >> 2)) * TM_STAGGER;
                while (clock64() - t0 < wait) {}
                restagger = false;
            }
            if (FIX && t.fixup != 0) restagger = true;
        }

        const Dest d = resolve(a, t);
        double acc[FM][FN][2];
        const bool src_vec = d.src != nullptr && ((reinterpret_cast<uintptr_t>(d.src) & 15) | (d.ld_src & 1) |
                                                  (static_cast<int64_t>(t.i0) & 1)) == 0;
#pragma unroll
        for (int mi = 0; mi < FM; ++mi)
#pragma unroll
            for (int ni = 0; ni < FN; ++ni) {
                const int r = c_row<true>(wm0, mi, tq), c = c_col<true>(wn0, ni, g);
                const double* p = d.src + (t.i0 + r) + static_cast<int64_t>(t.j0 + c) * d.ld_src;
                if (src_vec && r + 1 < t.m && c < t.n) {
                    const double2 v = __ldcg(reinterpret_cast<const double2*>(p));
                    acc[mi][ni][0] = v.x;
                    acc[mi][ni][1] = v.y;
                } else {
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        acc[mi][ni][e] = (d.src && r + e < t.m && c < t.n) ? __ldcg(p + e) : 0.0;
                }
            }
        TM_TRACE_EV(2, ti);

        for (int s = 0; s < nk; ++s) {
            const uint32_t stage = n_use % STAGES;
            mbar_wait_warp(&full[stage], (n_use / STAGES) & 1);
#ifdef TM_TRACE
            if (s == 0) TM_TRACE_EV(3, ti);
#endif
            const unsigned char* st = sgen + stage * STAGE_BYTES;
            uint32_t dep = 0;
#pragma unroll
            for (int kk = 0; kk < KK; ++kk) {
                double af[FM], bf[FN];
#pragma unroll
                for (int mi = 0; mi < FM; ++mi)
                    af[mi] = *reinterpret_cast<const double*>(st + (aoff ^ ((mi & 1) << 5) ^ ((kk & 1) << 6)) +
                                                              (mi >> 1) * A_CHUNK + kk * 512);
#pragma unroll
                for (int ni = 0; ni < FN; ++ni)
                    bf[ni] = *reinterpret_cast<const double*>(st + (boff ^ ((kk & 3) << 5)) + (kk >> 2) * B_CHUNK +
                                                              ni * 1024);
                if (kk >= KK - 2) {
#pragma unroll
                    for (int mi = 0; mi < FM; ++mi) dep ^= static_cast<uint32_t>(__double2hiint(af[mi]));
#pragma unroll
                    for (int ni = 0; ni < FN; ++ni) dep ^= static_cast<uint32_t>(__double2hiint(bf[ni]));
                }
#pragma unroll
                for (int mi = 0; mi < FM; ++mi)
#pragma unroll
                    for (int ni = 0; ni < FN; ++ni) dmma884(acc[mi][ni], bf[ni], af[mi]);
                if constexpr (!PW) {
                    if (kk == ISSUE_KK && warp == 0) top_up(n_use + PD + 1, ti);
                }
            }
            // Release the stage only once its fragment loads have RETURNED: the arrive's address depends on
            // the slab's last loaded values (dep & a.zero == 0, known only at run time). ptxas otherwise
            // hoists the arrive above the last DMMAs, right behind the issue of the last LDS, and a producer
            // that refills the stage at once (the producer warpgroup) overwrites data still being read
            // (measured: wrong A fragments in warps 0-2, whose boxes the refill writes first).
            __syncwarp();
            if (lane == 0) mbar_arrive_after(&empty[stage], dep & static_cast<uint32_t>(a.zero));
            ++n_use;
        }
        TM_TRACE_EV(4, ti);
        if constexpr (FIX) {
            if (t.fixup == 2) fold_partials<FM, FN, true, NC>(a, t, acc, wm0, wn0, g, tq);
        }
        TM_TRACE_EV(5, ti);

        const int64_t di = d.oi, dj = d.oj;
        const bool dst_vec = ((reinterpret_cast<uintptr_t>(d.dst) & 15) | (d.ld_dst & 1) | (di & 1)) == 0;
#pragma unroll
        for (int mi = 0; mi < FM; ++mi)
#pragma unroll
            for (int ni = 0; ni < FN; ++ni) {
                const int r = c_row<true>(wm0, mi, tq), c = c_col<true>(wn0, ni, g);
                double* p = d.dst + (di + r) + (dj + c) * d.ld_dst;
                if (dst_vec && r + 1 < t.m && c < t.n) {
                    *reinterpret_cast<double2*>(p) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
                } else {
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        if (r + e < t.m && c < t.n) p[e] = acc[mi][ni][e];
                }
            }
        if (FIX && t.fixup == 1) signal_partial<NC>(a, t);
        else signal_done<NC>(a, t, ti);
        TM_TRACE_EV(6, ti);
    }
    TM_TRACE_EV(7, 0);
}

// ============================== SIMT kernels =============================
// Thread (tx, ty) owns rows ty*TM.., columns tx*TN.. of the CTA tile; each
// entry accumulates one k at a time, in ascending order, only over k that
// exist (no zero-padded steps), so results are bit-reproducible on the CPU.
template <int BM, int BN, int TM, int TN, int STAGES, bool EXACT>
__global__ void __launch_bounds__((BM / TM) * (BN / TN)) k_simt(Args a) {
    constexpr int NTX = BN / TN, NT = (BM / TM) * (BN / TN);
    using G = Geo<BM, BN, true>;
    extern __shared__ __align__(128) double smem[];
    const int tx = threadIdx.x % NTX, ty = threadIdx.x / NTX;
    const int r0 = ty * TM, c0 = tx * TN;

    const int t_lo = a.cta_first ? a.cta_first[blockIdx.x] : static_cast<int>(blockIdx.x);
    const int t_hi = a.cta_first ? a.cta_first[blockIdx.x + 1] : a.ntasks;
    const int t_step = a.cta_first ? 1 : static_cast<int>(gridDim.x);
    for (int ti = t_lo; ti < t_hi; ti += t_step) {
        const Task t = a.tasks[ti];
        wait_ready(a, t);
        wait_turn(a, t);
        const int nk = (t.k + kBK - 1) / kBK;
#pragma unroll
        for (int s = 0; s < STAGES - 1; ++s) {
            if (s < nk) load_slab<BM, BN, NT, false, true>(smem + s * G::STAGE, smem + s * G::STAGE + G::A_ELEMS, a, t,
                                                          t.p0 + s * kBK);
            cp_commit();
        }
        const Dest d = resolve(a, t);
        double acc[TM][TN];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) {
                const int r = r0 + i, c = c0 + j;
                acc[i][j] = (d.src && r < t.m && c < t.n)
                                ? __ldcg(d.src + (t.i0 + r) + static_cast<int64_t>(t.j0 + c) * d.ld_src)
                                : 0.0;
            }

        auto step = [&](const double* As, const double* Bt, int kk) {
            double av[TM], bv[TN];
#pragma unroll
            for (int i = 0; i < TM; ++i) av[i] = As[kk * G::LDA + r0 + i];
#pragma unroll
            for (int j = 0; j < TN; ++j) bv[j] = Bt[kk * G::LDB + c0 + j];
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) {
                    if constexpr (EXACT)
                        acc[i][j] = __dadd_rn(acc[i][j], __dmul_rn(av[i], bv[j]));
                    else
                        acc[i][j] = __fma_rn(av[i], bv[j], acc[i][j]);
                }
        };

        for (int s = 0; s < nk; ++s) {
            cp_wait<STAGES - 2>();
            __syncthreads();
            const int nx = s + STAGES - 1;
            if (nx < nk) {
                double* st = smem + (nx % STAGES) * G::STAGE;
                load_slab<BM, BN, NT, false, true>(st, st + G::A_ELEMS, a, t, t.p0 + nx * kBK);
            }
            cp_commit();
            const double* As = smem + (s % STAGES) * G::STAGE;
            const double* Bt = As + G::A_ELEMS;
            const int kv = min(kBK, t.k - s * kBK);
            if (kv == kBK) {
#pragma unroll
                for (int kk = 0; kk < kBK; ++kk) step(As, Bt, kk);
            } else {
                for (int kk = 0; kk < kv; ++kk) step(As, Bt, kk);
            }
        }
        cp_wait<0>();
        __syncthreads();
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) {
                const int r = r0 + i, c = c0 + j;
                if (r < t.m && c < t.n)
                    d.dst[(d.oi + r) + (d.oj + c) * d.ld_dst] = acc[i][j];
            }
        signal_done(a, t, ti);
    }
}

// Deterministic split-k reduction, one CTA per split tile:
// C(tile) = slot0 + slot1 + ... in slot order.
__global__ void k_reduce_tiles(double* C, int64_t ldc, const double* W, int64_t wld, int64_t wslot,
                               const ReduceTile* tiles) {
    const ReduceTile rt = tiles[blockIdx.x];
    const int64_t total = static_cast<int64_t>(rt.m) * rt.n;
    const double* base = W + static_cast<int64_t>(rt.slot0) * wslot;
    for (int64_t x = threadIdx.x; x < total; x += blockDim.x) {
        const int64_t i = x % rt.m, j = x / rt.m;
        double s = base[i + j * wld];
        for (int q = 1; q < rt.nslots; ++q) s = __dadd_rn(s, base[q * wslot + i + j * wld]);
        C[(rt.i0 + i) + (rt.j0 + j) * ldc] = s;
    }
}

// Counter-based uniform[-1,1): v = 2u - 1, u = top 53 bits of
// splitmix64(seed + (index + 1) * golden). `index` is the element's position
// in the GLOBAL column-major matrix, so any block of a distributed matrix is
// reproducible from (seed, row, col) alone (oracle/oracle.py restates it).
__device__ __forceinline__ double counter_uniform(uint64_t seed, uint64_t index) {
    uint64_t z = seed + (index + 1) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return 2.0 * (static_cast<double>(z >> 11) * 0x1.0p-53) - 1.0;
}

__global__ void k_fill(double* x, int64_t count, uint64_t seed, uint64_t offset) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        x[i] = counter_uniform(seed, offset + static_cast<uint64_t>(i));
}

// x(i, j) (ld) = value of global element (row0 + i, col0 + j) of a matrix
// with global leading dimension gld.
__global__ void k_fill_block(double* x, int64_t rows, int64_t cols, int64_t ld, uint64_t seed, int64_t row0,
                             int64_t col0, int64_t gld) {
    const int64_t total = rows * cols;
    for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < total;
         q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = q % rows, j = q / rows;
        x[i + j * ld] = counter_uniform(seed, static_cast<uint64_t>((row0 + i) + (col0 + j) * gld));
    }
}

// ------------------------------ registry ---------------------------------
constexpr int kStagesBig = 3, kStagesSmall = 4, kStagesSimt = 3;
// 128x64 (two CTAs per SM, short-k tasks): 3 stages of BK=16 measured 84 % of
// peak on the rank-k config vs 75 % with 4 stages (profiles/sweep_r01_fp64.jsonl).
constexpr int kStagesRankK = 3;
constexpr int kBKBig = 32, kBKSmall = 16;

template <int BM, int BN, int BK, int STAGES>
constexpr int dmma_smem() {
    return ((BM + 4) * BK + BN * (BK + 4)) * STAGES * static_cast<int>(sizeof(double));
}

template <int BM, int BN, bool BT, int STAGES>
constexpr int smem_of() {
    return Geo<BM, BN, BT>::STAGE * STAGES * static_cast<int>(sizeof(double));
}

struct Entry {
    const void* fn[2];  // [vec16]
    int tile_m, tile_n, threads, smem;
};

const Entry kTable[kKernelCount] = {
    {{(const void*)k_dmma<128, 128, kBKBig, 32, 32, kStagesBig, false>, (const void*)k_dmma<128, 128, kBKBig, 32, 32, kStagesBig, true>},
     128, 128, 512, dmma_smem<128, 128, kBKBig, kStagesBig>()},
    {{(const void*)k_dmma<64, 64, kBKSmall, 32, 32, kStagesSmall, false>, (const void*)k_dmma<64, 64, kBKSmall, 32, 32, kStagesSmall, true>},
     64, 64, 128, dmma_smem<64, 64, kBKSmall, kStagesSmall>()},
    {{(const void*)k_simt<64, 64, 4, 4, kStagesSimt, false>, (const void*)k_simt<64, 64, 4, 4, kStagesSimt, false>},
     64, 64, 256, smem_of<64, 64, true, kStagesSimt>()},
    {{(const void*)k_simt<64, 64, 4, 4, kStagesSimt, true>, (const void*)k_simt<64, 64, 4, 4, kStagesSimt, true>},
     64, 64, 256, smem_of<64, 64, true, kStagesSimt>()},
    {{(const void*)k_simt<128, 128, 8, 8, kStagesSimt, false>, (const void*)k_simt<128, 128, 8, 8, kStagesSimt, false>},
     128, 128, 256, smem_of<128, 128, true, kStagesSimt>()},
    {{(const void*)k_dmma<128, 64, kBKSmall, 64, 32, kStagesRankK, false, false>, (const void*)k_dmma<128, 64, kBKSmall, 64, 32, kStagesRankK, true, false>},
     128, 64, 128, dmma_smem<128, 64, kBKSmall, kStagesRankK>()},
};

template <int BM, int BN, int BK, int STAGES>
constexpr int tma_smem() {
    return (BM + BN) * BK * STAGES * static_cast<int>(sizeof(double)) + 1024;  // + alignment to the swizzle period
}

// TMA-fed variants of the DMMA kernels (same tiles, k-slab depth and stage
// count as their cp.async counterparts; fn == nullptr: none).
struct TmaEntry {
    const void* fn;
    int bk, box_n, smem;
    int extra_threads = 0;  // a producer warpgroup behind the task-running warps
};
const TmaEntry kTmaTable[kKernelCount] = {
    {(const void*)k_dmma_tma<128, 128, TM_TMA_BK128, 32, 32, TM_TMA_ST128, true, TM_PRODUCER_WARP != 0>, TM_TMA_BK128, 128,
     tma_smem<128, 128, TM_TMA_BK128, TM_TMA_ST128>(), TM_PRODUCER_WARP != 0 ? 128 : 0},
    {(const void*)k_dmma_tma<64, 64, kBKSmall, 32, 32, kStagesSmall>, kBKSmall, 64, tma_smem<64, 64, kBKSmall, kStagesSmall>()},
    {nullptr, 0, 0, 0},
    {nullptr, 0, 0, 0},
    {nullptr, 0, 0, 0},
    {(const void*)k_dmma_tma<128, 64, kBKSmall, 64, 32, kStagesRankK, false>, kBKSmall, 64,
     tma_smem<128, 64, kBKSmall, kStagesRankK>()},
};
int g_tma_occ[kKernelCount];  // 0 = not prepared

KernelInfo g_info[kKernelCount];
bool g_ready[kKernelCount][2];
int g_device = -1;
std::mutex g_mu;  // first-use attribute setup may race between host threads

cudaError_t prepare(Kernel k, bool v16) {
    std::lock_guard<std::mutex> lk(g_mu);
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev != g_device) {
        for (auto& r : g_ready) r[0] = r[1] = false;
        for (int& o : g_tma_occ) o = 0;
        g_device = dev;
    }
    if (g_ready[k][v16]) return cudaSuccess;
    const Entry& en = kTable[k];
    e = cudaFuncSetAttribute(en.fn[v16], cudaFuncAttributeMaxDynamicSharedMemorySize, en.smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, en.fn[v16], en.threads, en.smem);
    if (e != cudaSuccess) return e;
    g_info[k] = KernelInfo{en.tile_m, en.tile_n, en.threads, en.smem, occ};
    g_ready[k][v16] = true;
    return cudaSuccess;
}

}  // namespace

cudaError_t kernel_info(Kernel kernel, KernelInfo* info) {
    cudaError_t e = prepare(kernel, false);
    if (e == cudaSuccess) {
        std::lock_guard<std::mutex> lk(g_mu);
        *info = g_info[kernel];
    }
    return e;
}

cudaError_t launch(Kernel kernel, bool vec16, const Args& args, int grid, cudaStream_t stream) {
    cudaError_t e = prepare(kernel, vec16);
    if (e != cudaSuccess) return e;
    if (args.ntasks <= 0) return cudaSuccess;
    const Entry& en = kTable[kernel];
    Args local = args;
    void* params[] = {&local};
    return cudaLaunchKernel(en.fn[vec16], dim3(grid), dim3(en.threads), params, en.smem, stream);
}

int tma_bk(Kernel kernel) { return kernel >= 0 && kernel < kKernelCount ? kTmaTable[kernel].bk : 0; }

cudaError_t launch_tma(Kernel kernel, const Args& args, int64_t M, int64_t N, int64_t K, int grid,
                       cudaStream_t stream, bool pdl) {
    if (kernel < 0 || kernel >= kKernelCount || kTmaTable[kernel].fn == nullptr) return cudaErrorNotSupported;
    const TmaEntry& en = kTmaTable[kernel];
    if ((args.lda & 1) || (args.ldb & 1) || (reinterpret_cast<uintptr_t>(args.A) & 15) ||
        (reinterpret_cast<uintptr_t>(args.B) & 15))
        return cudaErrorNotSupported;  // TMA: 16-byte aligned bases and strides
    cudaError_t e = prepare(kernel, true);
    if (e != cudaSuccess) return e;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if (g_tma_occ[kernel] == 0) {
            if ((e = cudaFuncSetAttribute(en.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, en.smem)) != cudaSuccess)
                return e;
            int occ = 0;
            if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, en.fn, kTable[kernel].threads + en.extra_threads, en.smem)) !=
                cudaSuccess)
                return e;
            g_tma_occ[kernel] = occ > 0 ? occ : -1;
        }
        // the persistent grid was sized for the cp.async kernel; every CTA must be co-resident
        if (g_tma_occ[kernel] < g_info[kernel].ctas_per_sm) return cudaErrorNotSupported;
    }
    if (args.ntasks <= 0) return cudaSuccess;
    auto* encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tensor_map_encoder());
    if (encode == nullptr) return cudaErrorNotSupported;
    CUtensorMap ma, mb, mc;
    std::memset(&mc, 0, sizeof(mc));
    const cuuint32_t estr[2] = {1, 1};
    {
        const cuuint64_t dims[2] = {static_cast<cuuint64_t>(M), static_cast<cuuint64_t>(K)};
        const cuuint64_t strides[1] = {static_cast<cuuint64_t>(args.lda) * 8};
        const cuuint32_t box[2] = {16, static_cast<cuuint32_t>(en.bk)};
        if (encode(&ma, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(args.A), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    {
        const cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(N)};
        const cuuint64_t strides[1] = {static_cast<cuuint64_t>(args.ldb) * 8};
        const cuuint32_t box[2] = {16, static_cast<cuuint32_t>(en.box_n)};
        if (encode(&mb, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(args.B), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    bool cmap = false;
    if (!(args.ldc & 1) && !(reinterpret_cast<uintptr_t>(args.C) & 15)) {
        const cuuint64_t dims[2] = {static_cast<cuuint64_t>(M), static_cast<cuuint64_t>(N)};
        const cuuint64_t strides[1] = {static_cast<cuuint64_t>(args.ldc) * 8};
        // one box = one C tile (prefetch only, so no swizzle constraint on the inner extent)
        const cuuint32_t box[2] = {static_cast<cuuint32_t>(kTable[kernel].tile_m), static_cast<cuuint32_t>(en.box_n)};
        cmap = encode(&mc, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, args.C, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    Args local = args;
    local.prefetch_c = cmap ? 1 : 0;
    static const int prefetch_knob = [] {  // TILEMUL_TMA_PREFETCH_C=0: A/B knob
        const char* env = std::getenv("TILEMUL_TMA_PREFETCH_C");
        return env ? std::atoi(env) : 1;
    }();
    local.prefetch_c &= prefetch_knob;
    local.pdl_trigger = 1;  // (harmless without a dependent launch)
    if (!pdl) {
        void* params[] = {&local, &ma, &mb, &mc};
        return cudaLaunchKernel(en.fn, dim3(grid), dim3(kTable[kernel].threads + en.extra_threads), params, en.smem, stream);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(static_cast<unsigned>(kTable[kernel].threads + en.extra_threads));
    cfg.dynamicSmemBytes = static_cast<size_t>(en.smem);
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    void* params[] = {&local, &ma, &mb, &mc};
    return cudaLaunchKernelExC(&cfg, en.fn, params);
}

cudaError_t launch_reduce_tiles(double* C, int64_t ldc, const double* work, int64_t work_ld, int64_t work_slice,
                                const ReduceTile* tiles, int ntiles, cudaStream_t stream) {
    if (ntiles <= 0) return cudaSuccess;
    k_reduce_tiles<<<ntiles, 512, 0, stream>>>(C, ldc, work, work_ld, work_slice, tiles);
    return cudaGetLastError();
}

cudaError_t launch_fill_block(double* x, int64_t rows, int64_t cols, int64_t ld, uint64_t seed, int64_t row0,
                              int64_t col0, int64_t gld, cudaStream_t stream) {
    if (rows <= 0 || cols <= 0) return cudaSuccess;
    int blocks = static_cast<int>(std::min<int64_t>((rows * cols + 255) / 256, 148 * 32));
    k_fill_block<<<blocks, 256, 0, stream>>>(x, rows, cols, ld, seed, row0, col0, gld);
    return cudaGetLastError();
}

cudaError_t launch_fill(double* x, int64_t count, uint64_t seed, uint64_t offset, cudaStream_t stream) {
    if (count <= 0) return cudaSuccess;
    int blocks = static_cast<int>(std::min<int64_t>((count + 255) / 256, 148 * 32));
    k_fill<<<blocks, 256, 0, stream>>>(x, count, seed, offset);
    return cudaGetLastError();
}

}  // namespace gpu
}  // namespace mmm

#ifdef TM_TRACE
// Experiment builds only: copy the per-CTA timeline out and reset it.
// out: ctas x events x 3 u64 (globaltimer ns, clock64, event | task << 8); counts: events per CTA.
extern "C" __attribute__((visibility("default"))) int tm_trace_read(unsigned long long* out, int* counts) {
    using namespace mmm::gpu;
    if (cudaDeviceSynchronize() != cudaSuccess) return 3;
    if (cudaMemcpyFromSymbol(out, g_trace, sizeof(unsigned long long) * kTraceCtas * kTraceEv * 3) != cudaSuccess)
        return 3;
    if (cudaMemcpyFromSymbol(counts, g_trace_n, sizeof(int) * kTraceCtas) != cudaSuccess) return 3;
    static int zero[kTraceCtas] = {};
    return cudaMemcpyToSymbol(g_trace_n, zero, sizeof(zero)) == cudaSuccess ? 0 : 3;
}
extern "C" __attribute__((visibility("default"))) int tm_trace_dims(int* ctas, int* events) {
    *ctas = mmm::gpu::kTraceCtas;
    *events = mmm::gpu::kTraceEv;
    return 0;
}
#endif
