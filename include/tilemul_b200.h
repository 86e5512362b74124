/*
 * tilemul_b200 — C ABI of the B200-native MOMMS GEMM (C += A·B, FP64,
 * column-major), a drop-in for the reference toolkit's execution path.
 *
 * Every entry point replaces one reference interface, cited as
 * /root/reference/proj/<file>:<line>. Plain pointers and sizes only; device
 * pointers are CUDA global-memory addresses, `stream` is a cudaStream_t
 * (NULL = legacy default stream).
 *
 * Status codes (the reference CLI's exit codes, tools/tilemul_main.cpp:519-535,
 * extended): 0 ok; 1 a family/blocksize rule is broken (ParseError,
 * ValidationFailure, InfeasibleError — tm_last_rules() lists the rule ids);
 * 2 usage/config error (std::invalid_argument, ConfigError); 3 CUDA runtime
 * error. The error text of the calling thread is in tm_last_error().
 */
#ifndef TILEMUL_B200_H
#define TILEMUL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One memory level; replaces tilemul::CacheLevel (include/tilemul/cache.hpp:12-19).
 * Capacity in elements of the operand type (FP64 = 8 bytes). */
typedef struct {
    int64_t capacity_elements;
    int64_t granularity;
    int32_t inclusive;
    int32_t write_allocate;
    int32_t write_back;
} tm_level;

/* One blocksize entry; replaces BlocksizeSet::set(level, dim, value)
 * (include/tilemul/blocksizes.hpp:30-33). dim is 'm', 'n' or 'k'. */
typedef struct {
    int32_t level;
    char dim;
    int64_t value;
} tm_blocksize;

/* One partition loop of the nest, outermost first; replaces NestStep
 * (include/tilemul/blocksizes.hpp:428-434). */
typedef struct {
    int32_t level;
    char dim;
    int64_t blocksize;
    int32_t cap;
} tm_loop;

/* One planned level of a family member; replaces LevelPlan
 * (include/tilemul/descriptor.hpp:18-25). */
typedef struct {
    int32_t level;
    char resident; /* 'A' 'B' 'C' */
    char outer_dim;
    char inner_dim;
} tm_tier;

/* Derivation knobs; replaces AccessCosts + DeriveOptions + MicroTile
 * (include/tilemul/blocksizes.hpp:59-87). */
typedef struct {
    double slack;   /* default 1/16 */
    int64_t m_r;    /* register tile (the CTA's C tile on the GPU) */
    int64_t n_r;
    double beta_a, beta_b, beta_c;
} tm_derive_opts;

/* Kernel numerics. All accumulate every C entry in ascending k from C's
 * incoming value (the reference's cell semantics, exec.hpp:35-46). */
enum {
    TM_NUMERICS_DMMA = 0,  /* FP64 tensor pipe, mma.sync m8n8k4 (SASS DMMA.8x8x4) */
    TM_NUMERICS_FMA = 1,   /* DFMA chain, one rounding per step: bit-exact vs a sequential fma oracle */
    TM_NUMERICS_EXACT = 2  /* DMUL then DADD, two roundings: bit-exact vs the reference's execute() */
};
/* How the nest's cells map onto CTA tasks. */
enum {
    TM_SCHEDULE_FUSED = 0,    /* k loops sunk below the tile loops: one task per C tile, C in registers */
    TM_SCHEDULE_FAITHFUL = 1  /* one task per nest cell in nest order; C round-trips per cell */
};

/* Replaces tilemul::ExecOptions (include/tilemul/exec.hpp:48-53). */
typedef struct {
    int32_t numerics;   /* TM_NUMERICS_* */
    int32_t schedule;   /* TM_SCHEDULE_* */
    int32_t split_k;    /* fused schedule: k parts per tile, deterministic reduction. 1 = none; n > 1 = every
                           tile; 0 = auto (DMMA numerics only): all tiles when C is too small to fill the
                           GPU, else only the tiles of the last partial wave */
    int32_t ctas;       /* persistent grid size (0 = SMs x occupancy) */
    int32_t tile;       /* CTA tile rows: 128 or 64 (0 = auto from the register tile); tensor-core path:
                           128 = one SM (cta_group::1), 0/256 = an SM pair (cta_group::2) */
    int32_t tile_n;     /* CTA tile columns (0 = same as tile); 128 x 64 runs two CTAs per SM; tensor-core
                           SM pairs: 512 (the default, 0) or 256 */
    /* Faithful schedule: the m/n loop whose iterations run as independent
     * workers (ExecOptions::parallel_loop, exec.hpp:50-53, :125-131), as
     * loop index + 1; 0 = plain nest order (consecutive cells on the CTAs,
     * the member's own traffic). A k loop is rejected (status 2), like the
     * reference. */
    int32_t parallel_loop;
    /* DMMA kernels: how the SMEM level is filled. TM_STAGING_AUTO picks TMA
     * for the 128x128 kernel when it applies (16-byte aligned A/B, leading
     * dimensions and task origins; every task's k range a whole number of
     * slabs or ending at k), launching a long task list in segments of whole
     * rounds of at most 4096 k-slabs per CTA; else cp.async. Bitwise equal. */
    int32_t staging;
} tm_exec_opts;
enum { TM_STAGING_AUTO = 0, TM_STAGING_CPASYNC = 1, TM_STAGING_TMA = 2 };

typedef struct tm_plan tm_plan;

/* --- errors ------------------------------------------------------------ */
const char* tm_last_error(void);
/* Rule ids of the last failure, one per line "rule:level:lhs:rhs". */
const char* tm_last_rules(void);
const char* tm_version(void);
/* sha256[:16] of all the sources this library was built from (build.py
 * source_hash); the Python loader refuses a library built from other sources. */
const char* tm_build_id(void);
/* sha256[:16] of the sources that decide the device work (kernels, lowering,
 * host pipeline: build.py kernel_hash). ncu summaries under profiles/ carry
 * the kernel id they measured; bench.py uses their bytes only on a match. */
const char* tm_kernel_id(void);

/* --- family descriptors (include/tilemul/descriptor.hpp) ---------------- */
/* parse_name (:111-125): fills up to `cap` tiers, sets *count. */
int tm_parse_name(const char* name, int allow_non_c_registers, tm_tier* tiers, int cap, int* count);
/* make_descriptor (:68-107) from (level, resident) pairs, then format_name (:128-136). */
int tm_compose(const int32_t* levels, const char* residents, int count, int allow_non_c_registers, char* name_out,
               int name_cap, tm_tier* tiers, int cap, int* tier_count);
/* validate_structure (:140-173) of an explicit tier list; returns #issues, rules in tm_last_rules(). */
int tm_validate_structure(const tm_tier* tiers, int count, int allow_non_c_registers);
/* skip_level (:177-195). */
int tm_skip_level(const char* name, int level, char* name_out, int name_cap);
/* select_algorithm (:206-218): writes 'A', 'B' or 'C'. */
int tm_select_outer(int64_t m, int64_t n, int64_t k, int64_t outer_capacity, char* resident);

/* --- blocksizes (include/tilemul/blocksizes.hpp) ------------------------- */
/* derive_blocksizes (:243-425). Writes up to `cap` entries in (level, dim) order. */
int tm_derive(const char* name, const tm_level* levels, int nlevels, int64_t m, int64_t n, int64_t k,
              const tm_derive_opts* opts, const tm_blocksize* pinned, int npinned, tm_blocksize* out, int cap,
              int* count);
/* validate_blocksizes (:125-235): returns the number of violated rules (>= 0) or -status. */
int tm_validate(const char* name, const tm_level* levels, int nlevels, int64_t m, int64_t n, int64_t k,
                const tm_blocksize* bs, int nbs);
/* The B200 memory hierarchy of the current device in FP64 elements:
 * level 0 = CTA C tile (tile x tile), 1 = shared memory per block (opt-in),
 * 2 = L2. Queried from the device; fails with 3 when no GPU is present. */
int tm_gpu_hierarchy(int tile, tm_level* levels, int cap, int* count);

/* --- plans (include/tilemul/plan.hpp) ----------------------------------- */
/* build_plan (:90-108): validates and builds the nest; register level must be C. */
int tm_plan_create(const char* name, const tm_level* levels, int nlevels, int64_t m, int64_t n, int64_t k,
                   const tm_blocksize* bs, int nbs, tm_plan** plan);
/* A plan straight from an executable LoopNest (plan.hpp:25-31: loops in
 * nest order, m_r, n_r, shape), for callers that hold a nest but not the
 * hierarchy it was validated against -- the reference's execute(nest, A, B,
 * C, opts) (exec.hpp:94-95) takes exactly that. `name` (optional) records the
 * family member. Checks what execute relies on: extents >= 1, blocksizes
 * >= 1, cells no larger than the m_r x n_r register tile (exec.hpp:107).
 * Such a plan executes like any other; it has no I/O model (no hierarchy). */
int tm_plan_create_loops(const char* name, const tm_loop* loops, int nloops, int64_t m_r, int64_t n_r, int64_t m,
                         int64_t n, int64_t k, tm_plan** plan);
void tm_plan_destroy(tm_plan* plan);
int tm_plan_loops(const tm_plan* plan, tm_loop* loops, int cap, int* count);
int64_t tm_plan_cells(const tm_plan* plan);

/* --- the I/O model (include/tilemul/costmodel.hpp) ----------------------- */
/* multilevel_cost (:163-229): out[(h*3 + operand)*2 + {0 reads, 1 writes}], operands A,B,C. */
int tm_plan_model(const tm_plan* plan, int64_t* out, int cap);
/* multilevel_cost for any validated family member (no executable plan needed). */
int tm_model(const char* name, int allow_non_c_registers, const tm_level* levels, int nlevels, int64_t m, int64_t n,
             int64_t k, const tm_blocksize* bs, int nbs, int64_t* out, int cap);
/* GPU-mode I/O model of the schedule tm_execute would run with `opts` on a
 * device with `sms` SMs and an L2 of `l2_bytes` (no GPU needed; gpu_model.cpp):
 *   out[0..5]   elements into the SMEM level (L2 <-> SM), (reads, writes) for
 *               A, B, C -- exact over the task list (FIFO staging: a task
 *               streams m_t k_t of A and k_t n_t of B; C once in and out,
 *               plus split-k partials);
 *   out[6..11]  bytes across the HBM boundary, (read, written) for A, B, C,
 *               from a lockstep run of the task list (one k-slab per CTA per
 *               step, strided rounds or stream-K ranges as the kernel takes
 *               them) through a write-back LRU of l2_bytes at slab granularity;
 *   out[12..17] tasks, grid, lockstep steps, kernel id, tile_m, tile_n.
 * elem_bytes: bytes per element of A, B, C (NULL = 8, 8, 8). Extends the
 * reference's multilevel_cost (costmodel.hpp:163-229), which assumes a
 * resident block per level and 8-byte elements. */
int tm_plan_gpu_model(const tm_plan* plan, const tm_exec_opts* opts, int sms, int64_t l2_bytes,
                      const double* elem_bytes, int64_t* out, int cap);
/* The same model for the tcgen05 path tm_execute_tc runs (dtype TM_DTYPE_BF16 / TM_DTYPE_TF32; the
 * opts' tile / tile_n pick the kernel as there): 2- or 4-byte inputs, fp32 C, SM-pair tiles one per
 * cluster with sms / 2 clusters in flight. Same 18-entry output. */
int tm_plan_gpu_model_tc(const tm_plan* plan, int dtype, const tm_exec_opts* opts, int sms, int64_t l2_bytes,
                         int64_t* out, int cap);
/* The task list behind the model: 10 int32 per task (i0, j0, p0, m, n, k,
 * slice, from_c, fixup, seq), the grid, and for stream-K the per-CTA task
 * ranges (cta_first[0] = -1 when CTA c runs tasks c, c + grid, ...). */
int tm_plan_tasks(const tm_plan* plan, const tm_exec_opts* opts, int sms, int32_t* tasks, int64_t cap,
                  int64_t* count, int32_t* grid, int32_t* cta_first, int first_cap);
/* Number of levels of the hierarchy the plan was validated against. */
int tm_plan_levels(const tm_plan* plan);
/* io_lower_bound (:67-76). */
int tm_io_lower_bound(int64_t m, int64_t n, int64_t k, int64_t fast_capacity, int64_t* reads, int64_t* writes);
/* resident_cost (:85-100): out[operand*2 + {0,1}]. */
int tm_resident_cost(char variant, int64_t m, int64_t n, int64_t k, int64_t b1, int64_t b2, int64_t* out);
double tm_streaming_efficiency(char variant, int64_t b1, int64_t b2); /* :252-263 */
double tm_goto_efficiency(int64_t k_c, int64_t n_c);                  /* :267-270 */
double tm_roofline_bound(double intensity, double peak, double bandwidth); /* :278-284 */

/* --- execution (include/tilemul/exec.hpp) ------------------------------ */
/* execute (:94-138) on DEVICE buffers, asynchronous on `stream`:
 * C(m x n, ldc) += A(m x k, lda) · B(k x n, ldb), column-major FP64. */
int tm_execute(tm_plan* plan, const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
               const tm_exec_opts* opts, void* stream);
/* execute on HOST buffers (the reference's own calling convention): copies
 * A, B, C to the device, runs, copies C back; synchronous. Host memory may be
 * pinned (fast path) or pageable. */
int tm_execute_host(tm_plan* plan, const double* A, const double* B, double* C, const tm_exec_opts* opts);
/* The upload order tm_execute_host's copy-engine-fed pipeline uses for the plan's
 * extents (host logic only, no device call): records of 6 int64, in issue
 * order -- {1|2|3 = a piece of A|B|C, r0, rows, c0, cols, 0} for every upload,
 * then {0, i0, i1, j0, j1, q} = the data flag written after them and the cell
 * box (rows [i0,i1) x columns [j0,j1) of k-chunk q) whose tasks wait for it.
 * *count = records in total (call with records = NULL to size the buffer).
 * Pipelines apply when k >= 4096 or n >= 4096 (fused, unsplit). */
int tm_host_pipe_steps(const tm_plan* plan, int64_t* records, int64_t cap, int64_t* count);
/* Mixed precision on the 5th-generation tensor cores (tcgen05 + TMEM,
 * BASELINE configs[3]): C(m x n, fp32) += A·B with A, B column-major in BF16
 * (dtype TM_DTYPE_BF16) or in fp32 holding TF32 values (TM_DTYPE_TF32),
 * fp32 accumulation. Fused schedule only; bases and leading dimensions must
 * be 16-byte aligned (TMA). opts->tile = 128: one SM per 128 x 256 tile;
 * 0 / 256: SM pairs, 256 x 512 tiles (tile_n 0 / 512, the default) or
 * 256 x 256 (tile_n = 256). Plan the nest with a register tile of the same
 * shape so every task fills its tile. */
enum { TM_DTYPE_BF16 = 1, TM_DTYPE_TF32 = 2 };
int tm_execute_tc(tm_plan* plan, int dtype, const void* A, int64_t lda, const void* B, int64_t ldb, float* C,
                  int64_t ldc, const tm_exec_opts* opts, void* stream);
/* Device rounding of FP64 inputs: to BF16 (RNE; y is uint16 storage) or to
 * TF32 values in fp32 storage (RNE to 11 significant bits). */
int tm_round_inputs(int dtype, const double* x, void* y, int64_t count, void* stream);
/* --- prepacked ("hierarchical") operand layouts (layout.hpp:17-145, plan.hpp:113-124) --- */
/* BlockLayout::element_address for a cut chain (on_rows[s], sizes[s]), outermost first. */
int tm_layout_address(int64_t rows, int64_t cols, const int32_t* on_rows, const int64_t* sizes, int ncuts, int64_t i,
                      int64_t j, int64_t* address);
/* layout_for(nest, operand): the plan's hierarchical layout of 'A', 'B' or 'C'. */
int tm_plan_layout(const tm_plan* plan, char operand, int32_t* on_rows, int64_t* sizes, int cap, int* ncuts);
/* pack / unpack on the device (column-major <-> the plan's layout of the operand). */
int tm_pack(const tm_plan* plan, char operand, const double* colmajor, double* packed, void* stream);
int tm_unpack(const tm_plan* plan, char operand, const double* packed, double* colmajor, void* stream);
/* execute() on device buffers prepacked in the plan's layouts (exec.hpp:94-138 with
 * blocked MatrixBuffers): relaid to column-major scratch, executed, C packed back. */
int tm_execute_packed(tm_plan* plan, const double* A, const double* B, double* C, const tm_exec_opts* opts,
                      void* stream);
/* Number of CTA tasks and kernel launches the last tm_execute issued. */
int tm_plan_last_launch(const tm_plan* plan, int64_t* tasks, int32_t* launches, int32_t* ctas);
/* Staging the last task-kernel launch used: TM_STAGING_CPASYNC or TM_STAGING_TMA
 * (0 for the SIMT and tensor-core kernels, which have one staging each). */
int tm_plan_last_staging(const tm_plan* plan, int32_t* staging);

/* Sustained FP64 tensor-pipe (DMMA) rate of the current device in TFLOP/s,
 * from `launches` ~7 ms probe launches: the roofline denominator. */
int tm_measure_fp64_peak(int launches, double* tflops);
/* Peak tcgen05 MMA rate (M=128 x N=256, fp32 accumulate) for dtype
 * TM_DTYPE_BF16 or TM_DTYPE_TF32, best of `launches` launches of ~5 ms
 * (sustained = 0: full clocks) or ~200 ms (sustained != 0: under the power
 * cap, like a long GEMM): the measured roofline denominator of the
 * tensor-core path. */
int tm_measure_tc_peak(int dtype, int launches, int sustained, double* tflops);

/* The reference `run` command's inputs on the host (tools/tilemul_main.cpp:236-242):
 * mt19937_64(seed), uniform(-1,1), filling A, then B, then C (C may be NULL). */
int tm_fill_seeded(uint64_t seed, double* a, int64_t na, double* b, int64_t nb, double* c, int64_t nc);

/* --- seeded device inputs ------------------------------------------------ */
/* Counter-based uniform[-1,1) generator on the device (for operands too large
 * to produce on the host): v = 2u - 1 with u from splitmix64(seed, index). */
int tm_fill_uniform_device(double* x, int64_t count, uint64_t seed, uint64_t offset, void* stream);
/* Block (row0.., col0..) of a global column-major matrix (leading dimension
 * global_ld) filled with the same counter-based values, stored at x with
 * leading dimension ld: every rank can generate its own block. */
int tm_fill_uniform_block(double* x, int64_t rows, int64_t cols, int64_t ld, uint64_t seed, int64_t row0,
                          int64_t col0, int64_t global_ld, void* stream);

/* --- trace-driven model check (include/tilemul/trace.hpp, cachesim.hpp) --- */
/* Counts of one simulated level; replaces SimLevelStats (cachesim.hpp:18-38).
 * Operand arrays are indexed A, B, C. */
typedef struct {
    int32_t level;
    int64_t capacity_lines, granularity;
    int64_t hits, read_misses, write_misses;
    int64_t fetched_lines, passthrough_writes, writebacks;
    int64_t per_operand_misses[3], per_operand_writebacks[3];
} tm_sim_level;
typedef struct tm_sim tm_sim;

/* trace_event_count (trace.hpp:73-79): 2mn + k(m+n) events per cell. */
int64_t tm_trace_event_count(const tm_plan* plan);
/* generate_trace (trace.hpp:51-71): the first `cap` events of the plan's
 * element-access stream, operand letter / flat index / 1 = write; packed != 0
 * addresses operands in the plan's prepacked layouts (TraceLayouts::packed),
 * else column-major. *count = the full stream length. */
int tm_trace(const tm_plan* plan, int packed, int64_t cap, char* ops, int64_t* indices, uint8_t* writes,
             int64_t* count);
/* LruSimulator (cachesim.hpp:61-96): fully associative LRU per level over the
 * address space of an m x n x k problem (A, then B, then C); level 0 is only
 * simulated when include_registers != 0. Fails with 2 when the address space
 * exceeds 2^31 elements (the reference's limit, :71-72). */
int tm_sim_create(const tm_level* levels, int nlevels, int64_t m, int64_t n, int64_t k, int include_registers,
                  int flush_dirty_at_end, tm_sim** sim);
void tm_sim_destroy(tm_sim* sim);
/* LruSimulator::access (:98-160) for `count` events (ops 'A'/'B'/'C'; writes may be NULL = all reads). */
int tm_sim_access(tm_sim* sim, const char* ops, const int64_t* indices, const uint8_t* writes, int64_t count);
/* simulate (:356-362) without the buffer round-trip: replays the plan's trace into sim. */
int tm_sim_replay(tm_sim* sim, const tm_plan* plan, int packed);
/* LruSimulator::finish (:162-169): flushes dirty lines when configured; levels innermost first. */
int tm_sim_finish(tm_sim* sim, tm_sim_level* out, int cap, int* count, int64_t* events);
/* Lines resident at one simulated level (position innermost first), in slot order (:174-182). */
int tm_sim_resident_lines(const tm_sim* sim, int position, int64_t* lines, int cap, int* count);

/* --- multi-GPU exchange (no reference counterpart: the
 * reference is single-node shared memory, exec.hpp:121-137) -------------- */
/* Export the CUDA IPC handle (64 bytes into `handle`) of the device
 * allocation holding `ptr`, and ptr's byte offset inside it. */
int tm_ipc_export(const void* ptr, void* handle, int64_t* offset);
/* Map a peer process's allocation on the CURRENT device (lazy peer access);
 * *ptr = its base + offset. */
int tm_ipc_open(const void* handle, int64_t offset, void** ptr);
int tm_ipc_close(void* ptr, int64_t offset);
/* Device-to-device copy on `stream` by the copy engines (peer memory over
 * NVLink when src is a mapped peer allocation). */
int tm_copy_async(void* dst, const void* src, int64_t bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TILEMUL_B200_H */
