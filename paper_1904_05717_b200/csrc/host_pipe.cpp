// Host-buffer execution (tm_execute_host): copies in, the GEMM, C back,
// pipelined. Preferred: one persistent launch over every (A row block, C
// column block, k-chunk) cell, fed by the copy engine through stream memory
// operations; fallback: one launch per (column block, k-chunk) unit.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include <cuda.h>

#include "engine.hpp"

namespace mmm {
namespace engine {

namespace {

using StreamValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
struct MemOps {
    StreamValueFn write = nullptr, wait = nullptr;
};
// cuStreamWriteValue32 / cuStreamWaitValue32 through the runtime's driver
// entry point (the library links the static runtime, not libcuda); null
// when the driver does not provide them.
const MemOps& memops() {
    static const MemOps m = [] {
        MemOps r;
        void* fw = nullptr;
        void* fv = nullptr;
        cudaDriverEntryPointQueryResult qw{}, qv{};
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fw, cudaEnableDefault, &qw) == cudaSuccess &&
            qw == cudaDriverEntryPointSuccess &&
            cudaGetDriverEntryPoint("cuStreamWaitValue32", &fv, cudaEnableDefault, &qv) == cudaSuccess &&
            qv == cudaDriverEntryPointSuccess) {
            r.write = reinterpret_cast<StreamValueFn>(fw);
            r.wait = reinterpret_cast<StreamValueFn>(fv);
        }
        return r;
    }();
    return m;
}

// The persistent pipeline's tasks wait on flags written by another stream's
// copies: that needs the kernel and the copies to run concurrently, which
// CUDA_LAUNCH_BLOCKING=1 (the launch returns only when the kernel is done)
// and injected tools that serialize GPU work (Nsight Compute, sanitizers:
// CUDA_INJECTION64_PATH) rule out. Those get the one-launch-per-unit path.
bool serialized_launches() {
    const char* lb = std::getenv("CUDA_LAUNCH_BLOCKING");
    return (lb != nullptr && std::atoi(lb) != 0) || std::getenv("CUDA_INJECTION64_PATH") != nullptr;
}

void cu_check(CUresult r, const char* what) {
    if (r != CUDA_SUCCESS) throw Failure(kDevice, "", std::string(what) + ": CUresult " + std::to_string(static_cast<int>(r)));
}

// Cut points of [0, total) into `pieces` equal pieces, aligned.
std::vector<i64> even_cuts(i64 total, int pieces, i64 align) {
    const i64 each = cdiv(cdiv(total, std::max(1, pieces)), align) * align;
    std::vector<i64> start{0};
    while (start.back() < total) start.push_back(std::min(total, start.back() + each));
    return start;
}

// The upload order is a growing box over (A row blocks, C column blocks,
// k-chunks): after the first block of each, the next extension is whichever
// of a new A row block, a new C column block or a new k-chunk enables the
// most GEMM work per element copied, and every piece of an extension is one
// step with its own data flag. Each step's sub-nest is lowered (fused,
// unsplit) and the task lists are spliced into one, in step order, with
// global coordinates; a task waits for its step's flag and for the previous
// chunk of its C tile (progress counters, as in the faithful schedule), so
// every C entry still sees its k chunks in ascending order. Cutting A into
// row blocks (round 2) lets the first GEMM start after ~100 MB instead of a
// whole 512 MB k-chunk of A at 16384^3.
}  // namespace

void pipe_order(const Extents& e, HostPipe& P) {
    // k-chunks of >= 4096 (at most 4) and column blocks of >= 256 (at most
    // 64): at 16384^3 on PCIe Gen5 these measured best among 4..16 chunks x
    // 8..64 blocks (tools/e2e_probe.py); smaller k-chunks cost more C round
    // trips. Row blocks of A of >= 2048 (at most 8; TILEMUL_PIPE_ROWBLOCKS: A/B knob): 16 KB runs per
    // column in their 2-D copies.
    static const int row_knob = [] {
        const char* env = std::getenv("TILEMUL_PIPE_ROWBLOCKS");
        return env ? std::max(1, std::atoi(env)) : 8;
    }();
    // (a small C, < 64 MB, costs nothing to revisit, and its few tiles make a chunk's tasks long: up to 32 chunks
    // there, so the work left after the last upload is one short chunk -- 512^2 x 131072: 23.9 -> 20.x ms)
    const i64 max_chunks = e.m * e.n * 8 < (i64{64} << 20) ? 32 : 4;
    P.kcut = even_cuts(e.k, static_cast<int>(std::max<i64>(1, std::min<i64>(max_chunks, e.k / 4096))), 32);
    P.ncut = even_cuts(e.n, static_cast<int>(std::max<i64>(1, std::min<i64>(64, e.n / 256))), 128);
    static const i64 row_min = [] {  // (TILEMUL_PIPE_ROWMIN: A/B knob; 512 measured +-2 % on 2048^3..4096^3)
        const char* env = std::getenv("TILEMUL_PIPE_ROWMIN");
        return env ? std::max<i64>(128, std::atoll(env)) : i64{2048};
    }();
    P.mcut = even_cuts(e.m, static_cast<int>(std::max<i64>(1, std::min<i64>(row_knob, e.m / row_min))), 128);
    P.steps.clear();
    const auto& mc = P.mcut;
    const auto& nc = P.ncut;
    const auto& kc = P.kcut;
    const int NI = static_cast<int>(mc.size()) - 1, NJ = static_cast<int>(nc.size()) - 1,
              NQ = static_cast<int>(kc.size()) - 1;
    auto at = [](const std::vector<i64>& v, int x) { return v[static_cast<std::size_t>(x)]; };
    auto a_piece = [&](int i, int q) {
        return HostPipe::Piece{'A', at(mc, i), at(mc, i + 1) - at(mc, i), at(kc, q), at(kc, q + 1) - at(kc, q)};
    };
    auto b_piece = [&](int q, i64 j0, i64 j1) {
        return HostPipe::Piece{'B', at(kc, q), at(kc, q + 1) - at(kc, q), j0, j1 - j0};
    };
    auto c_piece = [&](int j) { return HostPipe::Piece{'C', 0, e.m, at(nc, j), at(nc, j + 1) - at(nc, j)}; };
    auto step = [&](std::vector<HostPipe::Piece> pieces, i64 i0, i64 i1, i64 j0, i64 j1, int q) {
        HostPipe::Step s;
        s.pieces = std::move(pieces);
        s.i0 = i0, s.i1 = i1, s.j0 = j0, s.j1 = j1, s.q = q;
        P.steps.push_back(std::move(s));
    };
    step({c_piece(0), a_piece(0, 0), b_piece(0, nc[0], nc[1])}, mc[0], mc[1], nc[0], nc[1], 0);
    int ni = 1, nj = 1, nq = 1;
    while (ni < NI || nj < NJ || nq < NQ) {
        const double Mi = static_cast<double>(at(mc, ni)), Nj = static_cast<double>(at(nc, nj)),
                     Kq = static_cast<double>(at(kc, nq)), M = static_cast<double>(e.m);
        // GEMM work enabled per element copied. A C column block is copied whole (all M rows, contiguous):
        // cutting C into row blocks too would enable work sooner per byte, but measured worse (16384^3:
        // 262.4 ms against 259.2 with 2048-row blocks, 280.2 with 1024-row blocks;
        // profiles/ab_r02_pipe_rowblocks.json).
        const double ri = ni < NI ? Nj : -1.0;
        const double rj = nj < NJ ? Mi * Kq / (M + Kq) : -1.0;
        const double rq = nq < NQ ? Mi * Nj / (Mi + Nj) : -1.0;
        if (ri > rj && ri > rq) {  // a new row block of A, chunk by chunk
            for (int q = 0; q < nq; ++q) step({a_piece(ni, q)}, at(mc, ni), at(mc, ni + 1), nc[0], at(nc, nj), q);
            ++ni;
        } else if (rq > rj) {  // a new k-chunk: its B rows for the loaded columns, then A row block by row block
            for (int i = 0; i < ni; ++i) {
                std::vector<HostPipe::Piece> pcs;
                if (i == 0) pcs.push_back(b_piece(nq, nc[0], at(nc, nj)));
                pcs.push_back(a_piece(i, nq));
                step(std::move(pcs), at(mc, i), at(mc, i + 1), nc[0], at(nc, nj), nq);
            }
            ++nq;
        } else {  // a new C column block with its B columns, chunk by chunk
            for (int q = 0; q < nq; ++q) {
                std::vector<HostPipe::Piece> pcs;
                if (q == 0) pcs.push_back(c_piece(nj));
                pcs.push_back(b_piece(q, at(nc, nj), at(nc, nj + 1)));
                step(std::move(pcs), mc[0], at(mc, ni), at(nc, nj), at(nc, nj + 1), q);
            }
            ++nj;
        }
    }
}

namespace {

std::unique_ptr<HostPipe> build_pipe(const tm_plan& plan, const tm_exec_opts& o, cudaStream_t st) {
    const Extents& e = plan.nest.ext;
    auto P = std::make_unique<HostPipe>();
    P->opts = o;
    pipe_order(e, *P);
    const auto& nc = P->ncut;
    const auto& kc = P->kcut;
    const auto& mc = P->mcut;
    const int NI = static_cast<int>(mc.size()) - 1, NJ = static_cast<int>(nc.size()) - 1,
              NQ = static_cast<int>(kc.size()) - 1;
    tm_exec_opts uo = o;
    uo.split_k = 1;
    Nest first = plan.nest;
    first.ext.m = P->mcut[1];
    first.ext.n = nc[1];
    first.ext.k = kc[1];
    const gpu::Kernel kernel = pick_kernel(first, uo, uo.staging != TM_STAGING_CPASYNC && e.m % 2 == 0 && e.k % 2 == 0);
    gpu::KernelInfo info{};
    cuda_check(gpu::kernel_info(kernel, &info), "kernel_info");
    const i64 mt = cdiv(e.m, info.tile_m);
    P->regions = static_cast<int>(mt * cdiv(e.n, info.tile_n));
    // Downloads: whole column blocks (contiguous), unless C has too few of them to overlap anything -- a tall C
    // (65536 x 256) goes back row block by row block. (Cutting every column block into row cells costs the
    // C-dominated shapes: rank-k 16384^2 x 256 50.3 -> 57.1 ms, 16384^3 only 254.8 -> 254.4.)
    P->done_rows = NJ < 8 ? NI : 1;
    const int ND = P->done_rows;
    P->block_tasks.assign(static_cast<std::size_t>(NJ) * static_cast<std::size_t>(ND), 0);
    auto sched = std::make_unique<Schedule>();
    sched->kernel = kernel;
    auto& T = sched->host_tasks;
    for (std::size_t u = 0; u < P->steps.size(); ++u) {
        const HostPipe::Step& sp = P->steps[u];
        Nest sn = plan.nest;
        sn.ext.m = sp.i1 - sp.i0;
        sn.ext.n = sp.j1 - sp.j0;
        sn.ext.k = kc[static_cast<std::size_t>(sp.q) + 1] - kc[static_cast<std::size_t>(sp.q)];
        const auto part = lower(sn, uo, kernel, st, false);
        for (gpu::Task tk : part->host_tasks) {
            tk.i0 += static_cast<int32_t>(sp.i0);
            tk.j0 += static_cast<int32_t>(sp.j0);
            tk.p0 += static_cast<int32_t>(kc[static_cast<std::size_t>(sp.q)]);
            tk.tile = static_cast<int32_t>(tk.i0 / info.tile_m + (tk.j0 / info.tile_n) * mt);
            tk.seq = sp.q;
            tk.ready = static_cast<int32_t>(u) + 1;
            // its C cell: tiles never straddle a cut (cuts are multiples of 128, tiles 64 or 128 wide)
            const int b = static_cast<int>(std::upper_bound(nc.begin(), nc.end(), static_cast<i64>(tk.j0)) - nc.begin()) - 1;
            const int i = ND == 1 ? 0 : static_cast<int>(std::upper_bound(mc.begin(), mc.end(), static_cast<i64>(tk.i0)) - mc.begin()) - 1;
            const int cell = b * ND + i;
            tk.done = sp.q == NQ - 1 ? cell + 1 : 0;
            if (sp.q == NQ - 1) ++P->block_tasks[static_cast<std::size_t>(cell)];
            T.push_back(tk);
        }
        if (sp.q == NQ - 1)  // the cells this step finishes, in the order they go back to the host
            for (int b = 0; b < NJ; ++b)
                for (int i = 0; i < ND; ++i)
                    if (nc[static_cast<std::size_t>(b)] >= sp.j0 && nc[static_cast<std::size_t>(b)] < sp.j1 &&
                        (ND == 1 ? sp.i1 == e.m  // (a column block is done with the step that brings its last rows)
                                 : mc[static_cast<std::size_t>(i)] >= sp.i0 && mc[static_cast<std::size_t>(i)] < sp.i1))
                        P->cells.push_back({b, i});
    }
    if (T.size() > static_cast<std::size_t>(INT32_MAX)) fail_usage("too many tasks");
    sched->grid = std::max(1, std::min<int>(sm_count() * std::max(1, info.ctas_per_sm), static_cast<int>(T.size())));
    sched->regions = P->regions;
    cuda_check(cudaGetDevice(&sched->device), "cudaGetDevice");
    cuda_check(cudaMalloc(&sched->progress, sizeof(int32_t) * static_cast<std::size_t>(P->regions)), "cudaMalloc(progress)");
    cuda_check(cudaMalloc(&sched->tasks, sizeof(gpu::Task) * T.size()), "cudaMalloc(tasks)");
    cuda_check(cudaMemcpyAsync(sched->tasks, T.data(), sizeof(gpu::Task) * T.size(), cudaMemcpyHostToDevice, st),
               "upload tasks");
    cuda_check(cudaMalloc(&P->flags, sizeof(int32_t) * (P->steps.size() + P->block_tasks.size())),
               "cudaMalloc(pipeline flags)");
    cuda_check(cudaStreamSynchronize(st), "upload tasks (sync)");
    P->sched = std::move(sched);
    return P;
}

bool same_opts(const tm_exec_opts& a, const tm_exec_opts& b) {
    return a.numerics == b.numerics && a.schedule == b.schedule && a.split_k == b.split_k && a.ctas == b.ctas &&
           a.tile == b.tile && a.tile_n == b.tile_n && a.parallel_loop == b.parallel_loop &&
           a.staging == b.staging;
}

void run_pipe(tm_plan* plan, const double* A, const double* B, double* C, const tm_exec_opts& o) {
    const Extents& e = plan->nest.ext;
    cudaStream_t st = plan->host_stream, cs = plan->copy_stream, ds = plan->d2h_stream;
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    if (!plan->pipe || !same_opts(plan->pipe->opts, o) || plan->pipe->sched->device != dev)
        plan->pipe = build_pipe(*plan, o, st);
    HostPipe& P = *plan->pipe;
    Schedule& S = *P.sched;
    const std::size_t nu = P.steps.size(), nd = P.block_tasks.size(), ND = static_cast<std::size_t>(P.done_rows);
    if (plan->chunk_ready.empty()) {
        cudaEvent_t ev;
        cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
        plan->chunk_ready.push_back(ev);
    }
    cudaEvent_t zero = plan->chunk_ready[0];
    cuda_check(cudaMemsetAsync(S.progress, 0, sizeof(int32_t) * static_cast<std::size_t>(P.regions), st), "reset progress");
    cuda_check(cudaMemsetAsync(P.flags, 0, sizeof(int32_t) * (nu + nd), st), "reset flags");
    cuda_check(cudaEventRecord(zero, st), "event");
    const bool vec16 = e.m % 2 == 0 && e.k % 2 == 0 && origins_even(S.host_tasks);
    gpu::Args a{plan->dA, e.m, plan->dB, e.k, plan->dC, e.m, S.tasks, static_cast<int32_t>(S.host_tasks.size()),
                S.progress, nullptr, 0, 0, nullptr, P.flags, P.flags + nu};
    // long_ok: the copy-engine-fed launch is paced by the uploads, so auto takes TMA for any length
    // here (e2e 33.2 vs 32.8 TF/s at 16384^3); the HBM-traffic rule is the device path's
    plan->last_staging = launch_tasks(S, a, e.m, e.n, e.k, vec16, o.staging, st, true);

    // uploads in first-need order, a flag after each step's pieces
    cuda_check(cudaStreamWaitEvent(cs, zero, 0), "wait flags reset");
    for (std::size_t u = 0; u < nu; ++u) {
        for (const HostPipe::Piece& pc : P.steps[u].pieces) {
            const i64 ld = pc.op == 'B' ? e.k : e.m;  // leading dimension of the operand (host and device alike)
            const double* src = (pc.op == 'A' ? A : pc.op == 'B' ? B : C) + pc.r0 + pc.c0 * ld;
            double* dst = (pc.op == 'A' ? plan->dA : pc.op == 'B' ? plan->dB : plan->dC) + pc.r0 + pc.c0 * ld;
            if (pc.rows == ld)
                cuda_check(cudaMemcpyAsync(dst, src, static_cast<std::size_t>(pc.rows * pc.cols) * 8, cudaMemcpyHostToDevice, cs),
                           "H2D piece");
            else
                cuda_check(cudaMemcpy2DAsync(dst, static_cast<std::size_t>(ld) * 8, src, static_cast<std::size_t>(ld) * 8,
                                             static_cast<std::size_t>(pc.rows) * 8, static_cast<std::size_t>(pc.cols),
                                             cudaMemcpyHostToDevice, cs),
                           "H2D piece (2-D)");
        }
        cu_check(memops().write(reinterpret_cast<CUstream>(cs), reinterpret_cast<CUdeviceptr>(P.flags + u), 1, 0),
                 "cuStreamWriteValue32");
    }
    // each C cell (column block x row block) goes back once its last chunk's tasks are done, in the order
    // the task list finishes them (a tall C -- 65536 x 256 -- goes back row block by row block under the uploads)
    cuda_check(cudaStreamWaitEvent(ds, zero, 0), "wait flags reset");
    for (const auto& [b, i] : P.cells) {
        const std::size_t cell = static_cast<std::size_t>(b) * ND + static_cast<std::size_t>(i);
        const i64 j0 = P.ncut[static_cast<std::size_t>(b)], w = P.ncut[static_cast<std::size_t>(b) + 1] - j0;
        const i64 i0 = ND == 1 ? 0 : P.mcut[static_cast<std::size_t>(i)];
        const i64 r = ND == 1 ? e.m : P.mcut[static_cast<std::size_t>(i) + 1] - i0;
        cu_check(memops().wait(reinterpret_cast<CUstream>(ds), reinterpret_cast<CUdeviceptr>(P.flags + nu + cell),
                               static_cast<cuuint32_t>(P.block_tasks[cell]), CU_STREAM_WAIT_VALUE_GEQ),
                 "cuStreamWaitValue32");
        if (r == e.m)
            cuda_check(cudaMemcpyAsync(C + j0 * e.m, plan->dC + j0 * e.m, static_cast<std::size_t>(w * e.m) * 8,
                                       cudaMemcpyDeviceToHost, ds),
                       "D2H C block");
        else
            cuda_check(cudaMemcpy2DAsync(C + i0 + j0 * e.m, static_cast<std::size_t>(e.m) * 8, plan->dC + i0 + j0 * e.m,
                                         static_cast<std::size_t>(e.m) * 8, static_cast<std::size_t>(r) * 8,
                                         static_cast<std::size_t>(w), cudaMemcpyDeviceToHost, ds),
                       "D2H C cell (2-D)");
    }
    cuda_check(cudaStreamSynchronize(ds), "execute_host sync");
    cuda_check(cudaStreamSynchronize(st), "execute_host sync");
    plan->last_tasks = static_cast<int64_t>(S.host_tasks.size());
    plan->last_launches = 1;
    plan->last_ctas = S.grid;
}

}  // namespace

void execute_host(tm_plan* plan, const double* A, const double* B, double* C, const tm_exec_opts* opts) {
    if (!plan) fail_usage("null plan");
    if (!A || !B || !C) fail_usage("null operand pointer");
    std::lock_guard<std::mutex> hold(plan->host_mu);
    const Extents& e = plan->nest.ext;
    const std::size_t na = static_cast<std::size_t>(e.m * e.k), nb = static_cast<std::size_t>(e.k * e.n),
                      nc = static_cast<std::size_t>(e.m * e.n);
    auto mkstream = [](cudaStream_t& s) {
        if (!s) cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
    };
    mkstream(plan->host_stream);
    if (!plan->dA) {
        cuda_check(cudaMalloc(&plan->dA, na * sizeof(double)), "cudaMalloc(A)");
        cuda_check(cudaMalloc(&plan->dB, nb * sizeof(double)), "cudaMalloc(B)");
        cuda_check(cudaMalloc(&plan->dC, nc * sizeof(double)), "cudaMalloc(C)");
    }
    cudaStream_t st = plan->host_stream;
    tm_exec_opts o{};
    if (opts) o = *opts;
    // Pipelined when there is enough to overlap: a long k or a wide n, or (round 2) any problem of >= 4 column
    // blocks or >= 4 row blocks whose operands take >= ~1 ms on the bus (2048^3: 2.95 -> 2.52 ms, 3072^3: 7.05 -> 5.24 ms, 1536^3:
    // 1.61 -> 1.52 ms; 1024^3, 25 MB, is slower pipelined: 0.71 -> 0.77 ms; TILEMUL_PIPE_MIN_MB: A/B knob).
    static const double min_mb = [] {
        const char* env = std::getenv("TILEMUL_PIPE_MIN_MB");
        return env ? std::atof(env) : 48.0;
    }();
    const double mbytes = static_cast<double>(na + nb + nc) * 8.0 / 1e6;
    const bool pipelined = o.schedule == TM_SCHEDULE_FUSED && o.split_k <= 1 &&
                           (e.k >= 4096 || e.n >= 4096 || ((e.n >= 1024 || e.m >= 8192) && mbytes >= min_mb));
    if (!pipelined) {
        cuda_check(cudaMemcpyAsync(plan->dA, A, na * sizeof(double), cudaMemcpyHostToDevice, st), "H2D A");
        cuda_check(cudaMemcpyAsync(plan->dB, B, nb * sizeof(double), cudaMemcpyHostToDevice, st), "H2D B");
        cuda_check(cudaMemcpyAsync(plan->dC, C, nc * sizeof(double), cudaMemcpyHostToDevice, st), "H2D C");
        run(plan, plan->dA, e.m, plan->dB, e.k, plan->dC, e.m, opts, st);
        cuda_check(cudaMemcpyAsync(C, plan->dC, nc * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H C");
        cuda_check(cudaStreamSynchronize(st), "execute_host sync");
        return;
    }
    // Copy/compute pipeline over (C column block, k-chunk) units; every
    // C entry still sees its k chunks in ascending order (chunks are
    // multiples of the 32-deep slab), i.e. exactly the unpipelined
    // operation sequence. Preferred: one persistent launch fed by the
    // copy engine (run_pipe).
    mkstream(plan->copy_stream);
    mkstream(plan->d2h_stream);
    if (memops().write && memops().wait && !serialized_launches()) {
        run_pipe(plan, A, B, C, o);
        return;
    }
    // Fallback (driver without stream memory operations): one launch per
    // unit, units in wavefront order (b + q ascending), uploads on one
    // copy stream in first-need order, downloads on a third stream.
    const std::vector<i64> kcut = even_cuts(e.k, e.k >= 4096 ? static_cast<int>(std::min<i64>(8, e.k / 2048)) : 1, 32);
    const std::vector<i64> ncut = even_cuts(e.n, e.n >= 2048 ? static_cast<int>(std::min<i64>(16, e.n / 1024)) : 1, 128);
    const int nq = static_cast<int>(kcut.size()) - 1;
    const int nbk = static_cast<int>(ncut.size()) - 1;
    const std::size_t nev = static_cast<std::size_t>(nq + 2 * nbk + nbk * nq);
    while (plan->chunk_ready.size() < nev) {
        cudaEvent_t ev;
        cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
        plan->chunk_ready.push_back(ev);
    }
    cudaEvent_t* evA = plan->chunk_ready.data();
    cudaEvent_t* evC = evA + nq;
    cudaEvent_t* evDone = evC + nbk;
    cudaEvent_t* evB = evDone + nbk;
    auto sub = [&](i64 nn, i64 kk) -> tm_plan* {
        auto& slot = plan->chunk_plans[{nn, kk}];
        if (!slot) {
            slot = std::make_unique<tm_plan>();
            slot->nest = plan->nest;
            slot->nest.ext.n = nn;
            slot->nest.ext.k = kk;
            slot->hier = plan->hier;
        }
        return slot.get();
    };
    cudaStream_t cs = plan->copy_stream, ds = plan->d2h_stream;
    const std::size_t ld = static_cast<std::size_t>(e.k) * sizeof(double);
    int64_t tasks = 0;
    int32_t launches = 0, ctas = 0;
    auto d2h = [&](int b) {
        const i64 j0 = ncut[static_cast<std::size_t>(b)], w = ncut[static_cast<std::size_t>(b) + 1] - j0;
        cuda_check(cudaStreamWaitEvent(ds, evDone[b], 0), "wait block");
        cuda_check(cudaMemcpyAsync(C + j0 * e.m, plan->dC + j0 * e.m, static_cast<std::size_t>(w * e.m) * 8,
                                   cudaMemcpyDeviceToHost, ds),
                   "D2H C block");
    };
    std::vector<char> have_a(static_cast<std::size_t>(nq), 0);
    std::vector<int> finished;  // blocks whose D2H is issued one unit later (a pageable D2H blocks the host)
    std::vector<std::pair<int, int>> units;
    for (int wave = 0; wave < nbk + nq - 1; ++wave)
        for (int b = std::max(0, wave - nq + 1); b <= std::min(nbk - 1, wave); ++b) units.push_back({b, wave - b});
    {
        for (auto [b, q] : units) {
            const i64 j0 = ncut[static_cast<std::size_t>(b)], w = ncut[static_cast<std::size_t>(b) + 1] - j0;
            const i64 p0 = kcut[static_cast<std::size_t>(q)], kq = kcut[static_cast<std::size_t>(q) + 1] - p0;
            if (q == 0) {
                cuda_check(cudaMemcpyAsync(plan->dC + j0 * e.m, C + j0 * e.m, static_cast<std::size_t>(w * e.m) * 8,
                                           cudaMemcpyHostToDevice, cs),
                           "H2D C block");
                cuda_check(cudaEventRecord(evC[b], cs), "event");
            }
            if (!have_a[static_cast<std::size_t>(q)]) {
                have_a[static_cast<std::size_t>(q)] = 1;
                cuda_check(cudaMemcpyAsync(plan->dA + p0 * e.m, A + p0 * e.m,
                                           static_cast<std::size_t>(kq * e.m) * 8, cudaMemcpyHostToDevice, cs),
                           "H2D A chunk");
                cuda_check(cudaEventRecord(evA[q], cs), "event");
            }
            cuda_check(cudaMemcpy2DAsync(plan->dB + p0 + j0 * e.k, ld, B + p0 + j0 * e.k, ld,
                                         static_cast<std::size_t>(kq) * 8, static_cast<std::size_t>(w),
                                         cudaMemcpyHostToDevice, cs),
                       "H2D B piece");
            cudaEvent_t eb = evB[b * nq + q];
            cuda_check(cudaEventRecord(eb, cs), "event");
            // issue the GEMM right away so pageable-memory copies (which
            // block the host while staging) still overlap device compute
            if (q == 0) cuda_check(cudaStreamWaitEvent(st, evC[b], 0), "wait C block");
            cuda_check(cudaStreamWaitEvent(st, evA[q], 0), "wait A chunk");
            cuda_check(cudaStreamWaitEvent(st, eb, 0), "wait B piece");
            tm_plan* pq = sub(w, kq);
            run(pq, plan->dA + p0 * e.m, e.m, plan->dB + p0 + j0 * e.k, e.k, plan->dC + j0 * e.m, e.m, &o, st);
            tasks += pq->last_tasks;
            launches += pq->last_launches;
            ctas = pq->last_ctas;
            plan->last_staging = pq->last_staging;
            for (int f : finished) d2h(f);
            finished.clear();
            if (q == nq - 1) {
                cuda_check(cudaEventRecord(evDone[b], st), "event");
                finished.push_back(b);
            }
        }
    }
    for (int f : finished) d2h(f);
    cuda_check(cudaStreamSynchronize(ds), "execute_host sync");
    cuda_check(cudaStreamSynchronize(st), "execute_host sync");
    plan->last_tasks = tasks;
    plan->last_launches = launches;
    plan->last_ctas = ctas;
}

}  // namespace engine
}  // namespace mmm
