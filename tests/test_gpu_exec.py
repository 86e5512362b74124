"""GPU parity of the execution path: the sm_100a kernels through the C ABI
against the CPU oracle (oracle/) and the reference itself (oracle/_ref),
restating the reference's own execution tests (tests/test_exec.cpp:22-254,
tests/acceptance.cpp:66-103) plus full-size property checks.

Bars (written here, per numerics):
  exact — bitwise equal to the reference's execute() (and to the restated
          oracle), for every plan and schedule;
  fma   — bitwise equal to the sequential-fma oracle;
  dmma  — entrywise |C_gpu - C_ref| <= 4·k·u·(|A||B|)_ij (u = 2^-53; with
          C0 != 0: (k+1) and + |C0|), and the reference's own gate
          rel_frobenius <= 1e-12 (tools/tilemul_main.cpp:299).
"""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1904_05717_b200 import tilemul as T
import helpers as H

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    yield


def dev(x):
    return torch.from_numpy(x).cuda()


def run_gpu(nest, a, b, c, **kw):
    A, B, Cd = dev(a), dev(b), dev(c.copy())
    T.execute(nest, A, B, Cd, T.ExecOptions(**kw))
    torch.cuda.synchronize()
    return Cd.cpu().numpy()


def oracle_exec(nest, a, b, c, fused=False):
    out = c.copy()
    O.execute_nest(nest.shape.m, nest.shape.n, nest.shape.k, [(L.dim, L.blocksize) for L in nest.loops], nest.m_r,
                   nest.n_r, a, b, out, fused=fused)
    return out


MODES = [("exact", "fused"), ("exact", "faithful"), ("fma", "fused"), ("fma", "faithful"), ("dmma", "fused"),
         ("dmma", "faithful")]


def check(mode, got, a, b, c0, nest, ref_out, fma_out):
    s = nest.shape
    if mode == "exact":
        assert np.array_equal(got.view(np.uint64), ref_out.view(np.uint64)), "exact numerics not bitwise"
    elif mode == "fma":
        assert np.array_equal(got.view(np.uint64), fma_out.view(np.uint64)), "fma numerics not bitwise"
    else:
        ab = O.abs_product(s.m, s.n, s.k, a, b)
        ok, worst = H.entrywise_ok(got, ref_out, ab, s.k, c0=c0)
        assert ok, f"entrywise bound exceeded (worst {worst:.3g} of bound)"
        assert H.rel_frobenius(got, ref_out) <= 1e-12


# --- test_exec.cpp:22-43 / :45-55 (KATs through the GPU) ------------------
def test_kat_1x1x1_and_dot():
    for mode in ("exact", "fma", "dmma"):
        bs = T.BlocksizeSet({(0, "m"): 1, (0, "n"): 1})
        nest = T.build_plan(T.parse_name("C0"), bs, T.CacheHierarchy.from_capacities([64]), T.Shape(1, 1, 1))
        got = run_gpu(nest, np.array([3.0]), np.array([4.0]), np.array([2.0]), numerics=mode)
        assert got[0] == 14.0
        nest = T.build_plan(T.parse_name("C0"), bs, T.CacheHierarchy.from_capacities([64]), T.Shape(1, 1, 2))
        got = run_gpu(nest, np.array([2.0, 3.0]), np.array([5.0, 7.0]), np.array([1.0]), numerics=mode)
        assert got[0] == 32.0


# --- acceptance.cpp:66-103: random plans, dims 1..96, random C --------------
@pytest.mark.parametrize("numerics,schedule", MODES)
def test_random_plans_match_reference(numerics, schedule):
    rng = np.random.default_rng(101)
    ref_ok = O.have_ref()
    for trial in range(40):
        d = H.random_descriptor(rng)
        shape = T.Shape(*[int(x) for x in rng.integers(1, 97, size=3)])
        bs = H.random_blocksizes(rng, d, shape)
        hier = H.roomy(3)
        nest = T.build_plan(d, bs, hier, shape)
        a, b, c = O.fill_uniform(1000 + trial, [(shape.m, shape.k), (shape.k, shape.n), (shape.m, shape.n)])
        want = oracle_exec(nest, a, b, c)
        if ref_ok:  # the reference itself, live
            ref = c.copy()
            O.ref_execute(T.format_name(d), [hier.capacity(i) for i in range(hier.size())],
                          (shape.m, shape.n, shape.k), bs.as_dict(), a, b, ref)
            assert np.array_equal(ref.view(np.uint64), want.view(np.uint64))
        fma = oracle_exec(nest, a, b, c, fused=True) if numerics == "fma" else None
        got = run_gpu(nest, a, b, c, numerics=numerics, schedule=schedule)
        check(numerics, got, a, b, c, nest, want, fma)


# --- test_exec.cpp:113-130: every (i,j,p) exactly once ----------------------
@pytest.mark.parametrize("numerics,schedule", MODES)
def test_iteration_space_exactness(numerics, schedule):
    rng = np.random.default_rng(7)
    for _ in range(12):
        d = H.random_descriptor(rng)
        shape = T.Shape(*[int(x) for x in rng.integers(1, 41, size=3)])
        bs = H.random_blocksizes(rng, d, shape)
        nest = T.build_plan(d, bs, H.roomy(3), shape)
        a = np.ones(shape.m * shape.k)
        b = np.ones(shape.k * shape.n)
        got = run_gpu(nest, a, b, np.zeros(shape.m * shape.n), numerics=numerics, schedule=schedule)
        assert np.all(got == float(shape.k))


# --- test_exec.cpp:184-197 / :199-221 ---------------------------------------
@pytest.mark.parametrize("numerics", ["exact", "fma", "dmma"])
def test_zero_a_leaves_c_and_reuse_accumulates(numerics):
    bs = T.BlocksizeSet({(0, "m"): 4, (0, "n"): 4})
    nest = T.build_plan(T.parse_name("C0"), bs, T.CacheHierarchy.from_capacities([1 << 20]), T.Shape(16, 16, 16))
    (b, c) = O.fill_uniform(17, [(16, 16), (16, 16)])
    got = run_gpu(nest, np.zeros(256), b, c, numerics=numerics)
    assert np.array_equal(got, c)

    bs = T.BlocksizeSet({(1, "m"): 8, (1, "k"): 8, (0, "n"): 3, (0, "m"): 2})
    nest = T.build_plan(T.parse_name("A1C0"), bs, H.roomy(1), T.Shape(20, 18, 22))
    a, b, x = O.fill_uniform(19, [(20, 22), (22, 18), (20, 18)])
    once = run_gpu(nest, a, b, np.zeros(20 * 18), numerics=numerics)
    A, B, X = dev(a), dev(b), dev(x.copy())
    for _ in range(2):
        T.execute(nest, A, B, X, T.ExecOptions(numerics=numerics))
    torch.cuda.synchronize()
    assert H.rel_frobenius(X.cpu().numpy(), x + 2.0 * once) < 1e-12


# --- test_exec.cpp:223-254: the schedule never changes the result ----------
def test_schedules_and_grids_are_bitwise_deterministic():
    bs = T.BlocksizeSet({(2, "n"): 48, (2, "k"): 48, (1, "m"): 24, (1, "k"): 16, (0, "n"): 6, (0, "m"): 4})
    shape = T.Shape(61, 83, 59)
    nest = T.build_plan(T.parse_name("B2A1C0"), bs, H.roomy(2), shape)
    a, b, c = O.fill_uniform(23, [(61, 59), (59, 83), (61, 83)])
    for numerics in ("exact", "fma", "dmma"):
        outs = [run_gpu(nest, a, b, c, numerics=numerics, schedule=s, ctas=g)
                for s in ("fused", "faithful") for g in (0, 1, 7)]
        if numerics == "dmma":  # the k grouping of DMMA is fixed: fused == fused, faithful == faithful
            assert all(np.array_equal(outs[0], o) for o in outs[:3])
            assert all(np.array_equal(outs[3], o) for o in outs[3:])
        else:
            assert all(np.array_equal(outs[0], o) for o in outs)


# --- config 1: 2048^3 C2A1C0, seed 12345, C = 0 (golden from the reference) --
def test_config1_golden():
    g = json.load(open(os.path.join(GOLDEN, "config1_2048.json")))
    m = n = k = 2048
    a, b = O.fill_uniform(12345, [(m, k), (k, n)])
    assert a[0] == g["A"][0] and b[0] == g["B"][0]
    bs = T.BlocksizeSet({(int(l), d): v for l, d, v in g["gpu_blocksizes"]})
    hier = T.CacheHierarchy.from_capacities(g["gpu_hierarchy"])
    nest = T.build_plan(T.parse_name("C2A1C0"), bs, hier, T.Shape(m, n, k))
    ii = np.array(g["sample_i"]), np.array(g["sample_j"])
    idx = ii[0] + ii[1] * m
    for numerics in ("exact", "dmma", "fma"):
        got = run_gpu(nest, a, b, np.zeros(m * n), numerics=numerics)
        if numerics == "exact":  # bit-for-bit the reference's checksums
            assert got[0] == g["C0"] and got[1] == g["C1"] and got[-1] == g["Clast"]
            assert float(np.abs(got).sum()) == pytest.approx(g["sum_abs"], rel=1e-13)
            assert np.array_equal(got[idx], np.array(g["sample_c"]))
        else:
            ok, worst = H.entrywise_ok(got[idx], np.array(g["sample_c"]), np.array(g["sample_absprod"]), k)
            assert ok, worst


# --- full-size property checks (configs 2-3 shapes) --------------------------
@pytest.mark.parametrize("shape,name,split", [((4096, 4096, 4096), "C2A1C0", 1), ((16384, 16384, 256), "C2A1C0", 1),
                                              ((512, 512, 131072), "C2A1C0", 0), ((65536, 256, 1024), "B2A1C0", 1)])
def test_large_shapes_sampled_entries(shape, name, split):
    m, n, k = shape
    hier = T.gpu_hierarchy(128)
    d = T.parse_name(name)
    pins = T.BlocksizeSet({(1, "m"): 128} if name.startswith("C") else {(1, "m"): 128})
    bs = T.derive_blocksizes(d, hier, T.Shape(m, n, k), opts=T.DeriveOptions(micro=T.MicroTile(128, 128)),
                             pinned=pins)
    nest = T.build_plan(d, bs, hier, T.Shape(m, n, k))
    A = torch.empty(m * k, dtype=torch.float64, device="cuda")
    B = torch.empty(k * n, dtype=torch.float64, device="cuda")
    Cd = torch.empty(m * n, dtype=torch.float64, device="cuda")
    T.fill_uniform_device(A, 1)
    T.fill_uniform_device(B, 2)
    T.fill_uniform_device(Cd, 3)
    c0 = Cd.cpu().numpy()
    T.execute(nest, A, B, Cd, T.ExecOptions(split_k=split))
    torch.cuda.synchronize()
    got = Cd.cpu().numpy()
    rng = np.random.default_rng(5)
    ii = rng.integers(0, m, 512)
    jj = rng.integers(0, n, 512)
    a, b = A.cpu().numpy(), B.cpu().numpy()
    want, ab = O.entries(k, a, m, b, k, c0, m, ii, jj)
    ok, worst = H.entrywise_ok(got[ii + jj * m], want, ab, k, c0=c0[ii + jj * m])
    assert ok, worst
    # the whole C moved: a checksum of rows, against the same product via torch (fp64 cuBLAS-free check:
    # C_final - C0 = A·B; compare column sums with A·(B·1))
    ones = torch.ones(n, dtype=torch.float64, device="cuda")
    lhs = (Cd.view(n, m).t() - torch.from_numpy(c0).cuda().view(n, m).t()) @ ones
    rhs = A.view(k, m).t() @ (B.view(n, k).t() @ ones)
    assert torch.allclose(lhs, rhs, rtol=0, atol=1e-9 * float(rhs.abs().max()) + 1e-9)


# --- host-buffer path (the reference's calling convention): the k-chunked
# copy/compute pipeline gives bitwise the device-path result -----------------
@pytest.mark.parametrize("numerics,shape", [("dmma", (520, 2200, 8224)), ("exact", (520, 2200, 8224)),
                                            ("dmma", (4200, 640, 8224)), ("exact", (4200, 640, 8224)),
                                            ("dmma", (6200, 1100, 12320)),
                                            ("dmma", (2048, 1280, 1100)), ("exact", (2048, 1280, 1100)),
                                            ("dmma", (16400, 200, 520)), ("exact", (16400, 200, 520))])
def test_host_buffer_pipeline_matches_device_path(numerics, shape):
    # 520 x 2200 x 8224: 2 k-chunks of 4128 / 4096, 8 column blocks of 384 (tail 296), one row block;
    # 4200 x 640 x 8224: 2 row blocks of A (2176 / 2024) x 2 column blocks x 2 k-chunks;
    # 6200 x 1100 x 12320: 3 row blocks x 4 column blocks x 3 k-chunks (every extension kind of the growing box);
    # 2048 x 1280 x 1100: a small problem (50 MB of operands, one k-chunk, 5 column blocks), pipelined since round 2;
    # 16400 x 200 x 520: a tall C (8 row blocks, one column block): uploaded and downloaded row block by row block
    m, n, k = shape
    hier = T.gpu_hierarchy(128)
    d = T.parse_name("C2A1C0")
    bs = T.derive_blocksizes(d, hier, T.Shape(m, n, k), opts=T.DeriveOptions(micro=T.MicroTile(128, 128)),
                             pinned=T.BlocksizeSet({(1, "m"): 128}))
    nest = T.build_plan(d, bs, hier, T.Shape(m, n, k))
    a, b, c = O.fill_uniform(31, [(m, k), (k, n), (m, n)])
    dev_out = run_gpu(nest, a, b, c, numerics=numerics)
    host_c = c.copy()
    T.execute(nest, a, b, host_c, T.ExecOptions(numerics=numerics))
    # one persistent launch over every (column block, k-chunk) unit, fed by the copy engine
    assert nest.last_launch()["tasks"] > 8  # (1 launch; one per unit under CUDA_LAUNCH_BLOCKING / profilers)
    assert np.array_equal(host_c.view(np.uint64), dev_out.view(np.uint64))
    if numerics == "exact" and m * n * k < 2 ** 34:  # (the larger shapes: the device path is pinned to the oracle elsewhere)
        want = c.copy()
        O.execute_nest(m, n, k, [(L.dim, L.blocksize) for L in nest.loops], nest.m_r, nest.n_r, a, b, want)
        assert np.array_equal(host_c.view(np.uint64), want.view(np.uint64))


def test_device_then_pinned_host_on_fresh_plan():
    """Regression: the task-list upload must be stream-ordered (a pageable
    cudaMemcpy could return before the DMA landed while pinned copies kept
    the copy engine busy -> kernels read a half-written task list)."""
    m = n = 2048
    k = 8192
    hier = T.gpu_hierarchy(128)
    d = T.parse_name("C2A1C0")
    mk = lambda: T.build_plan(d, T.derive_blocksizes(d, hier, T.Shape(m, n, k),  # noqa: E731
                                                     opts=T.DeriveOptions(micro=T.MicroTile(128, 128)),
                                                     pinned=T.BlocksizeSet({(1, "m"): 128})), hier, T.Shape(m, n, k))
    A = torch.empty(m * k, dtype=torch.float64, device="cuda")
    B = torch.empty(k * n, dtype=torch.float64, device="cuda")
    Cd = torch.empty(m * n, dtype=torch.float64, device="cuda")
    T.fill_uniform_device(A, 1)
    T.fill_uniform_device(B, 2)
    T.fill_uniform_device(Cd, 3)
    Ah, Bh, Ch = (x.cpu().pin_memory().numpy() for x in (A, B, Cd))
    T.execute(mk(), A, B, Cd)
    torch.cuda.synchronize()
    T.execute(mk(), Ah, Bh, Ch)
    assert np.array_equal(Ch, Cd.cpu().numpy())


def test_multigpu_driver_world1_nccl():
    """The SUMMA driver on the real GPU with an NCCL group of one rank: the
    chunked local GEMMs over the chunk-major B layout reproduce the product."""
    import socket

    import torch.distributed as dist

    from paper_1904_05717_b200 import multigpu as MG

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        lay = MG.make_layout(1, 384, 256, 4096)
        A = torch.empty(lay.mL * lay.K, dtype=torch.float64, device="cuda")
        B = torch.empty(lay.K * lay.nL, dtype=torch.float64, device="cuda")
        Cd = torch.empty(lay.mL * lay.nL, dtype=torch.float64, device="cuda")
        MG.fill_local(lay, 0, A, B, Cd, T.fill_uniform_block)
        c0 = Cd.cpu().numpy().copy()
        import bench

        nest, _, _ = bench.make_plan(T, lay.mL, lay.nL, lay.KC)
        rows, cols = MG.Summa.groups(dist, lay)
        MG.Summa(lay, 0, torch.device("cuda"), lambda a, b, c: T.execute(nest, a, b, c), dist, rows[0],
                 cols[0]).run(A, B, Cd)
        torch.cuda.synchronize()
        got = Cd.cpu().numpy()
        rng = np.random.default_rng(1)
        ii, jj = rng.integers(0, lay.mL, 256), rng.integers(0, lay.nL, 256)
        p = np.arange(lay.K)
        a_rows = O.counter_uniform(11, (ii[:, None] + p[None, :] * lay.M).astype(np.uint64))
        b_cols = O.counter_uniform(12, (p[None, :] + jj[:, None] * lay.K).astype(np.uint64))
        want = c0[ii + jj * lay.mL] + np.einsum("tp,tp->t", a_rows, b_cols)
        ab = np.einsum("tp,tp->t", np.abs(a_rows), np.abs(b_cols))
        ok, worst = H.entrywise_ok(got[ii + jj * lay.mL], want, ab, lay.K, c0=c0[ii + jj * lay.mL])
        assert ok, worst
    finally:
        dist.destroy_process_group()


def test_multigpu_host_step_world1_nccl():
    """The driver's e2e step (multigpu.HostStep): pinned-host pieces in, C in
    column blocks streamed under the first chunk's GEMM and sent back block by
    block after the last one; the device buffers start zeroed, so every input
    must arrive through the pipeline, and the host C must hold the product."""
    import socket

    import torch.distributed as dist

    from paper_1904_05717_b200 import multigpu as MG

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        lay = MG.make_layout(1, 384, 2560, 2048)  # 2 chunks, 2 C blocks of 1280 columns
        A = torch.empty(lay.mL * lay.K, dtype=torch.float64, device="cuda")
        B = torch.empty(lay.K * lay.nL, dtype=torch.float64, device="cuda")
        Cd = torch.empty(lay.mL * lay.nL, dtype=torch.float64, device="cuda")
        MG.fill_local(lay, 0, A, B, Cd, T.fill_uniform_block)
        Ah, Bh, Ch = (x.cpu().pin_memory() for x in (A, B, Cd))
        c0 = Ch.numpy().copy()
        for x in (A, B, Cd):
            x.zero_()
        import bench

        nest, _, _ = bench.make_plan(T, lay.mL, lay.nL, lay.KC)
        rows, cols = MG.Summa.groups(dist, lay)
        sm = MG.Summa(lay, 0, torch.device("cuda"), lambda a, b, c: T.execute(nest, a, b, c), dist, rows[0], cols[0])
        hs = MG.HostStep(sm, A, B, Cd, lambda w: bench.make_plan(T, lay.mL, w, lay.KC)[0],
                         lambda n, a, b, c: T.execute(n, a, b, c))
        assert len(hs.blocks) == 2
        hs.run(Ah, Bh, Ch)
        torch.cuda.synchronize()
        got = Ch.numpy()
        rng = np.random.default_rng(2)
        ii, jj = rng.integers(0, lay.mL, 512), rng.integers(0, lay.nL, 512)
        p = np.arange(lay.K)
        a_rows = O.counter_uniform(11, (ii[:, None] + p[None, :] * lay.M).astype(np.uint64))
        b_cols = O.counter_uniform(12, (p[None, :] + jj[:, None] * lay.K).astype(np.uint64))
        want = c0[ii + jj * lay.mL] + np.einsum("tp,tp->t", a_rows, b_cols)
        ab = np.einsum("tp,tp->t", np.abs(a_rows), np.abs(b_cols))
        ok, worst = H.entrywise_ok(got[ii + jj * lay.mL], want, ab, lay.K, c0=c0[ii + jj * lay.mL])
        assert ok, worst
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("split", [0, 3, -1])
def test_split_k_tail_and_uniform(split):
    """split_k=-1 (stream-K: equal contiguous (tile, k-slab) ranges per CTA),
    split_k=0 (auto; stream-K for this ragged 256-tile grid), split_k=3
    (every tile in 3 parts). All reduce the cut tiles in a fixed slot order:
    within the bound and bitwise reproducible run to run."""
    m = n = k = 2048
    hier = T.gpu_hierarchy(128)
    d = T.parse_name("C2A1C0")
    bs = T.derive_blocksizes(d, hier, T.Shape(m, n, k), opts=T.DeriveOptions(micro=T.MicroTile(128, 128)),
                             pinned=T.BlocksizeSet({(1, "m"): 128}))
    nest = T.build_plan(d, bs, hier, T.Shape(m, n, k))
    a, b, c = O.fill_uniform(41, [(m, k), (k, n), (m, n)])
    got1 = run_gpu(nest, a, b, c, split_k=split)
    launch = nest.last_launch()
    assert launch["launches"] == 1  # cut tiles are finished in-kernel (Task::fixup), no reduce launch
    assert launch["tasks"] > 256
    got2 = run_gpu(nest, a, b, c, split_k=split)
    assert np.array_equal(got1, got2)
    rng = np.random.default_rng(9)
    ii, jj = rng.integers(0, m, 4096), rng.integers(0, n, 4096)
    want, ab = O.entries(k, a, m, b, k, c, m, ii, jj)
    ok, worst = H.entrywise_ok(got1[ii + jj * m], want, ab, k, c0=c[ii + jj * m])
    assert ok, worst
    # a second launch on different inputs: the fix-up counters must start from
    # zero again, or an owner could fold the previous launch's (stale) partials
    b2 = b * 0.5
    got3 = run_gpu(nest, a, b2, c, split_k=split)
    want2, ab2 = O.entries(k, a, m, b2, k, c, m, ii, jj)
    ok, worst = H.entrywise_ok(got3[ii + jj * m], want2, ab2, k, c0=c[ii + jj * m])
    assert ok, worst
    # the SIMT kernels keep the separate fixed-order reduction launch
    if split == 3:
        f1 = run_gpu(nest, a, b, c, numerics="fma", split_k=3)
        assert nest.last_launch()["launches"] == 2
        assert np.array_equal(f1, run_gpu(nest, a, b, c, numerics="fma", split_k=3))
        ok, worst = H.entrywise_ok(f1[ii + jj * m], want, ab, k, c0=c[ii + jj * m])
        assert ok, worst
    # exact numerics ignore auto-splitting and stay bitwise equal to the reference
    if split == 0:
        ex = run_gpu(nest, a, b, c, numerics="exact", split_k=0)
        assert nest.last_launch()["launches"] == 1
        want_all = c.copy()
        O.execute_nest(m, n, k, [(L.dim, L.blocksize) for L in nest.loops], nest.m_r, nest.n_r, a, b, want_all)
        assert np.array_equal(ex, want_all)


# --- test_exec.cpp:154-182: execute consumes prepacked hierarchical buffers ---
@pytest.mark.parametrize("numerics", ["exact", "dmma"])
def test_prepacked_buffers(numerics):
    shape = T.Shape(37, 29, 41)
    bs = T.BlocksizeSet({(1, "m"): 12, (1, "k"): 16, (0, "n"): 6, (0, "m"): 4})
    hier = H.roomy(1)
    nest = T.build_plan(T.parse_name("A1C0"), bs, hier, shape)
    a, b, c = O.fill_uniform(13, [(37, 41), (41, 29), (37, 29)])
    Ap, Bp, Cp = (T.pack(dev(x), nest, op) for x, op in ((a, "A"), (b, "B"), (c, "C")))
    caps = [hier.capacity(i) for i in range(hier.size())]
    if O.have_ref():  # device pack == the reference's pack, bitwise
        for x, op, got in ((a, "A", Ap), (b, "B", Bp), (c, "C", Cp)):
            assert np.array_equal(got.cpu().numpy(), O.ref_pack("A1C0", caps, (37, 29, 41), bs.as_dict(), op, x))
    for x, op, got in ((a, "A", Ap), (b, "B", Bp)):  # round trip
        assert np.array_equal(T.unpack(got, nest, op).cpu().numpy(), x)
    T.execute_packed(nest, Ap, Bp, Cp, T.ExecOptions(numerics=numerics))
    torch.cuda.synchronize()
    out = T.unpack(Cp, nest, "C").cpu().numpy()
    want = oracle_exec(nest, a, b, c)
    if O.have_ref():
        ref = c.copy()
        O.ref_execute("A1C0", caps, (37, 29, 41), bs.as_dict(), a, b, ref, packed=True)
        assert np.array_equal(ref, want)
    check(numerics, out, a, b, c, nest, want, None)


def test_randomized_split_modes_and_tiles():
    """Odd shapes x every k-split lowering (none / uniform / auto tail /
    stream-K) x every DMMA tile variant: within the bound, and each
    configuration bitwise reproducible."""
    rng = np.random.default_rng(77)
    hier = T.gpu_hierarchy(128)
    d = T.parse_name("C2A1C0")
    for trial in range(10):
        m, n = (int(x) for x in rng.integers(130, 1400, size=2))
        k = int(rng.integers(600, 5000))
        bs = T.derive_blocksizes(d, hier, T.Shape(m, n, k), opts=T.DeriveOptions(micro=T.MicroTile(128, 128)),
                                 pinned=T.BlocksizeSet({(1, "m"): 128}))
        nest = T.build_plan(d, bs, hier, T.Shape(m, n, k))
        a, b, c = O.fill_uniform(500 + trial, [(m, k), (k, n), (m, n)])
        ii, jj = rng.integers(0, m, 600), rng.integers(0, n, 600)
        want, ab = O.entries(k, a, m, b, k, c, m, ii, jj)
        for split in (1, 3, 0, -1):
            for tile, tile_n in ((0, 0), (128, 128), (128, 64), (64, 64)):
                kw = dict(split_k=split, tile=tile, tile_n=tile_n)
                got = run_gpu(nest, a, b, c, **kw)
                ok, worst = H.entrywise_ok(got[ii + jj * m], want, ab, k, c0=c[ii + jj * m])
                assert ok, (trial, m, n, k, kw, worst)
                assert np.array_equal(got, run_gpu(nest, a, b, c, **kw)), (trial, kw)


def test_host_pipeline_fallback_under_launch_blocking():
    """With CUDA_LAUNCH_BLOCKING=1 (or a profiler injected) the persistent,
    copy-engine-fed pipeline cannot run (its tasks wait on another stream's
    copies); tm_execute_host takes the one-launch-per-unit path instead, with
    bitwise the same result."""
    import subprocess
    import sys

    code = r"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1904_05717_b200 import tilemul as T
from oracle import oracle as O
m, n, k = 520, 2200, 8224
hier = T.gpu_hierarchy(128)
d = T.parse_name('C2A1C0')
bs = T.derive_blocksizes(d, hier, T.Shape(m, n, k), opts=T.DeriveOptions(micro=T.MicroTile(128, 128)),
                         pinned=T.BlocksizeSet({(1, 'm'): 128}))
nest = T.build_plan(d, bs, hier, T.Shape(m, n, k))
a, b, c = O.fill_uniform(31, [(m, k), (k, n), (m, n)])
Cd = torch.from_numpy(c.copy()).cuda()
T.execute(nest, torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), Cd)
torch.cuda.synchronize()
hc = c.copy()
T.execute(nest, a, b, hc)
assert nest.last_launch()['launches'] > 1, nest.last_launch()
assert np.array_equal(hc.view(np.uint64), Cd.cpu().numpy().view(np.uint64))
print('ok')
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, CUDA_LAUNCH_BLOCKING="1"))
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-3000:]


# --- exec.hpp:106-131 / test_exec.cpp:223-254: the parallel loop never changes
# results (faithful schedule: each iteration of the chosen m/n loop is a worker)
def test_faithful_parallel_loop_choice_is_bitwise_invariant():
    m, n, k = 300, 260, 530
    d = T.parse_name("B2A1C0")
    hier = T.gpu_hierarchy(64)
    bs = T.BlocksizeSet({(2, "n"): 128, (2, "k"): 192, (1, "m"): 64, (1, "k"): 64, (0, "n"): 64, (0, "m"): 64})
    nest = T.build_plan(d, bs, hier, T.Shape(m, n, k))
    a, b, c = O.fill_uniform(17, [(m, k), (k, n), (m, n)])
    want = oracle_exec(nest, a, b, c)
    outs = []
    for par in (-1, 0, 2, 4, 5):  # auto, n2, m1, n0, m0 (k loops are at 1 and 3)
        got = run_gpu(nest, a, b, c, numerics="exact", schedule="faithful", parallel_loop=par)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), par
        outs.append(got)
    with pytest.raises(ValueError):
        run_gpu(nest, a, b, c, numerics="exact", schedule="faithful", parallel_loop=1)  # k2
