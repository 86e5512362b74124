"""TMA-fed DMMA kernels (k_dmma_tma) against the cp.async kernels and the
oracle.

The two stagings fill the same SMEM level of the family member (the A/B
k-slabs of exec.hpp:35-46's cell at CTA granularity) and feed the same DMMA
groups in the same k order, so the bar between them is BITWISE equality, on
every tile variant and k-split lowering; against the oracle the DMMA bound
of BASELINE.json holds (4·(k+1)·u·(|A||B|+|C0|), u = 2^-53).
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from paper_1904_05717_b200 import tilemul as T
import helpers as H

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    yield


def run(nest, A, B, c, **kw):
    Cd = torch.from_numpy(c.copy()).cuda() if isinstance(c, np.ndarray) else c.clone()
    T.execute(nest, A, B, Cd, T.ExecOptions(**kw))
    torch.cuda.synchronize()
    return Cd.cpu().numpy(), nest.last_launch()["staging"]


def fused_nest(m, n, k, name="C2A1C0"):
    hier = T.gpu_hierarchy(128)
    d = T.parse_name(name)
    bs = T.derive_blocksizes(d, hier, T.Shape(m, n, k), opts=T.DeriveOptions(micro=T.MicroTile(128, 128)),
                             pinned=T.BlocksizeSet({(1, "m"): 128}))
    return T.build_plan(d, bs, hier, T.Shape(m, n, k))


def test_tma_bitwise_equals_cpasync_over_tiles_and_splits():
    rng = np.random.default_rng(2024)
    for trial in range(6):
        # even m and k (TMA needs 16-byte columns of A and B), m not a multiple
        # of 16, k not a multiple of 32; any n
        m = 2 * int(rng.integers(60, 700)) + 2 * (trial % 2)
        n = int(rng.integers(100, 1300))
        k = 2 * int(rng.integers(150, 2000)) + 2 * (trial % 3 == 0)
        nest = fused_nest(m, n, k)
        a, b, c = O.fill_uniform(900 + trial, [(m, k), (k, n), (m, n)])
        A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        ii, jj = rng.integers(0, m, 500), rng.integers(0, n, 500)
        want, ab = O.entries(k, a, m, b, k, c, m, ii, jj)
        for split in (1, 3, 0, -1):
            for tile, tile_n in ((128, 128), (128, 64), (64, 64)):
                kw = dict(split_k=split, tile=tile, tile_n=tile_n)
                got_t, st_t = run(nest, A, B, c, staging="tma", **kw)
                got_c, st_c = run(nest, A, B, c, staging="cpasync", **kw)
                assert (st_t, st_c) == ("tma", "cpasync")
                assert np.array_equal(got_t.view(np.uint64), got_c.view(np.uint64)), (trial, m, n, k, kw)
                ok, worst = H.entrywise_ok(got_t[ii + jj * m], want, ab, k, c0=c[ii + jj * m])
                assert ok, (trial, kw, worst)
                got_a, st_a = run(nest, A, B, c, **kw)  # auto: TMA for the 128x128 kernel, cp.async otherwise
                assert st_a == ("tma" if (tile, tile_n) == (128, 128) else "cpasync")
                assert np.array_equal(got_a, got_t), (trial, m, n, k, kw, int((got_a != got_t).sum()))


def test_tma_small_and_ragged_edges():
    """Tiles smaller than one 16-row swizzle box, n = 1, k < one slab: the
    TMA unit zero-fills everything past the matrix edge."""
    for (m, n, k) in ((2, 1, 2), (16, 3, 6), (18, 130, 30), (130, 2, 34), (256, 257, 64)):
        nest = fused_nest(m, n, k)
        a, b, c = O.fill_uniform(m * 7 + n + k, [(m, k), (k, n), (m, n)])
        A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        for tile, tile_n in ((128, 128), (128, 64), (64, 64)):
            got_t, st = run(nest, A, B, c, staging="tma", tile=tile, tile_n=tile_n)
            assert st == "tma"
            got_c, _ = run(nest, A, B, c, staging="cpasync", tile=tile, tile_n=tile_n)
            assert np.array_equal(got_t.view(np.uint64), got_c.view(np.uint64)), (m, n, k, tile, tile_n)
            ii, jj = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
            ii, jj = ii.reshape(-1), jj.reshape(-1)
            want, ab = O.entries(k, a, m, b, k, c, m, ii, jj)
            ok, worst = H.entrywise_ok(got_t[ii + jj * m], want, ab, k, c0=c[ii + jj * m])
            assert ok, (m, n, k, worst)


@pytest.mark.parametrize("ldc", [310, 311])  # 311: C columns not 16-byte aligned (no C prefetch map, scalar C access)
def test_tma_strided_views(ldc):
    """Operands as column-major sub-views of larger buffers (ld > rows): the
    tensor maps carry the leading dimension, rows past the view are never read
    into C."""
    m, n, k = 300, 270, 530
    lda, ldb = 328, 544
    a, b, c = O.fill_uniform(5, [(lda, k), (ldb, n), (ldc, n)])
    A = torch.from_numpy(a).cuda().view(k, lda).t()[:m, :]
    B = torch.from_numpy(b).cuda().view(n, ldb).t()[:k, :]
    Cb = torch.from_numpy(c).cuda().view(n, ldc).t()
    nest = fused_nest(m, n, k)
    outs = {}
    for staging in ("tma", "cpasync"):
        Cd = Cb.clone()
        T.execute(nest, A, B, Cd[:m, :], T.ExecOptions(staging=staging))
        torch.cuda.synchronize()
        assert nest.last_launch()["staging"] == staging
        outs[staging] = Cd.t().contiguous().cpu().numpy().reshape(-1)
    assert np.array_equal(outs["tma"], outs["cpasync"])
    # rows m..ldc of C are untouched
    assert np.array_equal(outs["tma"].reshape(n, ldc)[:, m:], c.reshape(n, ldc)[:, m:])
    a2 = a.reshape(k, lda)[:, :m].T.copy(order="F").reshape(-1, order="F")
    b2 = b.reshape(n, ldb)[:, :k].T.copy(order="F").reshape(-1, order="F")
    c2 = c.reshape(n, ldc)[:, :m].T.copy(order="F").reshape(-1, order="F")
    got = outs["tma"].reshape(n, ldc)[:, :m].T.reshape(-1, order="F")
    ii, jj = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
    ii, jj = ii.reshape(-1), jj.reshape(-1)
    want, ab = O.entries(k, a2, m, b2, k, c2, m, ii, jj)
    ok, worst = H.entrywise_ok(got[ii + jj * m], want, ab, k, c0=c2[ii + jj * m])
    assert ok, worst


def test_tma_eligibility_and_fallback():
    """Odd leading dimensions (8-byte columns) or faithful cells whose k range
    is not a whole number of slabs: auto falls back to cp.async, an explicit
    staging='tma' is a usage error (status 2 -> ValueError)."""
    m, n, k = 301, 200, 518
    nest = fused_nest(m, n, k)
    a, b, c = O.fill_uniform(3, [(m, k), (k, n), (m, n)])
    A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    _, st = run(nest, A, B, c)
    assert st == "cpasync"
    with pytest.raises(ValueError):
        run(nest, A, B, c, staging="tma")
    # faithful cells of k1 = 106 (not a multiple of 32) -> cp.async; of k1 = 64 -> TMA
    m, k = 300, 518
    a, b, c = O.fill_uniform(4, [(m, k), (k, n), (m, n)])
    A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    hier = T.gpu_hierarchy(128)
    d = T.parse_name("C2A1C0")
    for k1, expect in ((106, "cpasync"), (64, "tma")):
        bs = T.BlocksizeSet({(2, "n"): 200, (2, "m"): 300, (1, "k"): k1, (1, "m"): 128, (0, "n"): 128,
                             (0, "m"): 128})
        nest = T.build_plan(d, bs, hier, T.Shape(m, n, k))
        got, st = run(nest, A, B, c, schedule="faithful")
        assert st == expect, (k1, st)
        ref, _ = run(nest, A, B, c, schedule="faithful", staging="cpasync")
        assert np.array_equal(got, ref)
        ex, _ = run(nest, A, B, c, schedule="faithful", numerics="exact")
        want = c.copy()
        O.execute_nest(m, n, k, [(L.dim, L.blocksize) for L in nest.loops], nest.m_r, nest.n_r, a, b, want)
        assert np.array_equal(ex, want)
        ab = O.abs_product(m, n, k, a, b)
        ok, worst = H.entrywise_ok(got, want, ab, k, c0=c)
        assert ok, worst
    with pytest.raises(ValueError):
        run(nest, A, B, c, numerics="fma", staging="tma")
    # odd task origins (register blocks of 33 rows): a TMA box must start on a
    # 16-byte boundary of its column, so auto falls back to cp.async
    shape = T.Shape(36, 81, 46)
    nest = T.build_plan(T.parse_name("A3C0"), T.BlocksizeSet({(3, "k"): 9, (3, "m"): 19, (0, "n"): 62, (0, "m"): 33}),
                        H.roomy(3), shape)
    a, b, c = O.fill_uniform(1005, [(36, 46), (46, 81), (36, 81)])
    A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    got, st = run(nest, A, B, c)
    assert st == "cpasync"
    with pytest.raises(ValueError):
        run(nest, A, B, c, staging="tma")
    ok, worst = H.entrywise_ok(got, want_of(nest, a, b, c), O.abs_product(36, 81, 46, a, b), 46, c0=c)
    assert ok, worst


def want_of(nest, a, b, c):
    out = c.copy()
    s = nest.shape
    O.execute_nest(s.m, s.n, s.k, [(L.dim, L.blocksize) for L in nest.loops], nest.m_r, nest.n_r, a, b, out)
    return out


def test_tma_host_pipeline_bitwise():
    """tm_execute_host: the copy-engine-fed persistent launch with TMA staging
    (the producer does not run ahead into a unit whose data flag is down)
    equals the cp.async pipeline and the device path, bitwise."""
    m, n, k = 520, 2200, 8224
    nest = fused_nest(m, n, k)
    a, b, c = O.fill_uniform(31, [(m, k), (k, n), (m, n)])
    outs = {}
    for staging in ("tma", "cpasync"):
        hc = c.copy()
        T.execute(nest, a, b, hc, T.ExecOptions(staging=staging))
        assert nest.last_launch()["staging"] == staging
        outs[staging] = hc
    dev_out, _ = run(nest, torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), c)
    assert np.array_equal(outs["tma"].view(np.uint64), outs["cpasync"].view(np.uint64))
    assert np.array_equal(outs["tma"].view(np.uint64), dev_out.view(np.uint64))


def test_tma_config1_golden_entries():
    """Config 1 (2048^3 C2A1C0, seed 12345, C = 0) through the TMA kernel with
    the auto split (stream-K here): the reference's golden entries within the
    bound, and bitwise equal to the cp.async kernel."""
    import json
    import os

    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "config1_2048.json")))
    m = n = k = 2048
    a, b = O.fill_uniform(12345, [(m, k), (k, n)])
    A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    nest = fused_nest(m, n, k)
    got, st = run(nest, A, B, np.zeros(m * n), split_k=0)
    assert st == "tma"
    idx = np.array(g["sample_i"]) + np.array(g["sample_j"]) * m
    ok, worst = H.entrywise_ok(got[idx], np.array(g["sample_c"]), np.array(g["sample_absprod"]), k)
    assert ok, worst
    ab0 = 522.0  # (|A||B|)_00
    assert abs(got[0] - g["C0"]) <= 4 * k * H.U64 * ab0
    ref, _ = run(nest, A, B, np.zeros(m * n), split_k=0, staging="cpasync")
    assert np.array_equal(got, ref)


def test_tma_long_launch_auto_stays_cpasync():
    """A launch whose one task streams more than the 4096-slab TMA limit per
    CTA and cannot be cut into segments (a single round): auto stays on
    cp.async (TMA CTAs drift apart over long launches and lose the wave's L2
    sharing, profiles/tma_l2_r01.json; longer task LISTS are segmented, see
    test_gpu_baseline_shapes.py::test_headline_16384_segmented_tma); an
    explicit TMA launch is bitwise equal. One 128 x 128 tile, k = 8193 slabs
    + 16."""
    m = n = 128
    k = 32 * 8193 + 16
    nest = fused_nest(m, n, k)
    a, b, c = O.fill_uniform(77, [(m, k), (k, n), (m, n)])
    A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    ref, st = run(nest, A, B, c, split_k=1)
    assert st == "cpasync"
    got, st = run(nest, A, B, c, split_k=1, staging="tma")
    assert st == "tma"
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))
    ii = np.arange(0, m, 3)
    jj = (ii * 5) % n
    want, ab = O.entries(k, a, m, b, k, c, m, ii, jj)
    ok, worst = H.entrywise_ok(got[ii + jj * m], want, ab, k, c0=c[ii + jj * m])
    assert ok, worst
    # a short launch of the same kernel: auto takes TMA
    nest2 = fused_nest(m, n, 4096)
    a2, b2, c2 = O.fill_uniform(78, [(m, 4096), (4096, n), (m, n)])
    _, st = run(nest2, torch.from_numpy(a2).cuda(), torch.from_numpy(b2).cuda(), c2, split_k=1)
    assert st == "tma"


def test_segments_and_programmatic_launch_are_bitwise_invisible():
    """A TMA task list longer than 4096 slabs per CTA runs in segments of whole rounds, the segments chained
    by programmatic dependent launch (default) or plain stream order (TILEMUL_TMA_PDL=0); both give C
    bitwise equal to the cp.async kernel in one launch: segmentation and launch chaining change when CTAs
    start, never which tasks run or their k order. Knobs are read once per process: one child per setting."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, hashlib; sys.path.insert(0, %r)\n"
            "import torch\n"
            "from paper_1904_05717_b200 import tilemul as T, planner as P\n"
            "m, n, k = 2048, 2048, 81920\n"
            "nest, bs, hier = P.plan_for_gpu('C2A1C0', (m, n, k), 'fused')\n"
            "A = torch.empty(m * k, dtype=torch.float64, device='cuda')\n"
            "B = torch.empty(k * n, dtype=torch.float64, device='cuda')\n"
            "C = torch.empty(m * n, dtype=torch.float64, device='cuda')\n"
            "for x, s in ((A, 1), (B, 2), (C, 3)): T.fill_uniform_device(x, s)\n"
            "T.execute(nest, A, B, C, T.ExecOptions(split_k=1, staging=sys.argv[1]))\n"
            "torch.cuda.synchronize()\n"
            "print(nest.last_launch()['launches'], nest.last_launch()['staging'],"
            " hashlib.sha256(C.cpu().numpy().tobytes()).hexdigest())\n") % root
    out = {}
    for name, staging, env in (("segments, PDL", "auto", {}),
                               ("segments, stream order", "auto", {"TILEMUL_TMA_PDL": "0"}),
                               ("cp.async, one launch", "cpasync", {})):
        r = subprocess.run([sys.executable, "-c", code, staging], env={**os.environ, **env}, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        launches, got_staging, digest = r.stdout.split()[-3:]
        out[name] = (int(launches), got_staging, digest)
    assert out["segments, PDL"][:2] == (2, "tma") and out["segments, stream order"][:2] == (2, "tma"), out
    assert out["cp.async, one launch"][:2] == (1, "cpasync"), out
    assert len({d for _, _, d in out.values()}) == 1, out


def test_repeated_tma_launches_are_deterministic():
    """Regression for the stage-release race the producer warpgroup exposed: the mbarrier
    arrive that releases a stage was hoisted above the slab's last DMMAs, right behind the issue of its last
    fragment loads, so a refill issued at once overwrote bytes still being read -- 30-60 % of 2048^3 launches
    then differed from the cp.async kernel in whole A fragments of warps 0-2. Every launch must be bitwise
    the cp.async result, launch after launch, for the unsplit, stream-K and uniformly split lowerings."""
    for (m, n, k) in ((2048, 2048, 2048), (4096, 4096, 512)):
        nest = fused_nest(m, n, k)
        A = torch.empty(m * k, dtype=torch.float64, device="cuda")
        B = torch.empty(k * n, dtype=torch.float64, device="cuda")
        C0 = torch.empty(m * n, dtype=torch.float64, device="cuda")
        T.fill_uniform_device(A, 11)
        T.fill_uniform_device(B, 12)
        T.fill_uniform_device(C0, 13)
        for split in (1, 0, 3):
            kw = dict(split_k=split, tile=128, tile_n=128)
            ref = C0.clone()
            T.execute(nest, A, B, ref, T.ExecOptions(staging="cpasync", **kw))
            bad = 0
            for _ in range(25):
                Cd = C0.clone()
                T.execute(nest, A, B, Cd, T.ExecOptions(staging="tma", **kw))
                bad += int(not torch.equal(Cd, ref))
            assert nest.last_launch()["staging"] == "tma"
            assert bad == 0, (m, n, k, split, bad)
