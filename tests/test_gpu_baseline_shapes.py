"""GPU parity at the BASELINE.json shapes themselves, on the code paths that
produce the credited numbers (VERDICT r01 "do this" #1).

The reference verifies every shape it times up to verify_max and gates on
rel-Frobenius (tools/tilemul_main.cpp:265-277, tests/acceptance.cpp:66-103).
Above the size a CPU oracle finishes in seconds, these tests check SAMPLED
entries: the inputs are the device's counter-based fills, regenerated on the
host by the oracle's restatement of the generator (oracle.counter_entries),
so nothing the GPU produced feeds the expected values. Bars:

  FP64 (DMMA)    |C - C_ref| <= 4(k+1)u(|A||B| + |C0|), u = 2^-53
  BF16 / TF32    |C - C_ref| <= (k+2)u(|A||B| + |C0|),  u = 2^-24, against
                 the FP64 oracle of the RNE-rounded inputs (rounding restated
                 by oracle.round_rne and checked bitwise on the samples)

plus size-independent properties: the TMA segments are bitwise equal to the
one-launch cp.async kernel over the WHOLE C (same DMMA groups in the same k
order), and C - C0 agrees with A·(B·1) column-sum checksums.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1904_05717_b200 import planner as P
from paper_1904_05717_b200 import tilemul as T
import helpers as H

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
U32 = 2.0 ** -24


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    yield
    torch.cuda.empty_cache()


def filled(m, n, k, seeds=(1, 2, 3)):
    A = torch.empty(m * k, dtype=torch.float64, device="cuda")
    B = torch.empty(k * n, dtype=torch.float64, device="cuda")
    C = torch.empty(m * n, dtype=torch.float64, device="cuda")
    for x, s in zip((A, B, C), seeds):
        T.fill_uniform_device(x, s)
    return A, B, C


def sampled_check(C, m, n, k, samples, seed=5, seeds=(1, 2, 3)):
    rng = np.random.default_rng(seed)
    ii, jj = rng.integers(0, m, samples), rng.integers(0, n, samples)
    got = C[torch.from_numpy(ii + jj * m).cuda()].cpu().numpy()
    want, ab, c0 = O.counter_entries(k, ii, jj, seeds=seeds, lda=m, ldb=k, ldc=m)
    ok, worst = H.entrywise_ok(got, want, ab, k, c0=c0)
    assert ok, f"sampled entries outside 4(k+1)u(|A||B|+|C0|): worst {worst:.3g} of the bound"
    assert H.rel_frobenius(got, want) <= 1e-12
    return worst


def checksum(A, B, C, C0, m, n, k):
    """(C - C0)·1 against A·(B·1): a whole-matrix property (torch fp64 on the
    device as the checker; 2(m+n)k flops)."""
    ones = torch.ones(n, dtype=torch.float64, device="cuda")
    lhs = (C.view(n, m).t() - C0.view(n, m).t()) @ ones
    rhs = A.view(k, m).t() @ (B.view(n, k).t() @ ones)
    assert torch.allclose(lhs, rhs, rtol=0, atol=1e-10 * float(rhs.abs().max()) * k ** 0.5)


# --- the bench's own path: config 2 at 16384^3 (BENCH_r01 headline) --------
def test_headline_16384_segmented_tma():
    """bench.py's exact plan and options: C2A1C0 on the derived hierarchy,
    fused DMMA, auto split (tail split of the last partial wave), auto
    staging = TMA in 14 segment launches of whole rounds. Sampled entries
    against the oracle, the checksum over all of C, and bitwise equality with
    the single-launch cp.async kernel over all 2.7e8 entries."""
    import bench

    m = n = k = 16384
    nest, bs, hier = bench.make_plan(T, m, n, k)
    A, B, C = filled(m, n, k)
    C0 = C.clone()
    opts = T.ExecOptions(numerics="dmma", schedule="fused", split_k=0, staging="auto")
    T.execute(nest, A, B, C, opts)
    torch.cuda.synchronize()
    launch = nest.last_launch()
    assert launch["staging"] == "tma", launch
    assert launch["launches"] == 14, launch
    assert launch["tasks"] > (m // 128) * (n // 128), "tail split: the last partial wave's tiles are cut"
    sampled_check(C, m, n, k, 768)
    checksum(A, B, C, C0, m, n, k)
    Ccp = C0.clone()
    T.execute(nest, A, B, Ccp, T.ExecOptions(numerics="dmma", schedule="fused", split_k=0, staging="cpasync"))
    torch.cuda.synchronize()
    assert nest.last_launch()["launches"] == 1 and nest.last_launch()["staging"] == "cpasync"
    assert torch.equal(C, Ccp), "14 TMA segments differ from the one-launch cp.async kernel"


# --- config 2 at 8192^3: every GPU family member (2 segments each) ---------
@pytest.mark.parametrize("name", P.GPU_MEMBERS)
def test_8192_every_member_segmented(name):
    m = n = k = 8192
    nest, bs, hier = P.plan_for_gpu(name, (m, n, k))
    A, B, C = filled(m, n, k, seeds=(21, 22, 23))
    C0 = C.clone()
    T.execute(nest, A, B, C, T.ExecOptions(split_k=0))
    torch.cuda.synchronize()
    launch = nest.last_launch()
    assert launch["staging"] == "tma" and launch["launches"] >= 2, launch  # ~7085 slabs per CTA -> segments
    sampled_check(C, m, n, k, 512, seed=int.from_bytes(name.encode(), "little") % 1000, seeds=(21, 22, 23))
    checksum(A, B, C, C0, m, n, k)
    Ccp = C0.clone()
    T.execute(nest, A, B, Ccp, T.ExecOptions(split_k=0, staging="cpasync"))
    torch.cuda.synchronize()
    assert torch.equal(C, Ccp), f"{name}: TMA segments differ from cp.async"


# --- config 4 at 16384^3: BF16 and TF32 on tcgen05 -------------------------
@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
def test_config4_16384_tensor_cores(dtype):
    """The default 256x512 SM-pair kernel at the config's own shape. C0 = 0
    as the config says (C init unspecified -> 0, stated). The sampled rows of
    the rounded A/B are checked bitwise against the restated RNE rounding."""
    m = n = k = 16384
    bits = 8 if dtype == "bf16" else 11
    hier = T.CacheHierarchy.from_capacities([256 * 512, 232448, 132644864 // 2])
    d = T.parse_name("C2A1C0")
    bs = T.derive_blocksizes(d, hier, T.Shape(m, n, k), opts=T.DeriveOptions(micro=T.MicroTile(256, 512)),
                             pinned=T.BlocksizeSet({(1, "m"): 256}))
    nest = T.build_plan(d, bs, hier, T.Shape(m, n, k))
    A64 = torch.empty(m * k, dtype=torch.float64, device="cuda")
    T.fill_uniform_device(A64, 31)
    A = T.round_inputs(A64, dtype)
    del A64
    B64 = torch.empty(k * n, dtype=torch.float64, device="cuda")
    T.fill_uniform_device(B64, 32)
    B = T.round_inputs(B64, dtype)
    del B64
    C = torch.zeros(m * n, dtype=torch.float32, device="cuda")
    T.execute_tc(nest, A, B, C, dtype)
    torch.cuda.synchronize()
    assert nest.last_launch()["tasks"] == (m // 256) * (n // 512)
    rng = np.random.default_rng(6)
    S = 512
    ii, jj = rng.integers(0, m, S), rng.integers(0, n, S)
    got = C[torch.from_numpy(ii + jj * m).cuda()].double().cpu().numpy()
    want, ab, _ = O.counter_entries(k, ii, jj, seeds=(31, 32, 0), lda=m, ldb=k, ldc=m, a_round=bits, c0=False)
    # the device rounding of the sampled rows/cols is the restated RNE, bitwise
    p = torch.arange(k, device="cuda")
    a_rows = A.view(k, m)[:, torch.from_numpy(ii[:8]).cuda()].t().double().cpu().numpy()
    b_cols = B.view(n, k)[torch.from_numpy(jj[:8]).cuda()].double().cpu().numpy()
    pp = np.arange(k, dtype=np.uint64)
    assert np.array_equal(a_rows, O.round_rne(O.counter_uniform(31, ii[:8, None].astype(np.uint64) +
                                                                pp[None, :] * np.uint64(m)), bits))
    assert np.array_equal(b_cols, O.round_rne(O.counter_uniform(32, pp[None, :] +
                                                                jj[:8, None].astype(np.uint64) * np.uint64(k)), bits))
    del p
    bound = (k + 2) * U32 * ab
    err = np.abs(got - want)
    assert np.all(err <= bound), f"worst {float(np.max(err / bound)):.3g} of (k+2)u|A||B|"


# --- config 5's local chunked GEMM (multigpu.Summa), segment-triggering ----
def test_config5_chunked_local_gemm_segmented():
    """The SUMMA driver's per-chunk GEMM at a reduced size whose chunks are
    long enough to take the TMA segments (8192 x 8192 C, K = 16384 in two
    chunks of 8192 -> 2 segment launches per chunk), through an NCCL group
    of one rank; sampled entries of C against the restated generator over
    global indices (the config-5 check of tools/config5.py)."""
    import socket

    import torch.distributed as dist

    import bench
    from paper_1904_05717_b200 import multigpu as MG

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        lay = MG.make_layout(1, 8192, 8192, 16384)
        assert lay.chunks == 2 and lay.KC == 8192
        A = torch.empty(lay.mL * lay.K, dtype=torch.float64, device="cuda")
        B = torch.empty(lay.K * lay.nL, dtype=torch.float64, device="cuda")
        Cd = torch.empty(lay.mL * lay.nL, dtype=torch.float64, device="cuda")
        MG.fill_local(lay, 0, A, B, Cd, T.fill_uniform_block)
        nest, _, _ = bench.make_plan(T, lay.mL, lay.nL, lay.KC)
        opts = T.ExecOptions(numerics="dmma", schedule="fused", split_k=0)
        rows, cols = MG.Summa.groups(dist, lay)
        launches = []

        def gemm(a, b, c):
            T.execute(nest, a, b, c, opts)
            launches.append(dict(nest.last_launch()))

        MG.Summa(lay, 0, torch.device("cuda"), gemm, dist, rows[0], cols[0]).run(A, B, Cd)
        torch.cuda.synchronize()
        assert len(launches) == 2 and all(x["staging"] == "tma" and x["launches"] == 2 for x in launches), launches
        rng = np.random.default_rng(12)
        ii, jj = rng.integers(0, lay.mL, 384), rng.integers(0, lay.nL, 384)
        got = Cd[torch.from_numpy(ii + jj * lay.mL).cuda()].cpu().numpy()
        want, ab, c0 = O.counter_entries(lay.K, ii, jj, seeds=(11, 12, 13), lda=lay.M, ldb=lay.K, ldc=lay.M)
        ok, worst = H.entrywise_ok(got, want, ab, lay.K, c0=c0)
        assert ok, worst
    finally:
        dist.destroy_process_group()
