"""GPU parity of the tcgen05 mixed-precision path (BASELINE configs[3]):
BF16 or TF32 inputs rounded from uniform[-1,1) FP64 values, FP32 accumulate,
checked against the FP64 oracle of the ROUNDED inputs with the bound
|C - C_ref| <= (k+2)·u·(|A||B| + |C0|)_ij, u = 2^-24 (fp32 accumulation;
tensor-core accumulation order is unspecified, so no bitwise claim)."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from paper_1904_05717_b200 import tilemul as T

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
U32 = 2.0 ** -24


def tc_plan(m, n, k, tile=128, tile_n=256):
    # register tile = the TMEM accumulator (128 x 256 fp32; 256 x 512 over an SM pair for the wide
    # tile, whose SMEM level is then the pair's); capacities in 2-byte elements
    if tile_n == 512:
        hier = T.CacheHierarchy.from_capacities([256 * 512, 232448, 132644864 // 2])
    else:
        hier = T.CacheHierarchy.from_capacities([128 * 512, 232448 // 2, 132644864 // 2])
    d = T.parse_name("C2A1C0")
    bs = T.derive_blocksizes(d, hier, T.Shape(m, n, k), opts=T.DeriveOptions(micro=T.MicroTile(tile, tile_n)),
                             pinned=T.BlocksizeSet({(1, "m"): min(tile, m)}))
    return T.build_plan(d, bs, hier, T.Shape(m, n, k))


def run_case(m, n, k, dtype, sample=None, seed=5, tile=0, tile_n=0):
    nest = tc_plan(m, n, k, tile if tile else 256, tile_n or (512 if tile != 128 else 256))
    A64 = torch.empty(m * k, dtype=torch.float64, device="cuda")
    B64 = torch.empty(k * n, dtype=torch.float64, device="cuda")
    T.fill_uniform_device(A64, seed)
    T.fill_uniform_device(B64, seed + 1)
    A = T.round_inputs(A64, dtype)
    B = T.round_inputs(B64, dtype)
    C0 = torch.empty(m * n, dtype=torch.float64, device="cuda")
    T.fill_uniform_device(C0, seed + 2)
    C = C0.float()
    c0 = C.double().cpu().numpy()
    T.execute_tc(nest, A, B, C, dtype, T.ExecOptions(tile=tile, tile_n=tile_n))
    torch.cuda.synchronize()
    got = C.double().cpu().numpy()
    a = A.double().cpu().numpy()
    b = B.double().cpu().numpy()
    # rounding is exact RNE: the rounded values differ from the fp64 originals by <= half an ulp
    ulp = 2.0 ** -8 if dtype == "bf16" else 2.0 ** -11
    assert np.all(np.abs(a - A64.cpu().numpy()) <= ulp * np.abs(A64.cpu().numpy()) + 1e-300)
    rng = np.random.default_rng(seed)
    if sample is None:
        ii, jj = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
        ii, jj = ii.ravel(), jj.ravel()
    else:
        ii, jj = rng.integers(0, m, sample), rng.integers(0, n, sample)
    want, ab = O.entries(k, a, m, b, k, c0, m, ii, jj)
    idx = ii + jj * m
    bound = (k + 2) * U32 * (ab + np.abs(c0[idx]))
    err = np.abs(got[idx] - want)
    assert np.all(err <= bound), f"worst {float(np.max(err / bound)):.3g} of bound"
    return nest


# one SM (cta_group::1) / SM pair (cta_group::2) 256x256 / SM pair 256x512 (one 512-column TMEM accumulator)
TILES = [(128, 0), (256, 256), (256, 0)]  # (256, 0): the default, 256 x 512 per pair


@pytest.mark.parametrize("tile,tile_n", TILES)
@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("shape", [(128, 256, 64), (256, 512, 1024), (136, 264, 520), (1000, 776, 328),
                                   (304, 1104, 208)])
def test_tc_small_full_check(dtype, shape, tile, tile_n):
    run_case(*shape, dtype, tile=tile, tile_n=tile_n)


@pytest.mark.parametrize("tile,tile_n", TILES)
@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
def test_tc_large_sampled(dtype, tile, tile_n):
    nest = run_case(4096, 4096, 4096, dtype, sample=2048, tile=tile, tile_n=tile_n)
    assert nest.last_launch()["tasks"] == (4096 // tile) * (4096 // (tile_n or (512 if tile == 256 else 256)))


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
def test_tc_wide_tiles_partial_interior(dtype):
    """256 x 512 pair tiles over a nest whose register blocks are 256 x 384:
    interior tasks do not fill their tile's box, so they keep the per-lane
    epilogue (a box store would overwrite the neighbouring task's C); the
    edge tasks take the TMA epilogue. Full check against the oracle."""
    m, n, k = 512, 1024, 200 if dtype == "tf32" else 208
    hier = T.CacheHierarchy.from_capacities([256 * 512, 232448, 132644864 // 2])
    d = T.parse_name("C2A1C0")
    bs = T.derive_blocksizes(d, hier, T.Shape(m, n, k), opts=T.DeriveOptions(micro=T.MicroTile(256, 384)),
                             pinned=T.BlocksizeSet({(1, "m"): 256}))
    nest = T.build_plan(d, bs, hier, T.Shape(m, n, k))
    assert nest.n_r == 384
    A64 = torch.empty(m * k, dtype=torch.float64, device="cuda")
    B64 = torch.empty(k * n, dtype=torch.float64, device="cuda")
    T.fill_uniform_device(A64, 7)
    T.fill_uniform_device(B64, 8)
    A, B = T.round_inputs(A64, dtype), T.round_inputs(B64, dtype)
    C0 = torch.empty(m * n, dtype=torch.float64, device="cuda")
    T.fill_uniform_device(C0, 9)
    C = C0.float()
    c0 = C.double().cpu().numpy()
    T.execute_tc(nest, A, B, C, dtype, T.ExecOptions(tile=256, tile_n=512))
    torch.cuda.synchronize()
    got = C.double().cpu().numpy()
    a, b = A.double().cpu().numpy(), B.double().cpu().numpy()
    ii, jj = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
    ii, jj = ii.ravel(), jj.ravel()
    want, ab = O.entries(k, a, m, b, k, c0, m, ii, jj)
    idx = ii + jj * m
    bound = (k + 2) * U32 * (ab + np.abs(c0[idx]))
    assert np.all(np.abs(got[idx] - want) <= bound)


def test_tc_rejects_unaligned_and_faithful():
    nest = tc_plan(130, 256, 64)  # lda = 130 bf16 = 260 bytes: not 16-byte aligned for TMA
    A = torch.zeros(130 * 64, dtype=torch.bfloat16, device="cuda")
    B = torch.zeros(64 * 256, dtype=torch.bfloat16, device="cuda")
    C = torch.zeros(130 * 256, dtype=torch.float32, device="cuda")
    with pytest.raises(T.CudaError):
        T.execute_tc(nest, A, B, C, "bf16")
    nest = tc_plan(128, 256, 64)
    with pytest.raises(ValueError):
        T.execute_tc(nest, A[:128 * 64], B, C[:128 * 256], "bf16", T.ExecOptions(schedule="faithful"))


def test_tc_peak_probe():
    """tm_measure_tc_peak: the tcgen05 issue-rate ceiling (roofline denominator
    of this path); tf32 runs at half the bf16 rate, as the instruction set says."""
    bf16 = T.measure_tc_peak("bf16", 3)
    tf32 = T.measure_tc_peak("tf32", 3)
    assert bf16 > 1000.0
    assert 0.4 < tf32 / bf16 < 0.6
    with pytest.raises(ValueError):
        T.measure_tc_peak("fp8", 1)


# The A/B knobs of the pair kernels are read once per process, so their non-default settings run in
# child processes: cluster launch control on the 256 x 512 kernel (TMA epilogue gated on the stage
# ring), off on the 256 x 256 kernel (static persistent stride), and the load-add-store epilogue in place
# of the TMA reduce-add. Shapes with several waves of tiles, so running clusters take unstarted tiles.
KNOB_CASES = [
    ({"TILEMUL_TC_CLC": "1"}, 256, 0),
    ({"TILEMUL_TC_CLC": "0"}, 256, 256),
    ({"TILEMUL_TC_TMA_REDUCE": "0"}, 256, 0),
    ({"TILEMUL_TC_TMA_EPILOGUE": "0"}, 256, 0),
]


@pytest.mark.parametrize("env,tile,tile_n", KNOB_CASES)
def test_tc_knob_variants_in_child_process(env, tile, tile_n):
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
            "import test_gpu_tc as M\n"
            "for dt in ('bf16', 'tf32'):\n"
            "    M.run_case(4096, 4608, 320, dt, sample=4096, tile=%d, tile_n=%d)\n"
            "    M.run_case(1000, 1304, 200, dt, tile=%d, tile_n=%d)\n"
            "print('ok')\n") % (root, os.path.join(root, "tests"), tile, tile_n, tile, tile_n)
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-2000:]
