"""The GPU-mode I/O model (LoopNest.gpu_model, csrc/gpu_model.cpp) against
closed forms and against the reference-semantics LRU simulator at desk scale
(SURVEY.md §7.1 FIFO-SMEM mode, §8 rows a15/f2; VERDICT r01 "do this" #3).
CPU only: the model and the task lists come from the host half of the
lowering (no GPU).

* FIFO-SMEM level, closed form: the fused schedule without splits moves
  mk*ceil(n/n_r) + kn*ceil(m/m_r) + 2mn elements into SMEM; the faithful
  schedule multiplies the reference's level-1 resident term by the
  replication factor (every CTA that runs an iteration of a spatial loop
  inside the SMEM-resident block stages its own copy).
* Simulator cross-check: the element-level trace of each CTA's tasks through
  the LRU simulator (cachesim.cpp, pinned count-for-count to the reference's
  cachesim.hpp) with a ring-sized level reproduces the SMEM term; the
  lockstep interleaving of all CTAs through an L2-sized level reproduces the
  HBM bytes of the model's slab-granular LRU.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

from paper_1904_05717_b200 import tilemul as T

ROOMY = T.CacheHierarchy.from_capacities([1 << 20, 1 << 22, 1 << 40])


def nest_of(name, shape, bs):
    return T.build_plan(T.parse_name(name), T.BlocksizeSet(bs), ROOMY, T.Shape(*shape))


def c2a1c0(shape, blk=(256, 256), k1=64, tile=128):
    return nest_of("C2A1C0", shape, {(0, "m"): tile, (0, "n"): tile, (1, "m"): tile, (1, "k"): k1,
                                     (2, "m"): blk[0], (2, "n"): blk[1]})


@pytest.mark.parametrize("shape", [(512, 384, 256), (640, 1000, 96), (384, 256, 1000)])
def test_fifo_smem_closed_form_fused(shape):
    m, n, k = shape
    nest = c2a1c0(shape)
    g = nest.gpu_model(T.ExecOptions(split_k=1), sms=7)
    A, B, C = g["smem_elements"]["A"], g["smem_elements"]["B"], g["smem_elements"]["C"]
    assert A == (m * k * math.ceil(n / 128), 0)
    assert B == (k * n * math.ceil(m / 128), 0)
    assert C == (m * n, m * n)


def test_split_parts_add_partials_to_the_smem_term():
    """Every cut tile's parts: the contributors write partials, the owner
    reads C and the partials and writes C once."""
    m, n, k = 512, 512, 4096
    nest = c2a1c0((m, n, k))
    base = nest.gpu_model(T.ExecOptions(split_k=1), sms=148)
    for split in (3, 0, -1):
        ts, grid, ranges = nest.tasks(T.ExecOptions(split_k=split), sms=148)
        g = nest.gpu_model(T.ExecOptions(split_k=split), sms=148)
        assert g["smem_elements"]["A"] == base["smem_elements"]["A"]  # k ranges partition k
        extra = sum(t["m"] * t["n"] for t in ts if t["fixup"] == 1)
        assert g["smem_elements"]["C"] == (m * n + extra, m * n + extra), split


@pytest.mark.parametrize("name,bs,resident,inner", [
    ("C2A1C0", {(2, "n"): 512, (2, "m"): 512, (1, "k"): 96, (1, "m"): 128, (0, "n"): 128, (0, "m"): 128}, "A", "n"),
    ("B2A1C0", {(2, "n"): 512, (2, "k"): 256, (1, "m"): 128, (1, "k"): 64, (0, "n"): 128, (0, "m"): 128}, "A", "n"),
    ("A2B1C0", {(2, "m"): 512, (2, "k"): 256, (1, "n"): 128, (1, "k"): 64, (0, "n"): 128, (0, "m"): 128}, "B", "m"),
])
def test_faithful_smem_is_reference_level1_times_replication(name, bs, resident, inner):
    """Faithful schedule (one task per nest cell): the reference's level-1
    traffic of the SMEM-resident operand times the replication factor of the
    spatial loop inside its block -- every n0 (m0) iteration is a separate
    CTA task that stages its own copy -- while the streamed operand and C
    keep the reference's terms."""
    shape = (768, 1024, 512)
    nest = nest_of(name, shape, bs)
    ref = nest.model().at_level(1)
    g = nest.gpu_model(T.ExecOptions(schedule="faithful"), sms=148)
    # replication: the register loop inside the SMEM block runs ceil(b/128) cells per enclosing L2 block
    # of extent b along `inner` (margins included); the resident's reads per block do not depend on b
    extent, blk = shape[0 if inner == "m" else 1], bs[(2, inner)]
    blocks = [min(blk, extent - s0) for s0 in range(0, extent, blk)]
    reps = [math.ceil(b / 128) for b in blocks]
    streamed = "B" if resident == "A" else "A"
    assert g["smem_elements"][resident][0] * len(blocks) == sum(reps) * ref.of(resident).reads
    assert g["smem_elements"][streamed][0] == ref.of(streamed).reads
    assert g["smem_elements"]["C"] == (ref.of("C").reads, ref.of("C").writes)


# ---------------------------------------------------------------- simulator
def _cta_streams(nest, opts, sms):
    ts, grid, ranges = nest.tasks(opts, sms=sms)
    if ranges is None:
        return ts, [[ts[q] for q in range(c, len(ts), grid)] for c in range(grid)]
    return ts, [[ts[q] for q in range(ranges[c], ranges[c + 1])] for c in range(grid)]


def _task_events(t, s, bk, m, k, phase):
    """Element events of task t at lockstep step s (phase 'start' / slab / 'end')."""
    ops, idx, wr = [], [], []
    ii = np.arange(t["i0"], t["i0"] + t["m"])
    jj = np.arange(t["j0"], t["j0"] + t["n"])
    if phase == "start":
        cc = (ii[:, None] + jj[None, :] * m).ravel()
        ops += ["C"] * cc.size
        idx += cc.tolist()
        wr += [False] * cc.size
    elif phase == "end":
        cc = (ii[:, None] + jj[None, :] * m).ravel()
        ops += ["C"] * cc.size
        idx += cc.tolist()
        wr += [True] * cc.size
    else:
        p0 = t["p0"] + s * bk
        pp = np.arange(p0, min(p0 + bk, t["p0"] + t["k"]))
        aa = (ii[:, None] + pp[None, :] * m).ravel()
        b_ = (pp[:, None] + jj[None, :] * k).ravel()
        ops += ["A"] * aa.size + ["B"] * b_.size
        idx += aa.tolist() + b_.tolist()
        wr += [False] * (aa.size + b_.size)
    return ops, idx, wr


def _lockstep(streams, bk, m, k, sink):
    """The model's lockstep order: each step, CTA 0..G-1 each run one k-slab
    (C read at a task's start, C written at its end)."""
    pos = [0] * len(streams)
    slab = [-1] * len(streams)
    while any(p < len(s) for p, s in zip(pos, streams)):
        for c, st in enumerate(streams):
            if pos[c] >= len(st):
                continue
            t = st[pos[c]]
            if slab[c] < 0:
                sink(*_task_events(t, 0, bk, m, k, "start"))
                slab[c] = 0
            n = -(-t["k"] // bk)
            if slab[c] < n:
                sink(*_task_events(t, slab[c], bk, m, k, "slab"))
                slab[c] += 1
            if slab[c] >= n:
                sink(*_task_events(t, 0, bk, m, k, "end"))
                pos[c] += 1
                slab[c] = -1


@pytest.mark.parametrize("shape,sms", [((384, 256, 160), 2), ((256, 512, 224), 3)])
def test_simulator_reproduces_fifo_smem_term(shape, sms):
    """Each CTA's own A/B slab stream through a one-level LRU of the SMEM
    ring's capacity (3 stages x (128x32 + 32x128) FP64 elements): the level's
    transfers equal the model's A and B SMEM terms. (C is not staged in
    SMEM: it sits in the CTA's registers for the task, one read and one write
    per task, the closed form checked above. k spans more slabs than the
    ring holds, so a task's stream is a FIFO pass, as in the kernel.)"""
    m, n, k = shape
    nest = c2a1c0(shape)
    opts = T.ExecOptions(split_k=1)
    _, streams = _cta_streams(nest, opts, sms)
    ring = 3 * (128 * 32 + 32 * 128)
    total = 0
    def ab_only(sim):
        def sink(o, i, w):
            keep = [q for q, op in enumerate(o) if op != "C"]
            if keep:
                sim.access_many([o[q] for q in keep], [i[q] for q in keep], [w[q] for q in keep])
        return sink

    for st in streams:
        sim = T.LruSimulator(T.CacheHierarchy.from_capacities([1, ring]), T.Shape(m, n, k))
        _lockstep([st], 32, m, k, ab_only(sim))
        total += sim.finish().at_level(1).transferred_elements()
    g = nest.gpu_model(opts, sms=sms)
    assert total == g["smem_elements"]["A"][0] + g["smem_elements"]["B"][0]


@pytest.mark.parametrize("shape,sms,l2_elems", [((512, 512, 256), 4, 80000), ((384, 640, 192), 6, 90000),
                                               ((768, 768, 256), 8, 120000), ((768, 768, 256), 8, 400000),
                                               ((256, 256, 512), 2, 1 << 20)])
def test_simulator_reproduces_lockstep_l2_model(shape, sms, l2_elems):
    """All CTAs interleaved in lockstep through one LRU level of the L2's
    capacity (element lines, no write-allocate fetch -- the L2 writes whole
    sectors): its traffic across the memory boundary equals the model's
    slab-granular LRU (exactly on these cases; units are whole k-slabs
    there, elements here, so a cache of only a few slabs can differ by a few
    percent), and equals the compulsory bytes when the L2 holds everything."""
    m, n, k = shape
    nest = c2a1c0(shape, blk=(256, 256))
    opts = T.ExecOptions(split_k=1)
    _, streams = _cta_streams(nest, opts, sms)
    # the L2 writes whole sectors without reading them: no write-allocate fetch (a write miss goes through)
    hier = T.CacheHierarchy([T.CacheLevel(0, 1), T.CacheLevel(1, l2_elems, 1, False, False, True)])
    sim = T.LruSimulator(hier, T.Shape(m, n, k))
    _lockstep(streams, 32, m, k, lambda o, i, w: sim.access_many(o, i, w) if i else None)
    simulated = 8 * sim.finish().at_level(1).transferred_elements()
    g = nest.gpu_model(opts, sms=sms, l2_bytes=8 * l2_elems)
    assert abs(simulated - g["hbm_total_bytes"]) <= 0.01 * simulated, (simulated, g["hbm_total_bytes"])
    if l2_elems >= m * k + k * n + m * n:
        assert g["hbm_total_bytes"] == 8 * (m * k + k * n + 2 * m * n)


def test_wave_model_explains_the_raster():
    """The fused schedule's HBM traffic is set by how many A row panels and B
    column panels one wave of co-resident CTAs streams: the C2A1C0 raster in
    wave-sized L2 blocks moves less than a raster along one long row of
    tiles, as the reference's model says for resident-C blocks (and with L2
    too small to carry panels from one wave to the next, both equal the
    per-wave panel count exactly)."""
    m = n = k = 2048
    sq = c2a1c0((m, n, k), blk=(512, 512), k1=64)   # 4 x 4 tiles per block
    row = c2a1c0((m, n, k), blk=(128, 2048), k1=64)  # 1 x 16 tiles per block
    l2 = 8 * 4 * (128 * 32) * 16  # a few slabs per CTA: no cross-wave reuse
    gs = sq.gpu_model(T.ExecOptions(split_k=1), sms=16, l2_bytes=l2)
    gr = row.gpu_model(T.ExecOptions(split_k=1), sms=16, l2_bytes=l2)
    assert gs["hbm_read_bytes"] < gr["hbm_read_bytes"]
    # per wave of 16 tiles: 4 A + 4 B panels (square) vs 1 A + 16 B panels (row)
    waves = (m // 128) * (n // 128) // 16
    assert gs["hbm_bytes"]["A"][0] + gs["hbm_bytes"]["B"][0] == waves * 8 * 8 * 128 * k
    assert gr["hbm_bytes"]["A"][0] + gr["hbm_bytes"]["B"][0] == waves * 17 * 8 * 128 * k


@pytest.mark.parametrize("dtype,eb", [("bf16", 2), ("tf32", 4)])
def test_tc_model_fifo_term_and_bounds(dtype, eb):
    """The tcgen05 path's model (gpu_model_tc): 256 x 512 SM-pair tiles, one per cluster, sms/2 clusters
    in flight, 2- or 4-byte inputs and fp32 C. Its SMEM term is the FIFO closed form over those tiles
    (mk*ceil(n/512) + kn*ceil(m/256) input elements, C once in and once out), its HBM bytes lie between the
    compulsory bytes and everything the tiles read."""
    m, n, k = 2048, 3072, 1024
    hier = T.CacheHierarchy.from_capacities([256 * 512, 232448, 132644864 // 2])
    d = T.parse_name("C2A1C0")
    bs = T.derive_blocksizes(d, hier, T.Shape(m, n, k), opts=T.DeriveOptions(micro=T.MicroTile(256, 512)),
                             pinned=T.BlocksizeSet({(1, "m"): 256, (2, "m"): 1024, (2, "n"): 1024}))
    nest = T.build_plan(d, bs, hier, T.Shape(m, n, k))
    g = nest.gpu_model_tc(dtype, T.ExecOptions(tile=256, tile_n=512), sms=148)
    tiles = (m // 256) * (n // 512)
    assert g["tile"] == (256, 512) and g["tasks"] == tiles and g["grid"] == min(74, tiles)
    a_el = m * k * math.ceil(n / 512)
    b_el = k * n * math.ceil(m / 256)
    assert g["smem_elements"]["A"] == (a_el, 0) and g["smem_elements"]["B"] == (b_el, 0)
    assert g["smem_elements"]["C"] == (m * n, m * n)
    assert g["smem_bytes"] == eb * (a_el + b_el) + 4 * 2 * m * n
    compulsory = eb * (m * k + k * n) + 4 * m * n
    assert compulsory <= g["hbm_read_bytes"] <= eb * (a_el + b_el) + 4 * m * n
    assert g["hbm_bytes"]["C"][1] == 4 * m * n  # C written back once
