"""GPU-aware planning: family members and blocksizes on
the B200 hierarchy, ranked by the GPU-mode I/O model.

The reference's `select_algorithm` (descriptor.hpp:206-218) returns C for
every BASELINE shape on a B200-sized L2 (its near/large tolerances never
trigger), and its `derive_blocksizes` keeps each level's aspect
ratio, which on the GPU hierarchy can squeeze a block below one CTA tile.
This planner keeps the reference's derivation but

(1) sizes each level by where the member's resident block physically lives
    on a B200 (gpu_hierarchy_for; no tuned constant):
      level 0  the CTA's C tile (registers / TMEM), m_r x n_r;
      level 1  shared memory per CTA (opt-in maximum);
      level 2  for a C-resident top plan under the fused schedule: the
               register files of the co-resident wave, G x m_r x n_r
               (G = SMs x CTAs per SM) -- the fused schedule keeps every C
               tile in registers for its whole k range, so the "L2 block" of
               C is the set of tiles one wave holds while their A/B slabs
               stream through L2; otherwise (A or B resident, or the faithful
               schedule, whose cells round-trip C through L2): the physical
               L2 (cudaDevAttrL2CacheSize);
(2) pins the dimensions the GPU realisation fixes -- the SMEM-level m/n
    block = the CTA tile, and, when the aspect-preserving shrink makes a
    member infeasible, the L2 block's m/n side to a wave-sized extent;
(3) ranks every expressible member by the GPU-mode model of the schedule the
    kernel will run (LoopNest.gpu_model: FIFO-SMEM term exact over the task
    list, HBM bytes from a lockstep run through an LRU of the physical L2),
    then by the reference's own model.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Tuple

from . import tilemul as T

# Members expressible on {registers/TMEM, SMEM, L2} with C in registers
# (SURVEY.md §7.1): two cache levels, or one with the SMEM level skipped.
GPU_MEMBERS = ("C2A1C0", "C2B1C0", "B2A1C0", "A2B1C0", "A2C0", "B2C0")
WAVE_TILES = 12  # an L2 block side of 12 CTA tiles: 144 tiles ~ one wave on 148 SMs
# B200 facts used when no device is visible (planning on a CPU host): SMs,
# shared memory per block (opt-in), L2 bytes -- the values the device reports.
B200_SMS = 148
B200_SMEM_OPTIN = 232448
B200_L2_BYTES = T.B200_L2_BYTES


def device_facts():
    """(SMs, opt-in shared memory per block, L2 bytes) of the current CUDA
    device, or the B200 values when none is visible."""
    try:
        import torch

        if torch.cuda.is_available():
            p = torch.cuda.get_device_properties(torch.cuda.current_device())
            h = T.gpu_hierarchy(128)
            return p.multi_processor_count, h.capacity(1) * 8, h.capacity(2) * 8
    except Exception:  # noqa: BLE001 -- planning must work without a GPU
        pass
    return B200_SMS, B200_SMEM_OPTIN, B200_L2_BYTES


def gpu_hierarchy_for(name: str, schedule: str = "fused", tile=(128, 128), facts=None,
                      ctas_per_sm: int = 1) -> T.CacheHierarchy:
    """The {C tile, SMEM, level 2} hierarchy in FP64 elements for family
    member `name` under `schedule` (module doc, point 1)."""
    sms, smem, l2 = facts or device_facts()
    tile_el = tile[0] * tile[1]
    top = T.parse_name(name).plans[0]
    if schedule == "fused" and top.resident == "C" and top.level == 2:
        lvl2 = sms * ctas_per_sm * tile_el  # the wave's register-file C tiles
    else:
        lvl2 = l2 // 8
    return T.CacheHierarchy.from_capacities([tile_el, smem // 8, max(lvl2, smem // 8 + 1)])


def plan_for_gpu(name: str, shape: Tuple[int, int, int], schedule: str = "fused", tile=(128, 128), facts=None):
    """(nest, blocksizes, hierarchy) of member `name` on the device's derived
    hierarchy -- the plan bench.py and the tests run."""
    hier = gpu_hierarchy_for(name, schedule, tile, facts)
    bs = derive_for_gpu(name, shape, hier, tile)
    return T.build_plan(T.parse_name(name), bs, hier, T.Shape(*shape)), bs, hier


@dataclass
class Candidate:
    name: str
    blocksizes: Optional[T.BlocksizeSet]
    hbm_bytes: float = float("inf")
    smem_bytes: float = float("inf")
    note: str = ""
    hier: Optional[T.CacheHierarchy] = None


def derive_for_gpu(name: str, shape: Tuple[int, int, int], hier: T.CacheHierarchy, tile=(128, 128),
                   wave_block: bool = False) -> T.BlocksizeSet:
    """derive_blocksizes on the GPU hierarchy with the GPU pins (see module doc).
    wave_block=True pins the L2 block's m/n sides to WAVE_TILES tiles up front
    (the raster the fused schedule runs best with)."""
    d = T.parse_name(name)
    m, n, _ = shape
    pins = {}
    lv1 = d.plan_at(1)
    if lv1 is not None:
        for dim in (lv1.outer_dim, lv1.inner_dim):
            if dim == "m":
                pins[(1, "m")] = min(tile[0], m)
            elif dim == "n":
                pins[(1, "n")] = min(tile[1], n)
    top = d.plans[0]

    def wave_pins():
        for dim in (top.outer_dim, top.inner_dim):
            if dim == "m":
                pins[(top.level, "m")] = min(WAVE_TILES * tile[0], m)
            elif dim == "n":
                pins[(top.level, "n")] = min(WAVE_TILES * tile[1], n)

    if wave_block and top.level >= 1:
        wave_pins()
    opts = T.DeriveOptions(micro=T.MicroTile(tile[0], tile[1]))
    try:
        return T.derive_blocksizes(d, hier, T.Shape(*shape), opts=opts, pinned=T.BlocksizeSet(pins))
    except T.InfeasibleError:
        wave_pins()
        return T.derive_blocksizes(d, hier, T.Shape(*shape), opts=opts, pinned=T.BlocksizeSet(pins))


def rank_members(shape: Tuple[int, int, int], hier: Optional[T.CacheHierarchy] = None, members=GPU_MEMBERS,
                 tile=(128, 128), wave_block: bool = False, elem_bytes=None, schedule: str = "fused",
                 facts=None, gpu_mode: bool = True) -> List[Candidate]:
    """Every member with its modelled bytes across the HBM boundary and into
    SMEM, cheapest first; infeasible members are kept with a note.

    gpu_mode (default): each member on its derived hierarchy
    (gpu_hierarchy_for), costed by the GPU-mode model of the schedule the
    kernel runs (LoopNest.gpu_model). gpu_mode=False: every member on the
    given `hier`, costed by the reference's multilevel_cost."""
    eb = elem_bytes or {"A": 8, "B": 8, "C": 8}
    out = []
    for name in members:
        try:
            h = gpu_hierarchy_for(name, schedule, tile, facts) if (gpu_mode or hier is None) else hier
            bs = derive_for_gpu(name, shape, h, tile, wave_block)
            d = T.parse_name(name)
            if gpu_mode:
                nest = T.build_plan(d, bs, h, T.Shape(*shape))
                sms = (facts or device_facts())[0]
                g = nest.gpu_model(T.ExecOptions(schedule=schedule, split_k=0), sms=sms,
                                   l2_bytes=(facts or device_facts())[2], elem_bytes=(eb["A"], eb["B"], eb["C"]))
                out.append(Candidate(name, bs, float(g["hbm_total_bytes"]), float(g["smem_bytes"]),
                                     hier=h))
            else:
                rep = T.multilevel_cost(d, bs, h, T.Shape(*shape))
                out.append(Candidate(name, bs, rep.at_level(h.top_level()).total_bytes(eb),
                                     rep.at_level(1).total_bytes(eb), hier=h))
        except (T.InfeasibleError, T.ValidationFailure, T.ParseError) as e:
            out.append(Candidate(name, None, note=f"{type(e).__name__}: {e}"))
    out.sort(key=lambda c: (c.hbm_bytes, c.smem_bytes, c.name))
    return out


def select_for_gpu(shape: Tuple[int, int, int], hier: Optional[T.CacheHierarchy] = None, tile=(128, 128),
                   wave_block: bool = False, facts=None):
    """The cheapest member by the model, with the plan built: (nest, candidate,
    ranking). With `hier` given, every member is derived on it and costed by
    the reference's model; without, each on its derived GPU hierarchy and
    costed by the GPU-mode model. Ties (equal modelled bytes) go to the
    member whose outermost resident the reference's select_algorithm picks."""
    ranked = rank_members(shape, hier, tile=tile, wave_block=wave_block, facts=facts, gpu_mode=hier is None)
    best = [c for c in ranked if c.blocksizes is not None]
    if not best:
        raise T.InfeasibleError(f"no GPU family member is feasible for shape {shape}")
    h0 = best[0].hier
    ref_outer = T.select_algorithm(T.Shape(*shape), h0.capacity(h0.top_level()))
    top = [c for c in best if c.hbm_bytes == best[0].hbm_bytes]
    pick = next((c for c in top if c.name[0] == ref_outer), top[0])
    nest = T.build_plan(T.parse_name(pick.name), pick.blocksizes, pick.hier, T.Shape(*shape))
    return nest, pick, ranked


# Config 4 (tcgen05, 256 x 512 SM-pair tiles, one fresh cluster per tile): the raster's L2 block. Measured at
# 16384^3 (profiles/tc_l2_blocks_r02.json): DRAM reads per launch and TF/s by block (m x n)
#   bf16: 2048x2048 / 3072x2048 / 4096x2048 8.9 GB, 1417 TF/s; 2048x1536 9.8 GB; 3072x3072 9.2 GB, 1386;
#         2048x4608 (the round-1 raster) 10.6 GB, 1385; 1024x1024 11.8 GB, 1386
#   tf32: 2048x2048 17.8 GB, 771 TF/s; 4096x1536 19.3 GB, 770; 2048x4608 21.1 GB, 755; 1024x1024 23.0 GB, 757
# Under the board power cap the rate follows the bytes moved. Blocks 2048 columns wide (4 pair tiles) win for
# both input widths: the column's B panels stay in L2 while the window of ~74 tiles in flight walks down it,
# and the A panels are re-read once per 2048 columns. The GPU-mode model of this kernel (gpu_model_tc: tiles
# staggered over the k range, random replacement) ranks the bf16 blocks the same way but not the tf32 ones,
# so the block is the measured one.
TC_L2_BLOCK = (2048, 2048)


def plan_tc_for_gpu(name: str, shape: Tuple[int, int, int], tile=(256, 512), l2_block=TC_L2_BLOCK):
    """(nest, blocksizes, hierarchy) for the tensor-core path (execute_tc): register tile = the SM pair's
    TMEM accumulator, SMEM level = the pair's shared memory, and the raster's L2 block pinned to the measured
    TC_L2_BLOCK (clipped to the shape)."""
    m, n, k = shape
    hier = T.CacheHierarchy.from_capacities([tile[0] * tile[1], B200_SMEM_OPTIN, B200_L2_BYTES // 2])
    d = T.parse_name(name)
    pins = {(1, "m"): min(tile[0], m)}
    top = d.plans[0]
    for dim in (top.outer_dim, top.inner_dim):
        if dim == "m":
            pins[(top.level, "m")] = min(l2_block[0], m)
        elif dim == "n":
            pins[(top.level, "n")] = min(l2_block[1], n)
    bs = T.derive_blocksizes(d, hier, T.Shape(m, n, k), opts=T.DeriveOptions(micro=T.MicroTile(*tile)),
                             pinned=T.BlocksizeSet(pins))
    return T.build_plan(d, bs, hier, T.Shape(m, n, k)), bs, hier
