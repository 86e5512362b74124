"""GPU-aware planning: family members and blocksizes on
the B200 hierarchy, ranked by the MOMMS I/O model.

The reference's `select_algorithm` (descriptor.hpp:206-218) returns C for
every BASELINE shape on a B200-sized L2 (its near/large tolerances never
trigger), and its `derive_blocksizes` keeps each level's aspect
ratio, which on the GPU hierarchy can squeeze a block below one CTA tile.
This planner keeps the reference's derivation but (1) pins the dimensions the
GPU realisation fixes — the SMEM-level m/n block = the CTA tile, and, when
the aspect-preserving shrink makes a member infeasible, the L2 block's m/n
side to a wave-sized extent — and (2) ranks every expressible member by the
modelled traffic into L2 (the HBM boundary), then into SMEM.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Tuple

from . import tilemul as T

# Members expressible on {registers/TMEM, SMEM, L2} with C in registers
# (SURVEY.md §7.1): two cache levels, or one with the SMEM level skipped.
GPU_MEMBERS = ("C2A1C0", "C2B1C0", "B2A1C0", "A2B1C0", "A2C0", "B2C0")
WAVE_TILES = 12  # an L2 block side of 12 CTA tiles: 144 tiles ~ one wave on 148 SMs
# Effective L2 capacity for MOMMS residency, as a fraction of the physical
# 126 MiB. Measured (profiles/model_check_r01_l2frac_*.json): with the L2
# level sized at 100% or 50%, C blocks derived by the reference's fit rules
# do not stay resident (faithful C2A1C0 at 8192^3 moves 17x / 3.1x the
# modelled HBM bytes); at 25% every faithful member lands within 0.95-1.03x
# of the model and the fused schedule within 0.81-1.26x. The L2 is split
# over two dies and also holds the streamed panels, so ~1/4 of it is what a
# resident block can count on.
L2_EFFECTIVE = 0.25


def gpu_hierarchy_effective(tile: int = 128, l2_fraction: float = L2_EFFECTIVE) -> T.CacheHierarchy:
    """The current device's {CTA tile, SMEM, L2} hierarchy with the L2 level
    at its effective capacity for residency."""
    h = T.gpu_hierarchy(tile)
    caps = [h.capacity(i) for i in range(h.size())]
    caps[-1] = max(caps[-2] + 1, int(caps[-1] * l2_fraction))
    return T.CacheHierarchy.from_capacities(caps)


@dataclass
class Candidate:
    name: str
    blocksizes: Optional[T.BlocksizeSet]
    hbm_bytes: float = float("inf")
    smem_bytes: float = float("inf")
    note: str = ""


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


def rank_members(shape: Tuple[int, int, int], hier: T.CacheHierarchy, members=GPU_MEMBERS, tile=(128, 128),
                 wave_block: bool = False, elem_bytes=None) -> List[Candidate]:
    """Every member with its modelled bytes into L2 (top level) and SMEM
    (level 1), cheapest first; infeasible members are kept with a note."""
    eb = elem_bytes or {"A": 8, "B": 8, "C": 8}
    out = []
    for name in members:
        try:
            bs = derive_for_gpu(name, shape, hier, tile, wave_block)
            rep = T.multilevel_cost(T.parse_name(name), bs, hier, T.Shape(*shape))
            out.append(Candidate(name, bs, rep.at_level(hier.top_level()).total_bytes(eb),
                                 rep.at_level(1).total_bytes(eb)))
        except (T.InfeasibleError, T.ValidationFailure, T.ParseError) as e:
            out.append(Candidate(name, None, note=f"{type(e).__name__}: {e}"))
    out.sort(key=lambda c: (c.hbm_bytes, c.smem_bytes, c.name))
    return out


def select_for_gpu(shape: Tuple[int, int, int], hier: Optional[T.CacheHierarchy] = None, tile=(128, 128),
                   wave_block: bool = False):
    """The cheapest member by the model, with the plan built: (nest, candidate).
    Ties (equal modelled bytes) go to the member whose outermost resident the
    reference's select_algorithm picks."""
    hier = hier or gpu_hierarchy_effective(tile[0])
    ranked = rank_members(shape, hier, tile=tile, wave_block=wave_block)
    best = [c for c in ranked if c.blocksizes is not None]
    if not best:
        raise T.InfeasibleError(f"no GPU family member is feasible for shape {shape}")
    ref_outer = T.select_algorithm(T.Shape(*shape), hier.capacity(hier.top_level()))
    top = [c for c in best if c.hbm_bytes == best[0].hbm_bytes]
    pick = next((c for c in top if c.name[0] == ref_outer), top[0])
    nest = T.build_plan(T.parse_name(pick.name), pick.blocksizes, hier, T.Shape(*shape))
    return nest, pick, ranked
