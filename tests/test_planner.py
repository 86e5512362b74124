"""The GPU-aware planner (paper_1904_05717_b200/planner.py) on the B200
hierarchy described as data (no device needed): ranks every expressible
family member by the MOMMS model and picks the cheapest; CPU only."""
from __future__ import annotations

import pytest

from paper_1904_05717_b200 import planner as P
from paper_1904_05717_b200 import tilemul as T

B200 = T.CacheHierarchy.from_capacities([128 * 128, 232448 // 8, 132644864 // 8])
B200_EFF = T.CacheHierarchy.from_capacities([128 * 128, 232448 // 8, int(132644864 // 8 * P.L2_EFFECTIVE)])


@pytest.mark.parametrize("shape,best", [((65536, 256, 1024), {"B2A1C0"}),    # panel-panel: B resident at L2
                                        ((512, 512, 131072), {"C2A1C0"}),    # inner product: C resident
                                        # rank-k: an A or B block of the full k=256 stays in L2 while
                                        # the other streams; C moves once either way (4.50 vs 4.63 GB)
                                        ((16384, 16384, 256), {"A2B1C0", "B2A1C0"})])
def test_selects_model_cheapest_member(shape, best):
    nest, pick, ranked = P.select_for_gpu(shape, B200)
    assert pick.name in best
    feasible = [c for c in ranked if c.blocksizes is not None]
    assert feasible[0].hbm_bytes == pick.hbm_bytes
    assert all(feasible[i].hbm_bytes <= feasible[i + 1].hbm_bytes for i in range(len(feasible) - 1))
    # every member is expressible on the GPU hierarchy (the planner's pins make A2C0/B2C0 feasible)
    assert len(feasible) == len(P.GPU_MEMBERS)


def test_gpu_pins_make_register_tiles_whole():
    bs = P.derive_for_gpu("C2A1C0", (8192, 8192, 8192), B200)
    assert bs.get(1, "m") == 128 and bs.get(0, "m") == 128 and bs.get(0, "n") == 128
    assert bs.get(2, "m") % 128 == 0 and bs.get(2, "n") % 128 == 0
    assert T.validate_blocksizes(T.parse_name("C2A1C0"), bs, B200, T.Shape(8192, 8192, 8192)) == []
    # the reference's aspect-preserving shrink alone makes A2C0 infeasible on this hierarchy
    with pytest.raises(T.InfeasibleError):
        T.derive_blocksizes(T.parse_name("A2C0"), B200, T.Shape(8192, 8192, 8192),
                            opts=T.DeriveOptions(micro=T.MicroTile(128, 128)))
    bs = P.derive_for_gpu("A2C0", (8192, 8192, 8192), B200)
    assert bs.get(2, "m") == P.WAVE_TILES * 128


def test_effective_l2_shrinks_the_resident_block():
    full = P.derive_for_gpu("C2A1C0", (16384, 16384, 16384), B200)
    eff = P.derive_for_gpu("C2A1C0", (16384, 16384, 16384), B200_EFF)
    assert eff.get(2, "m") < full.get(2, "m")
    assert eff.get(2, "m") * eff.get(2, "n") <= B200_EFF.capacity(2)
