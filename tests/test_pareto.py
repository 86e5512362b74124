"""pareto_sweep (costmodel.hpp:299-328) against the reference's own outputs
(tests/golden/pareto_cases.json, made by make_golden.py from oracle/_ref):
blocksizes exactly, efficiencies to the last bit, rejections alike."""
from __future__ import annotations

import json
import os

import pytest

from paper_1904_05717_b200 import tilemul as T

CASES = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "pareto_cases.json")))


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c['outer']}-{'-'.join(str(r) for r in c['ratios'])}")
def test_pareto_matches_reference(case):
    opts = T.DeriveOptions(case["slack"], T.MicroTile(case["mr"], case["nr"]))
    if "error" in case:
        with pytest.raises((ValueError, T.InfeasibleError)):
            T.pareto_sweep(case["outer"], case["ratios"], T.Shape(*case["shape"]), opts)
        return
    pts = T.pareto_sweep(case["outer"], case["ratios"], T.Shape(*case["shape"]), opts)
    got = [[p.ratio, p.inner_capacity, p.outer_block_k, p.outer_block_n, p.inner_block_m, p.inner_block_k,
            p.eff_outer_flops_per_element, p.eff_inner_flops_per_element] for p in pts]
    assert got == case["points"]


def test_pareto_rejects_ratio_not_above_one():
    with pytest.raises(ValueError):
        T.pareto_sweep(4096, [1.0], T.Shape(64, 64, 64))
