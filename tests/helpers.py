"""Shared test fixtures: the reference's random plan generators
(tests/helpers.hpp:18-73, acceptance.cpp:33-53) restated over numpy's
Generator, and the entrywise error bound of BASELINE.json."""
from __future__ import annotations

import numpy as np

from paper_1904_05717_b200 import tilemul as T

U64 = 2.0 ** -53  # unit roundoff of FP64


def roomy(top_level: int) -> T.CacheHierarchy:
    """Capacities large enough that any blocksizes pass the fit rules
    (helpers.hpp:65-73)."""
    return T.CacheHierarchy.from_capacities([(1 << 20) * 4 ** h for h in range(top_level + 1)])


def random_descriptor(rng: np.random.Generator, max_top_level: int = 3) -> T.AlgorithmDescriptor:
    count = int(rng.integers(1, 4))
    pool = list(range(1, max_top_level + 1))
    rng.shuffle(pool)
    levels = sorted(pool[: count - 1], reverse=True) + [0]
    chosen = ["C"] * len(levels)
    for i in range(len(levels) - 2, -1, -1):
        while True:
            pick = "ABC"[int(rng.integers(0, 3))]
            if pick != chosen[i + 1]:
                break
        chosen[i] = pick
    return T.make_descriptor(list(zip(levels, chosen)))


def random_blocksizes(rng, d: T.AlgorithmDescriptor, shape: T.Shape) -> T.BlocksizeSet:
    bs = T.BlocksizeSet()
    for p in d.plans:
        for dim in (p.outer_dim, p.inner_dim):
            bs.set(p.level, dim, int(rng.integers(1, max(1, shape.extent(dim)) + 1)))
    return bs


def rel_frobenius(got, want) -> float:
    num = float(np.sum((got - want) ** 2))
    den = float(np.sum(want ** 2))
    return float(np.sqrt(num / den)) if den > 0 else float(np.sqrt(num))


def entrywise_ok(got, want, absprod, k: int, c0=None, u: float = U64):
    """|got - want| <= 4·k·u·(|A||B|)_ij (+ |C0| term when C0 != 0: the
    standard bound for C0 + AB uses k+1 and adds |C0|)."""
    scale = absprod if c0 is None else absprod + np.abs(c0)
    kk = k if c0 is None else k + 1
    bound = 4.0 * kk * u * scale
    err = np.abs(got - want)
    ok = err <= bound
    worst = float(np.max(err / np.where(bound > 0, bound, 1.0))) if err.size else 0.0
    return bool(np.all(ok)), worst


def random_sim_case(seed: int):
    """A seeded random simulator configuration and event list (cachesim
    golden fixtures, tests/golden/make_golden.py): 1-4 simulated levels with
    random line sizes and inclusive / write-allocate / write-back flags, and
    a mixed read/write stream over all three operands."""
    rng = np.random.default_rng(seed)
    include_registers = bool(rng.integers(0, 4) == 0)
    nsim = int(rng.integers(1, 5))
    levels = [(int(rng.integers(1, 4)), 1, False, True, True)]  # registers
    cap = levels[0][0]
    for _ in range(nsim):
        cap = cap + int(rng.integers(2, 40)) * (1 if rng.integers(0, 2) else 4)
        gran = int(rng.choice([1, 1, 2, 4]))
        levels.append((cap, gran, bool(rng.integers(0, 2)), bool(rng.integers(0, 3) > 0), bool(rng.integers(0, 4) > 0)))
    if include_registers:
        levels[0] = (levels[0][0], 1, False, bool(rng.integers(0, 2)), bool(rng.integers(0, 2)))
    shape = tuple(int(x) for x in rng.integers(2, 12, size=3))
    sizes = {"A": shape[0] * shape[2], "B": shape[2] * shape[1], "C": shape[0] * shape[1]}
    n = int(rng.integers(200, 1500))
    ops = [("A", "B", "C")[int(x)] for x in rng.integers(0, 3, size=n)]
    # skewed indices so reuse happens at every capacity
    idx = [int(min(sizes[o] - 1, abs(rng.normal(0, sizes[o] / 3)))) for o in ops]
    writes = [bool(x) for x in (rng.integers(0, 5, size=n) == 0)]
    flush = bool(rng.integers(0, 5) > 0)
    return {"levels": levels, "shape": shape, "ops": ops, "idx": idx, "writes": writes,
            "include_registers": include_registers, "flush": flush}


def random_sim_plan(seed: int):
    """A seeded random (plan, simulated hierarchy) pair for the cachesim
    golden fixtures: any C-register family member up to 3 levels, random
    blocksizes on a roomy plan hierarchy, a random simulated hierarchy."""
    rng = np.random.default_rng(seed)
    d = random_descriptor(rng)
    shape = T.Shape(*(int(x) for x in rng.integers(2, 24, size=3)))
    bs = random_blocksizes(rng, d, shape)
    nsim = int(rng.integers(1, 4))
    levels = [(int(rng.integers(1, 9)), 1, False, True, True)]
    cap = levels[0][0]
    for _ in range(nsim):
        cap = cap + int(rng.integers(8, 300))
        levels.append((cap, int(rng.choice([1, 1, 2, 4, 8])), bool(rng.integers(0, 2)), bool(rng.integers(0, 3) > 0),
                       bool(rng.integers(0, 4) > 0)))
    return {"name": T.format_name(d), "top": d.top_level(), "shape": (shape.m, shape.n, shape.k),
            "bs": [[l, dim, v] for (l, dim), v in bs.entries()], "sim_levels": levels,
            "packed": bool(rng.integers(0, 2))}
