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
