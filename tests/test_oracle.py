"""Pins the CPU oracle (oracle/oracle.c, a restatement) before it is trusted:
against the reference's golden values (committed fixtures and the values the
reference's own tests assert) and, when oracle/_ref is built, against the
reference itself on seeded random inputs. CPU only."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

import helpers as H
from oracle import oracle as O
from paper_1904_05717_b200 import tilemul as T

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
needs_ref = pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built")


def test_generator_matches_golden_config1():
    g = json.load(open(os.path.join(GOLDEN, "config1_2048.json")))
    a, b = O.fill_uniform(12345, [(2048, 2048), (2048, 2048)])
    assert a[:3].tolist() == g["A"][:3] and a[-1] == g["A"][3]
    assert b[:3].tolist() == g["B"][:3] and b[-1] == g["B"][3]
    # survey golden values: A[0..2], B[0..2]
    assert a[0] == -0.28474055422314815 and b[0] == -0.3107348365662056


def test_sequential_entries_match_golden_config1():
    """The oracle's sequential-k entry values equal the reference's execute()
    output bit for bit on 4096 sampled entries of the 2048^3 golden run."""
    g = json.load(open(os.path.join(GOLDEN, "config1_2048.json")))
    a, b = O.fill_uniform(12345, [(2048, 2048), (2048, 2048)])
    ii, jj = np.array(g["sample_i"][:512]), np.array(g["sample_j"][:512])
    got, ab = O.entries(2048, a, 2048, b, 2048, None, 2048, ii, jj)
    assert np.array_equal(got, np.array(g["sample_c"][:512]))
    assert np.array_equal(ab, np.array(g["sample_absprod"][:512]))
    assert g["C0"] == 20.84727373830074  # C[0] = 20.847273738300739


def test_reference_kats_restated():
    # test_exec.cpp:22-55: 2 + 3*4 = 14; 1 + 2*5 + 3*7 = 32; identity A adds B exactly
    c = np.array([2.0])
    O.reference_gemm(1, 1, 1, np.array([3.0]), np.array([4.0]), c)
    assert c[0] == 14.0
    c = np.array([1.0])
    O.execute_nest(1, 1, 2, [("n", 1), ("m", 1)], 1, 1, np.array([2.0, 3.0]), np.array([5.0, 7.0]), c)
    assert c[0] == 32.0
    (b,) = O.fill_uniform(2, [(5, 7)])
    eye = np.eye(5).reshape(-1, order="F").copy()
    c = np.zeros(35)
    O.reference_gemm(5, 7, 5, eye, b, c)
    assert np.array_equal(c, b)


def test_oracle_execute_equals_reference_gemm_with_zero_c():
    # with C = 0, any nest's execute() is bitwise reference_gemm
    rng = np.random.default_rng(11)
    for _ in range(25):
        d = H.random_descriptor(rng)
        s = T.Shape(*[int(x) for x in rng.integers(1, 49, size=3)])
        bs = H.random_blocksizes(rng, d, s)
        nest = T.build_plan(d, bs, H.roomy(3), s)
        a, b = O.fill_uniform(int(rng.integers(0, 1 << 30)), [(s.m, s.k), (s.k, s.n)])
        c1 = np.zeros(s.m * s.n)
        O.execute_nest(s.m, s.n, s.k, [(L.dim, L.blocksize) for L in nest.loops], nest.m_r, nest.n_r, a, b, c1)
        c2 = np.zeros(s.m * s.n)
        O.reference_gemm(s.m, s.n, s.k, a, b, c2)
        assert np.array_equal(c1, c2)


@needs_ref
def test_generator_matches_reference_stream():
    for seed in (0, 1, 12345, 2 ** 63 + 5):
        x = O.fill_uniform(seed, [(37, 11), (11, 5), (37, 5)])
        y = O.fill_uniform(seed, [(37, 11), (11, 5), (37, 5)], lib_=O.ref())
        for u, v in zip(x, y):
            assert np.array_equal(u, v)


@needs_ref
def test_oracle_execute_matches_reference_on_random_plans():
    """acceptance.cpp:66-103 against the reference itself, bitwise."""
    rng = np.random.default_rng(101)
    hier = H.roomy(3)
    caps = [hier.capacity(i) for i in range(hier.size())]
    for t in range(60):
        d = H.random_descriptor(rng)
        s = T.Shape(*[int(x) for x in rng.integers(1, 97, size=3)])
        bs = H.random_blocksizes(rng, d, s)
        nest = T.build_plan(d, bs, hier, s)
        a, b, c = O.fill_uniform(t, [(s.m, s.k), (s.k, s.n), (s.m, s.n)])
        want = c.copy()
        O.ref_execute(T.format_name(d), caps, (s.m, s.n, s.k), bs.as_dict(), a, b, want)
        got = c.copy()
        cells = O.execute_nest(s.m, s.n, s.k, [(L.dim, L.blocksize) for L in nest.loops], nest.m_r, nest.n_r, a, b,
                               got)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
        assert cells == nest.cell_count()
        # workers never change the reference's result (test_exec.cpp:223-254)
        w = c.copy()
        par = [i for i, L in enumerate(nest.loops) if L.dim != "k"]
        O.ref_execute(T.format_name(d), caps, (s.m, s.n, s.k), bs.as_dict(), a, b, w, workers=3,
                      parallel_loop=par[-1])
        assert np.array_equal(w, want)


@needs_ref
def test_reference_cost_helpers_match_host_library():
    R = O.ref()
    assert R.ref_goto_efficiency(192, 3000) == T.goto_efficiency(192, 3000)
    for v in "ABC":
        for b1, b2 in ((3000, 192), (192, 3000), (768, 768), (7, 3)):
            assert R.ref_streaming_efficiency(v.encode(), b1, b2) == T.streaming_efficiency(v, b1, b2)
    out = np.zeros(6, dtype=np.int64)
    R.ref_resident_cost(b"A", 50, 60, 70, 12, 16, out)
    t = T.resident_cost("A", T.Shape(50, 60, 70), 12, 16)
    assert out.tolist() == [t.of(o).reads if i % 2 == 0 else t.of(o).writes for o in "ABC" for i in (0, 1)]
