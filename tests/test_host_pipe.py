"""Host logic of the copy-engine-fed pipeline behind execute() on host buffers
(tm_execute_host; the reference's calling convention, exec.hpp:94-138, takes
host MatrixBuffers): the upload order is a growing box over (row blocks,
column blocks, k-chunks). No GPU: tm_host_pipe_steps is the order alone."""
import numpy as np
import pytest

from paper_1904_05717_b200 import planner as P

SHAPES = [(520, 2200, 8224), (4200, 640, 8224), (6200, 1100, 12320), (16384, 16384, 16384), (2048, 8192, 300),
          (3000, 5000, 4096)]


def steps_of(shape):
    nest, _, _ = P.plan_for_gpu("C2A1C0", shape, "fused", (128, 128))
    return nest.host_pipe_steps()


def chunk_cuts(steps):
    """k-chunk boundaries, from the A pieces' column ranges."""
    cuts = sorted({p[3] for s in steps for p in s["pieces"] if p[0] == "A"} |
                  {p[3] + p[4] for s in steps for p in s["pieces"] if p[0] == "A"})
    return cuts


@pytest.mark.parametrize("shape", SHAPES)
def test_every_element_uploaded_once_and_before_its_tasks(shape):
    m, n, k = shape
    steps = steps_of(shape)
    g = 32  # every cut is a multiple of 32 or the operand's edge
    up = {"A": np.zeros((-(-m // g), -(-k // g)), np.int32), "B": np.zeros((-(-k // g), -(-n // g)), np.int32),
          "C": np.zeros((-(-m // g), -(-n // g)), np.int32)}
    ext = {"A": (m, k), "B": (k, n), "C": (m, n)}
    kc = chunk_cuts(steps)
    assert kc[0] == 0 and kc[-1] == k
    done = [np.zeros((-(-m // g), -(-n // g)), np.int32) for _ in kc[:-1]]
    last_chunk = np.full((-(-m // g), -(-n // g)), -1, np.int32)

    def sl(a, b, edge):
        assert a % g == 0 and (b % g == 0 or b == edge), (a, b, edge)
        return slice(a // g, -(-b // g))

    for s in steps:
        for op, r0, rows, c0, cols in s["pieces"]:
            assert rows > 0 and cols > 0 and r0 + rows <= ext[op][0] and c0 + cols <= ext[op][1]
            up[op][sl(r0, r0 + rows, ext[op][0]), sl(c0, c0 + cols, ext[op][1])] += 1
        i0, i1, j0, j1 = s["box"]
        q = s["chunk"]
        p0, p1 = kc[q], kc[q + 1]
        ri, cj, pk = sl(i0, i1, m), sl(j0, j1, n), sl(p0, p1, k)
        # the flag is written after the step's pieces: everything its tasks touch is up by then
        assert np.all(up["A"][ri, pk] == 1) and np.all(up["B"][pk, cj] == 1) and np.all(up["C"][ri, cj] == 1)
        done[q][ri, cj] += 1
        # every C entry sees its k-chunks in ascending order
        assert np.all(last_chunk[ri, cj] == q - 1)
        last_chunk[ri, cj] = q
    for op in "ABC":
        assert np.all(up[op] == 1), f"{op}: some element not uploaded exactly once"
    for d in done:
        assert np.all(d == 1), "some (row, column, k-chunk) cell not computed exactly once"


def test_first_flag_comes_early_at_the_bench_shape():
    """At 16384^3 the first GEMM tasks wait for ~110 MB, not for a whole 512 MB k-chunk of A."""
    steps = steps_of((16384, 16384, 16384))
    first = sum(p[2] * p[4] * 8 for p in steps[0]["pieces"])
    assert first <= 128 * 2 ** 20
    total = sum(p[2] * p[4] * 8 for s in steps for p in s["pieces"])
    assert total == 3 * 16384 * 16384 * 8
    # the box grows like a cube: 1 GB is 3 s^2 elements of a cube of side s = 6690, i.e. 2 s^3 = 6.8 % of
    # the flops; the order enables at least 6 % by then (the whole first k-chunk of A alone is 0.5 GB)
    up = fl = 0
    for s in steps:
        up += sum(p[2] * p[4] * 8 for p in s["pieces"])
        i0, i1, j0, j1 = s["box"]
        fl += 2 * (i1 - i0) * (j1 - j0) * 4096
        if up >= 2 ** 30:
            break
    assert fl >= 0.05 * 2 * 16384 ** 3


def test_small_problem_is_one_step_per_piece_group():
    steps = steps_of((256, 256, 256))
    assert len(steps) == 1 and steps[0]["box"] == (0, 256, 0, 256) and steps[0]["chunk"] == 0
    assert sorted(p[0] for p in steps[0]["pieces"]) == ["A", "B", "C"]
