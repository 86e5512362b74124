"""The multi-GPU schedule (paper_1904_05717_b200/multigpu.py) on CPU with
gloo, world sizes 2 and 4: the 2-D partition, chunk ownership, the row/column
broadcasts and their overlap order are the product code; only the local
GEMM is a host matmul injected for the test (the GPU path passes the sm_100a
kernel). Result checked against the globally assembled product."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_1904_05717_b200 import multigpu as MG  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _fill_block_cpu(x, rows, cols, ld, seed, row0, col0, gld):
    from oracle import oracle as O

    i = np.arange(rows)[:, None]
    j = np.arange(cols)[None, :]
    vals = O.counter_uniform(seed, ((row0 + i) + (col0 + j) * gld).astype(np.uint64))
    out = x.numpy()
    for jj in range(cols):
        out[jj * ld:jj * ld + rows] = vals[:, jj]


def _worker(rank, world, port, mL, nL, K, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import oracle as O

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lay = MG.make_layout(world, mL, nL, K)
    rows, cols = MG.Summa.groups(dist, lay)
    r, c = lay.coords(rank)
    A = torch.empty(lay.mL * lay.K // lay.Pc, dtype=torch.float64)
    B = torch.empty(lay.K // lay.Pr * lay.nL, dtype=torch.float64)
    C = torch.empty(lay.mL * lay.nL, dtype=torch.float64)
    MG.fill_local(lay, rank, A, B, C, _fill_block_cpu)
    C0 = C.clone()

    def gemm(a, b, cc):  # c += a·b, flat column-major (test-only host matmul)
        am = a.view(lay.KC, lay.mL).t()
        bm = b.view(lay.nL, lay.KC).t()
        cc.view(lay.nL, lay.mL).t().add_(am @ bm)

    s = MG.Summa(lay, rank, "cpu", gemm, dist, rows[r], cols[c])
    s.run(A, B, C)
    # global reference for this rank's block
    gi = np.arange(lay.mL) + r * lay.mL
    gj = np.arange(lay.nL) + c * lay.nL
    p = np.arange(lay.K)
    Ag = O.counter_uniform(11, (gi[:, None] + p[None, :] * lay.M).astype(np.uint64))
    Bg = O.counter_uniform(12, (p[:, None] + gj[None, :] * lay.K).astype(np.uint64))
    want = C0.view(lay.nL, lay.mL).t().numpy() + Ag @ Bg
    got = C.view(lay.nL, lay.mL).t().numpy()
    err = float(np.max(np.abs(got - want)))
    # exchanged volume: everything of A_r / B_c this rank does not own
    expect = 8 * (lay.mL * lay.K * (lay.Pc - 1) // lay.Pc + lay.nL * lay.K * (lay.Pr - 1) // lay.Pr)
    q.put((rank, err, s.exchanged_bytes, expect, (lay.Pr, lay.Pc)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_summa_gloo(world):
    """World 8 is the 2 x 4 grid the 8-GPU config-5 run uses."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    mL, nL, K = 24, 20, 32
    procs = [ctx.Process(target=_worker, args=(r, world, port, mL, nL, K, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, got_bytes, expect, grid in res:
        assert err < 1e-12, (rank, err)
        assert got_bytes == expect, (rank, got_bytes, expect)
    assert res[0][4] == MG.grid_shape(world)


def test_layout_and_ownership():
    assert [MG.grid_shape(p) for p in (1, 2, 4, 8)] == [(1, 1), (1, 2), (2, 2), (2, 4)]
    lay = MG.make_layout(8, 32768, 16384, 65536)
    assert (lay.Pr, lay.Pc, lay.chunks, lay.KC) == (2, 4, 8, 8192)
    assert [lay.a_owner(j) for j in range(8)] == [0, 0, 1, 1, 2, 2, 3, 3]
    assert [lay.b_owner(j) for j in range(8)] == [0, 0, 0, 0, 1, 1, 1, 1]
    with pytest.raises(ValueError):
        MG.make_layout(8, 16, 16, 12)


def test_config5_layouts_fit_one_b200():
    """BASELINE config 5 (65536^3, strong scaled) at N = 1, 2, 4, 8: the grid,
    chunking and each rank's resident bytes (pieces + receive buffers) fit in
    a B200's 180 GB; the exchanged volume per step is what a rank does not own
    of its A row panel and B column panel (SURVEY.md §8e volumes)."""
    S = 65536
    want_grid = {1: (1, 1), 2: (1, 2), 4: (2, 2), 8: (2, 4)}
    for P, (pr, pc) in want_grid.items():
        lay = MG.make_layout(P, S // pr, S // pc, S)
        assert (lay.Pr, lay.Pc, lay.M, lay.N, lay.K) == (pr, pc, S, S, S)
        resident = 8 * (lay.mL * lay.K // lay.Pc + lay.K // lay.Pr * lay.nL + lay.mL * lay.nL)
        recv = 8 * (2 * lay.mL * lay.KC * (lay.Pc > 1) + 2 * lay.KC * lay.nL * (lay.Pr > 1))
        assert resident + recv < 170e9, (P, resident, recv)
        exchanged = 8 * (lay.mL * lay.K * (lay.Pc - 1) // lay.Pc + lay.nL * lay.K * (lay.Pr - 1) // lay.Pr)
        if P == 8:  # A 12.9 GB + B 4.3 GB per rank
            assert abs(exchanged - 17.18e9) < 0.01e9
