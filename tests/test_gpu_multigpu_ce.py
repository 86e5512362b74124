"""The multi-GPU driver's copy-engine exchange (multigpu.Summa.attach_peers:
peer pieces mapped over CUDA IPC, chunks pulled by the DMA engines under the
local GEMM) with the sm_100a kernel as the local GEMM.

This box has one GPU, so the ranks are 2 and 4 processes sharing cuda:0
with gloo as the control plane (handle exchange, barriers). Nothing here
makes one rank's kernel wait on another's: the resident pulls read pieces
that are static after the fill, and in the e2e step (pieces re-uploaded
every step) only streams wait on other ranks' events, each recorded before
the wait is issued (host barriers), so sharing the device changes timing,
not the data flow. Checked entrywise against the oracle over each rank's
whole C block, and the pulled volume byte-exact.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mL, nL, K, q):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import helpers as H
    from oracle import oracle as O
    from paper_1904_05717_b200 import multigpu as MG
    from paper_1904_05717_b200 import tilemul as T

    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        lay = MG.make_layout(world, mL, nL, K)
        rows, cols = MG.Summa.groups(dist, lay)
        r, c = lay.coords(rank)
        A = torch.empty(lay.mL * lay.K // lay.Pc, dtype=torch.float64, device=dev)
        B = torch.empty(lay.K // lay.Pr * lay.nL, dtype=torch.float64, device=dev)
        C = torch.empty(lay.mL * lay.nL, dtype=torch.float64, device=dev)
        MG.fill_local(lay, rank, A, B, C, T.fill_uniform_block)
        torch.cuda.synchronize()
        C0 = C.cpu().numpy().copy()
        hier = T.gpu_hierarchy(128)
        d = T.parse_name("C2A1C0")
        bs = T.derive_blocksizes(d, hier, T.Shape(lay.mL, lay.nL, lay.KC),
                                 opts=T.DeriveOptions(micro=T.MicroTile(128, 128)),
                                 pinned=T.BlocksizeSet({(1, "m"): 128}))
        nest = T.build_plan(d, bs, hier, T.Shape(lay.mL, lay.nL, lay.KC))

        def gemm(a, b, cc):
            T.execute(nest, a, b, cc, T.ExecOptions())

        s = MG.Summa(lay, rank, dev, gemm, dist, rows[r], cols[c])
        assert s.attach_peers(A, B)
        s.run(A, B, C)
        torch.cuda.synchronize()
        with pytest.raises(ValueError):  # per-step uploads need the step events
            s.run(A, B, C, ready=[None] * lay.chunks)
        s.detach_peers()
        got = C.cpu().numpy()
        # reference: every entry of this rank's block from the global seeded matrices
        gi = np.arange(lay.mL) + r * lay.mL
        gj = np.arange(lay.nL) + c * lay.nL
        p = np.arange(lay.K)
        Ag = O.counter_uniform(11, (gi[:, None] + p[None, :] * lay.M).astype(np.uint64))
        Bg = O.counter_uniform(12, (p[:, None] + gj[None, :] * lay.K).astype(np.uint64))
        want = (C0.reshape(lay.nL, lay.mL).T + Ag @ Bg)
        ab = np.abs(Ag) @ np.abs(Bg)
        ok, worst = H.entrywise_ok(got.reshape(lay.nL, lay.mL).T.ravel(), want.ravel(), ab.ravel(), lay.K,
                                   c0=C0.reshape(lay.nL, lay.mL).T.ravel())
        expect = 8 * (lay.mL * lay.K * (lay.Pc - 1) // lay.Pc + lay.nL * lay.K * (lay.Pr - 1) // lay.Pr)
        q.put((rank, ok, worst, s.exchanged_bytes, expect, None))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:  # report instead of hanging the parent
        import traceback

        q.put((rank, False, float("nan"), 0, 0, traceback.format_exc()))


def _host_step_worker(rank, world, port, mL, nL, K, q):
    """Two e2e steps (multigpu.HostStep) with copy-engine pulls ordered by the
    cross-process step events; step 2 uploads 2·A, issued without a host sync
    in between, so a pull that read an owner's piece after its step-2 upload
    (or before its step-1 upload: the device buffers start zeroed) shows up
    in C = C0 + A·B + 2A·B."""
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import bench
    import helpers as H
    from oracle import oracle as O
    from paper_1904_05717_b200 import multigpu as MG
    from paper_1904_05717_b200 import tilemul as T

    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        lay = MG.make_layout(world, mL, nL, K)
        rows, cols = MG.Summa.groups(dist, lay)
        r, c = lay.coords(rank)
        A = torch.empty(lay.mL * lay.K // lay.Pc, dtype=torch.float64, device=dev)
        B = torch.empty(lay.K // lay.Pr * lay.nL, dtype=torch.float64, device=dev)
        C = torch.empty(lay.mL * lay.nL, dtype=torch.float64, device=dev)
        MG.fill_local(lay, rank, A, B, C, T.fill_uniform_block)
        torch.cuda.synchronize()
        Ah1, Bh, Ch = (x.cpu().pin_memory() for x in (A, B, C))
        Ah2 = (2.0 * A).cpu().pin_memory()
        C0 = Ch.numpy().copy()
        for x in (A, B, C):
            x.zero_()
        torch.cuda.synchronize()
        nest, _, _ = bench.make_plan(T, lay.mL, lay.nL, lay.KC)
        s = MG.Summa(lay, rank, dev, lambda a, b, cc: T.execute(nest, a, b, cc), dist, rows[r], cols[c])
        assert s.attach_peers(A, B)
        assert s.attach_step_sync()
        hs = MG.HostStep(s, A, B, C, lambda w: bench.make_plan(T, lay.mL, w, lay.KC)[0],
                         lambda n, a, b, cc: T.execute(n, a, b, cc))
        hs.run(Ah1, Bh, Ch)
        hs.run(Ah2, Bh, Ch)
        torch.cuda.synchronize()
        dist.barrier()
        s.detach_peers()
        got = Ch.numpy()
        gi = np.arange(lay.mL) + r * lay.mL
        gj = np.arange(lay.nL) + c * lay.nL
        p = np.arange(lay.K)
        Ag = O.counter_uniform(11, (gi[:, None] + p[None, :] * lay.M).astype(np.uint64))
        Bg = O.counter_uniform(12, (p[:, None] + gj[None, :] * lay.K).astype(np.uint64))
        c0 = C0.reshape(lay.nL, lay.mL).T
        want = c0 + 3.0 * (Ag @ Bg)
        ab = 3.0 * (np.abs(Ag) @ np.abs(Bg))
        ok, worst = H.entrywise_ok(got.reshape(lay.nL, lay.mL).T.ravel(), want.ravel(), ab.ravel(), 2 * lay.K,
                                   c0=c0.ravel())
        expect = 2 * 8 * (lay.mL * lay.K * (lay.Pc - 1) // lay.Pc + lay.nL * lay.K * (lay.Pr - 1) // lay.Pr)
        q.put((rank, ok, worst, s.exchanged_bytes, expect, None))
        dist.barrier()
        dist.destroy_process_group()
    except Exception:  # report instead of hanging the parent
        import traceback

        q.put((rank, False, float("nan"), 0, 0, traceback.format_exc()))


def _spawn(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for rank, ok, worst, got_bytes, want_bytes, tb in res:
        assert tb is None, tb
        assert ok, (rank, worst)
        assert got_bytes == want_bytes, (rank, got_bytes, want_bytes)


@pytest.mark.parametrize("world", [2, 4])
def test_copy_engine_host_step_matches_oracle(world):
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    _spawn(_host_step_worker, world, 256, 2048, 1024)


@pytest.mark.parametrize("world", [2, 4])
def test_copy_engine_exchange_matches_oracle(world):
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    _spawn(_worker, world, 256, 384, 1024)


def _bench_worker(rank, world, port, size, q):
    """bench.py's N > 1 arm (multigpu.bench) end to end, gloo in place of
    NCCL: the resident loop with copy-engine pulls, then the e2e steps with
    the step events; rank 0's JSON line comes back through the queue."""
    import argparse
    import contextlib
    import io
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench
    from paper_1904_05717_b200 import multigpu as MG
    from paper_1904_05717_b200 import tilemul as T

    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        args = argparse.Namespace(config="5", size=size, steps=2, warmup=3, no_e2e=False, no_verify=False, no_cpu=True)
        out = io.StringIO()
        with contextlib.redirect_stdout(out):
            rc = MG.bench(args, T, bench.make_plan, world, rank, 0)
        q.put((rank, rc, out.getvalue(), None))
    except Exception:  # report instead of hanging the parent
        import traceback

        q.put((rank, 1, "", traceback.format_exc()))


@pytest.mark.parametrize("world", [2, 4])
def test_multigpu_bench_arm_world_gt1(world):
    """The JSON line of the N > 1 bench arm: config 5 strong-scaled (a fixed
    size^3 problem over the Pr x Pc grid), pulls in both the resident and the
    e2e step, and every rank's sampled entries verified against the oracle."""
    import json

    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, world, port, 2048, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    for rank, rc, _, tb in res:
        assert tb is None, tb
        assert rc == 0, rank
    line = json.loads(res[0][2].strip().splitlines()[-1])
    assert line["n_gpus"] == world and line["scaling"] == "strong" and line["value"] > 0
    assert (line["config"]["m"], line["config"]["n"], line["config"]["k"]) == (2048, 2048, 2048)
    from paper_1904_05717_b200 import multigpu as MG

    assert line["config"]["grid"] == list(MG.grid_shape(world))
    assert line["verified"]["ok"] and line["verified"]["ranks"] == world
    assert line["config"]["exchange"].startswith("copy-engine pulls")
    assert line["e2e"]["exchange"].startswith("copy-engine pulls") and "events" in line["e2e"]["exchange"]
    assert line["e2e"]["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] > 0
    assert line["gpu_launches"] > 0 and line["exchanged_bytes_per_step_rank0"] > 0
