#!/usr/bin/env python
"""BASELINE configs[4]: FP64 m=n=k=65536 (34.4 GB per matrix), C 2-D
block-partitioned over the ranks, A row-panels / B column-panels exchanged in
k-chunks (paper_1904_05717_b200/multigpu.py). Runs under torchrun with any
world size (1 GPU here: the whole 103 GB problem on one B200).

    torchrun --nproc-per-node N tools/config5.py [--size 65536] [--steps 1]

Prints one JSON line from rank 0: TFLOP/s (max-over-ranks CUDA-event time),
exchanged bytes, and a sampled-entry check of rank 0's block against the
oracle restatement of the device generator (bound 4(k+1)u(|A||B| + |C0|)).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=65536)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--samples", type=int, default=128)
    args = ap.parse_args()
    import numpy as np
    import torch
    import torch.distributed as dist

    import bench
    from paper_1904_05717_b200 import multigpu as MG
    from paper_1904_05717_b200 import tilemul as T

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
    pr, pc = MG.grid_shape(world)
    size = args.size
    lay = MG.make_layout(world, size // pr, size // pc, size)
    rows, cols = MG.Summa.groups(dist, lay)
    r, c = lay.coords(rank)
    dev = torch.device("cuda", local)
    nest, bs, hier = bench.make_plan(T, lay.mL, lay.nL, lay.KC)
    A = torch.empty(lay.mL * lay.K // lay.Pc, dtype=torch.float64, device=dev)
    B = torch.empty(lay.K // lay.Pr * lay.nL, dtype=torch.float64, device=dev)
    C = torch.empty(lay.mL * lay.nL, dtype=torch.float64, device=dev)
    MG.fill_local(lay, rank, A, B, C, T.fill_uniform_block)
    rng = np.random.default_rng(7)
    ii = rng.integers(0, lay.mL, args.samples)
    jj = rng.integers(0, lay.nL, args.samples)
    c0 = C[torch.from_numpy(ii + jj * lay.mL).to(dev)].cpu().numpy()
    opts = T.ExecOptions(numerics="dmma", schedule="fused", split_k=0)
    s = MG.Summa(lay, rank, dev, lambda a, b, cc: T.execute(nest, a, b, cc, opts), dist, rows[r], cols[c])
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        s.run(A, B, C)
    e1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    t = float(ms.item()) / 1e3
    got = C[torch.from_numpy(ii + jj * lay.mL).to(dev)].cpu().numpy()
    # oracle: the device generator restated in numpy over global indices
    from oracle import oracle as O

    gi = ii + r * lay.mL
    gj = jj + c * lay.nL
    p = np.arange(lay.K, dtype=np.uint64)
    want = np.empty(args.samples)
    ab = np.empty(args.samples)
    for q in range(args.samples):
        arow = O.counter_uniform(11, np.uint64(gi[q]) + p * np.uint64(lay.M))
        bcol = O.counter_uniform(12, p + np.uint64(gj[q]) * np.uint64(lay.K))
        want[q] = c0[q] + args.steps * float(np.dot(arow, bcol))
        ab[q] = float(np.dot(np.abs(arow), np.abs(bcol)))
    bound = 4.0 * (args.steps * lay.K + 1) * 2.0 ** -53 * (args.steps * ab + np.abs(c0))
    ok = bool(np.all(np.abs(got - want) <= bound))
    flops = 2.0 * lay.M * lay.N * lay.K * args.steps
    if rank == 0:
        print(json.dumps({"config": "config5", "shape": [lay.M, lay.N, lay.K], "n_gpus": world,
                          "grid": [lay.Pr, lay.Pc], "local_block": [lay.mL, lay.nL], "chunks": lay.chunks,
                          "kc": lay.KC, "seconds": t, "tflops": flops / t / 1e12,
                          "tflops_per_gpu": flops / t / 1e12 / world,
                          "exchanged_bytes_rank0": s.exchanged_bytes,
                          "hbm_bytes_allocated_per_gpu": 8 * (A.numel() + B.numel() + C.numel() + sum(
                              x.numel() for x in s.abuf + s.bbuf)),
                          "sampled_entries_within_bound": ok, "samples": args.samples,
                          "worst_err_over_bound": float(np.max(np.abs(got - want) / bound))}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
