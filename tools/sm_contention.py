#!/usr/bin/env python
"""Evidence for the multi-GPU exchange design: while the
persistent FP64 task kernel holds every SM (148 CTAs x 512 threads x 128
registers = each SM's whole register file), can an exchange run under it?

  * copy engine: a 1 GiB cudaMemcpyAsync (tilemul.copy_async) on a side stream
  * SM kernel:   a 1 GiB elementwise copy kernel (torch add) on a side stream,
                 standing in for an NCCL broadcast kernel (which also needs SMs)

Both are issued right after the GEMM launch; CUDA events on each stream give
their start/end relative to the GEMM's. Prints one JSON line.

    python tools/sm_contention.py [--size 8192]
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
    ap.add_argument("--size", type=int, default=8192)
    ap.add_argument("--copy-gib", type=float, default=1.0)
    a = ap.parse_args()
    import torch

    import bench
    from paper_1904_05717_b200 import tilemul as T

    m = n = k = a.size
    nest, _, _ = bench.make_plan(T, m, n, k)
    A = torch.empty(m * k, dtype=torch.float64, device="cuda")
    B = torch.empty(k * n, dtype=torch.float64, device="cuda")
    C = torch.empty(m * n, dtype=torch.float64, device="cuda")
    for x, s in zip((A, B, C), (1, 2, 3)):
        T.fill_uniform_device(x, s)
    nel = int(a.copy_gib * 2 ** 30) // 8
    src = torch.ones(nel, dtype=torch.float64, device="cuda")
    dst = torch.empty_like(src)
    opts = T.ExecOptions(split_k=0)
    main_s = torch.cuda.current_stream()
    side = torch.cuda.Stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def one(kind):
        torch.cuda.synchronize()
        g0, g1, s0, s1 = ev(), ev(), ev(), ev()
        g0.record(main_s)
        T.execute(nest, A, B, C, opts)
        g1.record(main_s)
        if kind != "none":
            with torch.cuda.stream(side):
                side.wait_event(g0)  # issued after the GEMM has started
                s0.record(side)
                if kind == "copy_engine":
                    T.copy_async(dst.data_ptr(), src.data_ptr(), nel * 8, side)
                else:
                    torch.add(src, 0.0, out=dst)
                s1.record(side)
        torch.cuda.synchronize()
        r = {"gemm_ms": g0.elapsed_time(g1)}
        if kind != "none":
            r.update(side_start_ms=g0.elapsed_time(s0), side_end_ms=g0.elapsed_time(s1),
                     side_ms=s0.elapsed_time(s1))
        return r

    for _ in range(3):
        one("none")
    alone = [one("none") for _ in range(3)]
    ce = [one("copy_engine") for _ in range(3)]
    sm = [one("sm_kernel") for _ in range(3)]
    # the side work alone
    torch.cuda.synchronize()
    e0, e1 = ev(), ev()
    e0.record()
    T.copy_async(dst.data_ptr(), src.data_ptr(), nel * 8, main_s)
    e1.record()
    torch.cuda.synchronize()
    ce_alone = e0.elapsed_time(e1)
    e0.record()
    torch.add(src, 0.0, out=dst)
    e1.record()
    torch.cuda.synchronize()
    sm_alone = e0.elapsed_time(e1)
    print(json.dumps({
        "probe": "exchange under the persistent FP64 GEMM", "gemm_shape": [m, n, k], "side_bytes": nel * 8,
        "gemm_alone": alone, "with_copy_engine": ce, "with_sm_kernel": sm,
        "copy_engine_alone_ms": ce_alone, "sm_kernel_alone_ms": sm_alone,
        "reading": "side_end_ms < gemm_ms: the exchange finished under the GEMM; side_start_ms ~ gemm_ms: it "
                   "waited for the GEMM's SMs",
    }))


if __name__ == "__main__":
    main()
