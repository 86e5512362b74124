#!/usr/bin/env python
"""Host-buffer (e2e) pipeline probe at the bench workload: pinned copy
bandwidths, the device-resident GEMM time, and tm_execute_host (pinned A, B,
C in, C out) -- the gap between the last two is what the copy-engine-fed
pipeline leaves exposed."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1904_05717_b200 import tilemul as T  # noqa: E402


def t(f):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f()
    torch.cuda.synchronize()
    return time.perf_counter() - t0


def main():
    nb = 2 * 1024 ** 3 // 8
    h = torch.empty(nb, dtype=torch.float64).pin_memory()
    d = torch.empty(nb, dtype=torch.float64, device="cuda")
    d.copy_(h, non_blocking=True)
    print(json.dumps({"h2d_GBps": 2 * 1024 ** 3 / t(lambda: d.copy_(h, non_blocking=True)) / 1e9,
                      "d2h_GBps": 2 * 1024 ** 3 / t(lambda: h.copy_(d, non_blocking=True)) / 1e9}), flush=True)
    del h, d
    m = n = k = int(os.environ.get("SIZE", "16384"))
    nest, bs, hier = bench.make_plan(T, m, n, k)
    opts = T.ExecOptions(numerics="dmma", schedule="fused", split_k=0)
    Ad = torch.full((m * k,), 0.5, dtype=torch.float64, device="cuda")
    Bd = torch.full((k * n,), 0.25, dtype=torch.float64, device="cuda")
    Cd = torch.zeros(m * n, dtype=torch.float64, device="cuda")
    T.execute(nest, Ad, Bd, Cd, opts)
    print(json.dumps({"device_ms": min(t(lambda: T.execute(nest, Ad, Bd, Cd, opts)) for _ in range(3)) * 1e3}), flush=True)
    del Ad, Bd, Cd
    A = torch.empty(m * k, dtype=torch.float64).pin_memory().numpy()
    B = torch.empty(k * n, dtype=torch.float64).pin_memory().numpy()
    C = torch.empty(m * n, dtype=torch.float64).pin_memory().numpy()
    A[:] = 0.5
    B[:] = 0.25
    C[:] = 0.0
    T.execute(nest, A, B, C, opts)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        T.execute(nest, A, B, C, opts)
        ts.append(time.perf_counter() - t0)
    print(json.dumps({"e2e_ms": min(ts) * 1e3, "launches": nest.last_launch()["launches"],
                      "tasks": nest.last_launch()["tasks"]}), flush=True)


if __name__ == "__main__":
    main()
