#!/usr/bin/env python
"""Config 4 under sustained load: our tcgen05 kernels and cuBLAS at the same
shape, each run back to back for ~3 s while NVML samples SM clock and board
power every 20 ms. Reports TF/s, median clock, median power and joules per
PFLOP -- the energy-per-flop comparison behind the power-capped numbers."""
from __future__ import annotations

import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


class Nvml:
    def __init__(self, index=0):
        import pynvml as N

        self.N = N
        N.nvmlInit()
        self.h = N.nvmlDeviceGetHandleByIndex(index)
        self.samples = []
        self.stop = False

    def run(self):
        N = self.N
        while not self.stop:
            self.samples.append((N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM),
                                 N.nvmlDeviceGetPowerUsage(self.h) / 1000.0))
            time.sleep(0.02)

    def __enter__(self):
        self.t = threading.Thread(target=self.run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *e):
        self.stop = True
        self.t.join()


def main():
    import torch

    import tools.bench_tc as btc  # noqa: F401  (same plan helper path)
    from paper_1904_05717_b200 import tilemul as T

    m = n = k = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    hier1 = T.CacheHierarchy.from_capacities([128 * 512, 232448 // 2, 132644864 // 2])
    hier2 = T.CacheHierarchy.from_capacities([256 * 512, 232448, 132644864 // 2])  # 256x512 over an SM pair
    d = T.parse_name("C2A1C0")

    def plan(tile, tile_n=256):
        l2m, l2n = (btc.L2M, btc.L2N) if tile_n == 256 else (2048, 4608)
        hier = hier1 if tile_n == 256 else hier2
        bs = T.derive_blocksizes(d, hier, T.Shape(m, n, k), opts=T.DeriveOptions(micro=T.MicroTile(tile, tile_n)),
                                 pinned=T.BlocksizeSet({(1, "m"): tile, (2, "m"): l2m, (2, "n"): l2n}))
        return T.build_plan(d, bs, hier, T.Shape(m, n, k))

    A64 = torch.empty(m * k, dtype=torch.float64, device="cuda")
    B64 = torch.empty(k * n, dtype=torch.float64, device="cuda")
    T.fill_uniform_device(A64, 1)
    T.fill_uniform_device(B64, 2)
    A = T.round_inputs(A64, "bf16")
    B = T.round_inputs(B64, "bf16")
    C = torch.zeros(m * n, dtype=torch.float32, device="cuda")
    X = A64.view(k, m).t().to(torch.bfloat16)
    Y = B64.view(n, k).t().to(torch.bfloat16)
    cases = []
    for tile, tile_n in ((256, 512), (256, 256), (128, 256)):
        nest = plan(tile, tile_n)
        cases.append((f"ours bf16 tile {tile}x{tile_n}", lambda nest=nest, tile=tile, tile_n=tile_n: T.execute_tc(
            nest, A, B, C, "bf16", T.ExecOptions(tile=tile, tile_n=tile_n))))
    cases.append(("cuBLAS bf16 (torch.matmul, bf16 out)", lambda: X @ Y))
    for name, f in cases:
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        time.sleep(2.0)  # cool down between cases
        iters = 0
        with Nvml() as nv:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            t0 = time.perf_counter()
            while time.perf_counter() - t0 < 3.0:
                for _ in range(20):
                    f()
                iters += 20
                torch.cuda.synchronize()
            e1.record()
            torch.cuda.synchronize()
        sec = e0.elapsed_time(e1) * 1e-3
        tf = 2.0 * m * n * k * iters / sec / 1e12
        clk = statistics.median(s[0] for s in nv.samples)
        pw = statistics.median(s[1] for s in nv.samples)
        print(json.dumps({"case": name, "tflops": tf, "sm_mhz_median": clk, "power_w_median": pw,
                          "joules_per_pflop": pw / tf * 1e3, "samples": len(nv.samples)}), flush=True)


if __name__ == "__main__":
    main()
