#!/usr/bin/env python
"""Config 4 (BASELINE configs[3]): m=n=k=16384, BF16 / TF32 inputs rounded
from uniform[-1,1), FP32 accumulate on tcgen05, C (fp32) = 0 initially.
Times the task kernel with CUDA events (warm-up 2, median of 5) and reports
TFLOP/s against MEASURED_PEAKS.json's bf16 figure (tf32: half of it, the
nominal dense ratio, stated)."""
from __future__ import annotations

import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


# L2-level block of the C2A1C0 plan (m x n); 1536 x 3072 = 72 SM-pair tiles, one wave
L2M, L2N = (int(x) for x in os.environ.get("TC_L2_BLOCK", "1536x3072").split("x"))


def main():
    import torch

    from paper_1904_05717_b200 import tilemul as T

    size = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"bf16_tflops": 1590.0}
    m = n = k = size
    hier1 = T.CacheHierarchy.from_capacities([128 * 512, 232448 // 2, 132644864 // 2])
    hier2 = T.CacheHierarchy.from_capacities([256 * 512, 232448, 132644864 // 2])  # 256x512 over an SM pair
    d = T.parse_name("C2A1C0")
    def plan(tile, tile_n=256):
        # one wave of pair tiles per L2 block: 6 x 12 of 256 x 256, 8 x 9 of 256 x 512
        l2m, l2n = (L2M, L2N) if tile_n == 256 else tuple(int(x) for x in os.environ.get("TC_L2_BLOCK_WIDE", "2048x2048").split("x"))
        hier = hier1 if tile_n == 256 else hier2
        bs = T.derive_blocksizes(d, hier, T.Shape(m, n, k), opts=T.DeriveOptions(micro=T.MicroTile(tile, tile_n)),
                                 pinned=T.BlocksizeSet({(1, "m"): tile, (2, "m"): l2m, (2, "n"): l2n}))
        return T.build_plan(d, bs, hier, T.Shape(m, n, k)), bs

    A64 = torch.empty(m * k, dtype=torch.float64, device="cuda")
    B64 = torch.empty(k * n, dtype=torch.float64, device="cuda")
    T.fill_uniform_device(A64, 1)
    T.fill_uniform_device(B64, 2)
    # live tcgen05 issue-rate peaks: bursts at full clocks, and ~200 ms launches under the power cap
    probe = {dt: T.measure_tc_peak(dt, 10) for dt in ("bf16", "tf32")}
    probe_sus = {dt: T.measure_tc_peak(dt, 3, sustained=True) for dt in ("bf16", "tf32")}
    cases = os.environ.get("TC_CASES", "bf16:256:512,bf16:256:256,bf16:128,tf32:256:512,tf32:256:256,tf32:128").split(",")
    for dtype, tile, tile_n in ((c.split(":")[0], int(c.split(":")[1]), int((c.split(":") + ["256"])[2])) for c in cases):
        nest, bs = plan(tile, tile_n)
        A = T.round_inputs(A64, dtype)
        B = T.round_inputs(B64, dtype)
        C = torch.zeros(m * n, dtype=torch.float32, device="cuda")
        for _ in range(2):
            T.execute_tc(nest, A, B, C, dtype, T.ExecOptions(tile=tile, tile_n=tile_n))
        torch.cuda.synchronize()
        ts = []
        import bench
        clk = bench.ClockSampler(0)
        clk.__enter__()
        for _ in range(40):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            T.execute_tc(nest, A, B, C, dtype, T.ExecOptions(tile=tile, tile_n=tile_n))
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        clk.__exit__(None, None, None)
        t = statistics.median(ts)
        tf = 2.0 * m * n * k / t / 1e12
        peak = peaks["bf16_tflops"] if dtype == "bf16" else peaks["bf16_tflops"] / 2
        print(json.dumps({"config": "config4", "dtype": dtype, "shape": [m, n, k], "seconds": t, "tflops": tf,
                          "peak_tflops": peak,
                          "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst)" + (" / 2 (nominal tf32:bf16 dense ratio)" if dtype == "tf32" else ""),
                          "frac": tf / peak, "probe_peak_tflops": probe[dtype], "frac_of_probe": tf / probe[dtype],
                          "probe_sustained_tflops": probe_sus[dtype], "frac_of_probe_sustained": tf / probe_sus[dtype],
                          "probe_source": "tm_measure_tc_peak: one CTA per SM issuing 128x256 tcgen05.mma back to back "
                                          "(cta_group::1), same clocks/power state as this run",
                          "frac_of_sustained": tf / (peaks.get("bf16_tflops_sustained", peak * 2) /
                                                    (1 if dtype == "bf16" else 2)),
                          "cta_tile": (f"256x{tile_n} per SM pair (cta_group::2)" if tile == 256 else "128x256 (cta_group::1)"),
                          "blocksizes": {f"{lv}:{dd}": v for (lv, dd), v in bs.entries()},
                          "launch": nest.last_launch(), "clocks": clk.summary()}), flush=True)
        del A, B, C
    # cuBLAS at the same shape in the same process and power state (library
    # reference, not our path): bf16 in/out (torch.matmul), tf32 in / fp32 out
    if os.environ.get("TC_CUBLAS", "1") == "1":
        import bench

        for dtype in ("bf16", "tf32"):
            torch.backends.cuda.matmul.allow_tf32 = dtype == "tf32"
            dt = torch.bfloat16 if dtype == "bf16" else torch.float32
            X = A64.view(k, m).t().to(dt)
            Y = B64.view(n, k).t().to(dt)
            for _ in range(2):
                Z = X @ Y
            torch.cuda.synchronize()
            ts = []
            clk = bench.ClockSampler(0)
            clk.__enter__()
            for _ in range(40):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                Z = X @ Y
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e-3)
            clk.__exit__(None, None, None)
            t = statistics.median(ts)
            print(json.dumps({"config": "config4", "impl": "cuBLAS (torch.matmul) reference", "dtype": dtype,
                              "shape": [m, n, k], "seconds": t, "tflops": 2.0 * m * n * k / t / 1e12,
                              "output": "bf16" if dtype == "bf16" else "fp32", "clocks": clk.summary()}), flush=True)
            if dtype == "bf16":
                # the same contract as ours: fp32 C += A·B from bf16 inputs (beta = 1, fp32 out)
                C32 = torch.zeros(m, n, dtype=torch.float32, device="cuda")
                for _ in range(2):
                    Z = torch.addmm(C32, X, Y, out_dtype=torch.float32)
                torch.cuda.synchronize()
                ts = []
                clk = bench.ClockSampler(0)
                clk.__enter__()
                for _ in range(40):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    Z = torch.addmm(C32, X, Y, out_dtype=torch.float32)
                    e1.record()
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1) * 1e-3)
                clk.__exit__(None, None, None)
                t = statistics.median(ts)
                print(json.dumps({"config": "config4", "impl": "cuBLAS (torch.addmm out_dtype=fp32) reference",
                                  "dtype": dtype, "shape": [m, n, k], "seconds": t,
                                  "tflops": 2.0 * m * n * k / t / 1e12, "output": "fp32 C + A·B (beta 1)",
                                  "clocks": clk.summary()}), flush=True)
                del C32
            del X, Y, Z


if __name__ == "__main__":
    main()
