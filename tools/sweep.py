#!/usr/bin/env python
"""Config sweep on one B200: every BASELINE.json FP64 config shape, each
MOMMS family member that is expressible on the GPU hierarchy, timed with CUDA
events (warm-up 2, median of 3), with the member's modelled traffic per level
(multilevel_cost on {CTA tile, SMEM, L2}).

  python tools/sweep.py [--quick] [--once] > profiles/sweep_rNN.jsonl

--once: each case launches its kernel exactly once (no warm-up, no timing) so
an `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:k_dmma`
pass over this command yields one measured-bytes row per case, in order.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

MEMBERS_L2L1 = ["C2A1C0", "B2A1C0", "A2B1C0", "C2B1C0"]
MEMBERS_L2 = ["A2C0", "B2C0"]


def cases(quick: bool):
    out = [("config1", (2048, 2048, 2048), ["C2A1C0"], {"c_zero": True}),
           ("config1_no_split", (2048, 2048, 2048), ["C2A1C0"], {"c_zero": True, "split_k": 1})]
    sizes = [4096, 8192] if quick else [4096, 8192, 16384]
    for s in sizes:
        out.append(("config2", (s, s, s), MEMBERS_L2L1 + MEMBERS_L2, {}))
    out.append(("config3a_rank_k", (16384, 16384, 256), ["C2A1C0", "A2C0", "B2C0"], {}))
    out.append(("config3b_inner_product", (512, 512, 131072), ["C2A1C0", "C2B1C0"], {"split_k": 0}))
    out.append(("config3c_panel_panel", (65536, 256, 1024), ["B2A1C0", "C2A1C0", "B2C0"], {}))
    return out


L2_FRAC = 1.0


def plan_for(T, name, shape, tile=128):
    hier = T.gpu_hierarchy(tile)
    if L2_FRAC != 1.0:  # model an effective L2 capacity (fraction of the physical one) for residency
        caps = [hier.capacity(i) for i in range(hier.size())]
        caps[-1] = int(caps[-1] * L2_FRAC)
        hier = T.CacheHierarchy.from_capacities(caps)
    d = T.parse_name(name)
    pins = {}
    lv1 = d.plan_at(1)
    if lv1 is not None:  # the SMEM-level block must hold whole register tiles along the tile dims
        for dim in (lv1.outer_dim, lv1.inner_dim):
            if dim in ("m", "n"):
                pins[(1, dim)] = min(tile, shape[0] if dim == "m" else shape[1])
    opts = T.DeriveOptions(micro=T.MicroTile(tile, tile))
    try:
        bs = T.derive_blocksizes(d, hier, T.Shape(*shape), opts=opts, pinned=T.BlocksizeSet(pins))
    except T.InfeasibleError:
        # The reference's shrink keeps the L2 block's aspect ratio, so a
        # skipped SMEM level (guest panel k x n_r must fit it) squeezes the
        # block's m/n side below one register tile. Pin that side to a
        # wave-sized extent (12 tiles) and derive the rest.
        top = d.plans[0]
        for dim in (top.outer_dim, top.inner_dim):
            if dim in ("m", "n"):
                pins[(top.level, dim)] = min(12 * tile, shape[0] if dim == "m" else shape[1])
        bs = T.derive_blocksizes(d, hier, T.Shape(*shape), opts=opts, pinned=T.BlocksizeSet(pins))
    return T.build_plan(d, bs, hier, T.Shape(*shape)), bs, hier


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--once", action="store_true")
    ap.add_argument("--schedules", default="fused")
    ap.add_argument("--faithful-par", default="default", choices=["default", "outer"],
                    help="faithful: plain nest order, or the deepest m/n loop above the innermost k loop split into "
                         "workers (faster, not traffic-faithful)")
    ap.add_argument("--tiles", default="auto,128x128,128x64")
    ap.add_argument("--only", default="", help="comma-separated config names to run (default: all)")
    ap.add_argument("--members", default="", help="comma-separated family members (default: per config)")
    ap.add_argument("--staging", default="auto", choices=["auto", "cpasync", "tma"],
                    help="DMMA kernels: how A/B k-slabs reach shared memory")
    ap.add_argument("--l2-frac", type=float, default=1.0, help="effective L2 capacity fraction for derivation")
    a = ap.parse_args()
    import torch

    from paper_1904_05717_b200 import tilemul as T

    peak = None if a.once else T.measure_fp64_peak(20)
    only = set(x for x in a.only.split(",") if x)
    global L2_FRAC
    L2_FRAC = a.l2_frac
    keep = [x for x in a.members.split(",") if x]
    for cfg, shape, members, extra in cases(a.quick):
        if only and cfg not in only:
            continue
        m, n, k = shape
        A = torch.empty(m * k, dtype=torch.float64, device="cuda")
        B = torch.empty(k * n, dtype=torch.float64, device="cuda")
        C = torch.empty(m * n, dtype=torch.float64, device="cuda")
        T.fill_uniform_device(A, 1)
        T.fill_uniform_device(B, 2)
        for name in (keep or members):
            for sched, tile in [(sc, tl) for sc in a.schedules.split(",") for tl in a.tiles.split(",")]:
                if sched == "faithful" and tile != a.tiles.split(",")[0]:
                    continue
                tm, tn = (0, 0) if tile == "auto" else (int(x) for x in tile.split("x"))
                rec = {"config": cfg, "shape": shape, "family": name, "schedule": sched, "cta_tile": tile,
                       "l2_frac": L2_FRAC}
                try:
                    nest, bs, hier = plan_for(T, name, shape)
                except Exception as e:  # infeasible on this hierarchy: reported, not hidden
                    rec["error"] = f"{type(e).__name__}: {e}"
                    print(json.dumps(rec), flush=True)
                    continue
                if extra.get("c_zero"):
                    C.zero_()
                else:
                    T.fill_uniform_device(C, 3)
                par = -1
                if sched == "faithful" and a.faithful_par == "outer":
                    dims = [L.dim for L in nest.loops]
                    kin = max((i for i, d in enumerate(dims) if d == "k"), default=-1)
                    par = max((i for i in range(kin) if dims[i] != "k"), default=-1)
                    rec["parallel_loop"] = par
                opts = T.ExecOptions(numerics="dmma", schedule=sched, split_k=extra.get("split_k", 0), tile=tm,
                                     tile_n=tn, parallel_loop=par, staging=a.staging)
                rep = nest.model()
                rec["blocksizes"] = {f"{lv}:{d}": v for (lv, d), v in bs.entries()}
                rec["model_bytes"] = {f"L{lt.level}": lt.total_bytes() for lt in rep.levels}
                rec["cells"] = nest.cell_count()
                if sched == "faithful" and rec["cells"] > 4_000_000:
                    rec["error"] = "faithful schedule skipped: too many cells for a timed run"
                    print(json.dumps(rec), flush=True)
                    continue
                if a.once:
                    opts.split_k = 1 if extra.get("split_k", 0) == 0 and sched == "fused" and cfg != "config3b_inner_product" else opts.split_k
                    T.execute(nest, A, B, C, opts)
                    torch.cuda.synchronize()
                    rec["launch"] = nest.last_launch()
                    print(json.dumps(rec), flush=True)
                    continue
                for _ in range(2):
                    T.execute(nest, A, B, C, opts)
                torch.cuda.synchronize()
                times = []
                for _ in range(3):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    T.execute(nest, A, B, C, opts)
                    e1.record()
                    torch.cuda.synchronize()
                    times.append(e0.elapsed_time(e1) * 1e-3)
                t = statistics.median(times)
                tf = 2.0 * m * n * k / t / 1e12
                rec.update({"seconds": t, "tflops": tf, "pct_fp64_peak": 100.0 * tf / peak, "peak_tflops": peak,
                            "launch": nest.last_launch()})
                print(json.dumps(rec), flush=True)
        del A, B, C
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
