#!/usr/bin/env python
"""Per-CTA timeline of the FP64 TMA task kernel (experiment build with -DTM_TRACE).

  tools/build_variant.sh trace "-DTM_TRACE"
  TILEMUL_B200_LIB=exp_libs/trace.so python tools/cta_timeline.py --shape 2048,2048,2048 --out gpurun_out/tl_c1.json

Thread 0 of every CTA stamps task-boundary events (dgemm_sm100.cu TM_TRACE_EV):
0 kernel start, 1 task start, 2 C loaded into registers (issued), 3 first slab
landed, 4 k loop done, 5 split-k partials folded, 6 tile written, 7 CTA done.
The report splits each CTA's time into those phases (SM clock cycles) and
compares the k loop against the DMMA issue bound (64 FMA/clk/SM).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

PHASES = [("prologue_c_load", 1, 2), ("first_slab_wait", 2, 3), ("k_loop", 3, 4), ("fold", 4, 5), ("store", 5, 6)]


def read_trace(lib):
    nc, ne = ctypes.c_int(), ctypes.c_int()
    lib.tm_trace_dims(ctypes.byref(nc), ctypes.byref(ne))
    buf = (ctypes.c_ulonglong * (nc.value * ne.value * 3))()
    cnt = (ctypes.c_int * nc.value)()
    assert lib.tm_trace_read(buf, cnt) == 0
    out = []
    for c in range(nc.value):
        n = min(cnt[c], ne.value)
        ev = []
        for i in range(n):
            b = (c * ne.value + i) * 3
            ev.append((buf[b], buf[b + 1], buf[b + 2] & 0xFF, buf[b + 2] >> 8))
        out.append(ev)
    return out


def analyse(trace, tile_fma_per_slab):
    ctas = [t for t in trace if t]
    g0 = min(t[0][0] for t in ctas)
    g1 = max(t[-1][0] for t in ctas)
    tot = {p: 0 for p, _, _ in PHASES}
    tot["between_tasks"] = 0
    tot["cta_start_to_first_task"] = 0
    slabs_cycles = []
    per_cta = []
    for t in ctas:
        span = t[-1][1] - t[0][1]
        ph = {p: 0 for p, _, _ in PHASES}
        ph["between_tasks"] = 0
        by_task = {}
        order = []
        for gt, ck, e, ti in t:
            if e in (1, 2, 3, 4, 5, 6):
                if ti not in by_task:
                    by_task[ti] = {}
                    order.append(ti)
                by_task[ti][e] = ck
        ph["cta_start_to_first_task"] = by_task[order[0]][1] - t[0][1] if order else 0
        for j, ti in enumerate(order):
            d = by_task[ti]
            for p, a, b in PHASES:
                if a in d and b in d:
                    ph[p] += d[b] - d[a]
            if j + 1 < len(order) and 6 in d:
                ph["between_tasks"] += by_task[order[j + 1]][1] - d[6]
        ph["tail_after_last_task"] = t[-1][1] - by_task[order[-1]].get(6, t[-1][1]) if order else 0
        per_cta.append({"span_cycles": span, "tasks": len(order), "start_ns": t[0][0] - g0, "end_ns": t[-1][0] - g0,
                        **ph})
        for k in tot:
            tot[k] += ph.get(k, 0)
    n = len(per_cta)
    avg = {k: v / n for k, v in tot.items()}
    avg["span_cycles"] = sum(c["span_cycles"] for c in per_cta) / n
    return {"ctas": n, "kernel_ns": g1 - g0, "avg_cycles": avg,
            "start_ns_max": max(c["start_ns"] for c in per_cta),
            "end_ns_min": min(c["end_ns"] for c in per_cta),
            "end_ns_max": max(c["end_ns"] for c in per_cta),
            "per_cta": per_cta}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="2048,2048,2048")
    ap.add_argument("--family", default="C2A1C0")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--split", type=int, default=0, help="split_k (0 = auto, as bench.py)")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import torch
    from paper_1904_05717_b200 import _native, planner, tilemul as T

    lib = ctypes.CDLL(_native.LIB_PATH)
    m, n, k = (int(x) for x in a.shape.split(","))
    _, bs, hier = planner.plan_for_gpu(a.family, (m, n, k))
    nest = T.build_plan(T.parse_name(a.family), bs, hier, T.Shape(m, n, k))
    A = torch.empty(k, m, dtype=torch.float64, device="cuda").t()
    B = torch.empty(n, k, dtype=torch.float64, device="cuda").t()
    C = torch.empty(n, m, dtype=torch.float64, device="cuda").t()
    for x, s in ((A, 1), (B, 2), (C, 3)):
        T.fill_uniform_device(x, s)
    opts = T.ExecOptions(numerics="dmma", split_k=a.split)
    runs = []
    for r in range(a.reps + 1):
        read_trace(lib)  # reset
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        T.execute(nest, A, B, C, opts)
        e1.record()
        torch.cuda.synchronize()
        tr = read_trace(lib)
        if r == 0:
            continue
        res = analyse(tr, 0)
        res["event_ms"] = e0.elapsed_time(e1)
        res["tflops"] = 2.0 * m * n * k / (res["event_ms"] * 1e-3) / 1e12
        res["launch"] = nest.last_launch()
        res["ideal_dmma_cycles_per_cta"] = m * n * k / 64.0 / res["ctas"]
        runs.append(res)
        av = res["avg_cycles"]
        print(json.dumps({"shape": a.shape, "event_ms": round(res["event_ms"], 4), "tflops": round(res["tflops"], 2),
                          "kernel_ns": res["kernel_ns"], "start_ns_max": res["start_ns_max"],
                          "end_ns_min": res["end_ns_min"], "end_ns_max": res["end_ns_max"], "ideal_dmma_cycles_per_cta": round(res["ideal_dmma_cycles_per_cta"]),
                          "avg_cycles": {k: round(v) for k, v in av.items()}}))
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"shape": a.shape, "runs": runs}, f)


if __name__ == "__main__":
    main()
