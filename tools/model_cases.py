#!/usr/bin/env python
"""GPU half of the model check (tools/model_check.py): runs each case's
execute() exactly once so an ncu metrics pass over this command yields the
measured DRAM and L2<->SM bytes of every case, in order.

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,\\
lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,gpu__time_duration.sum \\
      -k regex:"k_dmma|k_reduce" --csv --log-file gpurun_out/mc.csv \\
      python tools/model_cases.py > gpurun_out/mc.jsonl

Plans come from planner.plan_for_gpu (the bench's derived hierarchy); one
JSON line per case with the plan, the options and the launches it issued.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

MEMBERS = ["C2A1C0", "C2B1C0", "B2A1C0", "A2B1C0", "A2C0", "B2C0"]


def cases(quick=False):
    out = [("config1", (2048, 2048, 2048), "C2A1C0", "fused", 0, "auto"),
           ("config1", (2048, 2048, 2048), "C2A1C0", "fused", 1, "auto")]
    for s in ((4096, 8192) if quick else (4096, 8192, 16384)):
        for name in MEMBERS:
            out.append(("config2", (s, s, s), name, "fused", 0, "auto"))
        out.append(("config2", (s, s, s), "C2A1C0", "fused", 1, "auto"))
        out.append(("config2", (s, s, s), "C2A1C0", "fused", 0, "cpasync"))
    for name in ("C2A1C0", "A2B1C0", "B2C0"):
        out.append(("config3a", (16384, 16384, 256), name, "fused", 0, "auto"))
    out.append(("config3b", (512, 512, 131072), "C2A1C0", "fused", 0, "auto"))
    for name in ("B2A1C0", "C2A1C0"):
        out.append(("config3c", (65536, 256, 1024), name, "fused", 0, "auto"))
    for s in (4096, 8192):
        for name in ("C2A1C0", "C2B1C0", "B2A1C0", "A2B1C0"):
            out.append(("config2", (s, s, s), name, "faithful", 1, "auto"))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    import torch

    from paper_1904_05717_b200 import planner as P
    from paper_1904_05717_b200 import tilemul as T

    facts = P.device_facts()
    cur = None
    for cfg, shape, name, sched, split, staging in cases(a.quick):
        m, n, k = shape
        if cur != shape:
            A = B = C = None
            torch.cuda.empty_cache()
            A = torch.empty(m * k, dtype=torch.float64, device="cuda")
            B = torch.empty(k * n, dtype=torch.float64, device="cuda")
            C = torch.empty(m * n, dtype=torch.float64, device="cuda")
            T.fill_uniform_device(A, 1)
            T.fill_uniform_device(B, 2)
            cur = shape
        T.fill_uniform_device(C, 3)
        rec = {"config": cfg, "shape": list(shape), "family": name, "schedule": sched, "split_k": split,
               "staging": staging, "facts": list(facts)}
        try:
            nest, bs, hier = P.plan_for_gpu(name, shape, sched, facts=facts)
        except Exception as e:  # infeasible on this hierarchy: reported, not hidden
            rec["error"] = f"{type(e).__name__}: {e}"
            print(json.dumps(rec), flush=True)
            continue
        rec["blocksizes"] = [[lv, d, v] for (lv, d), v in bs.entries()]
        rec["hierarchy"] = [hier.capacity(i) for i in range(hier.size())]
        torch.cuda.synchronize()
        T.execute(nest, A, B, C, T.ExecOptions(schedule=sched, split_k=split, staging=staging))
        torch.cuda.synchronize()
        rec["launch"] = nest.last_launch()
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
