#!/usr/bin/env python
"""Measured vs modelled traffic per case (CPU half; the GPU half is
tools/model_cases.py under ncu).

  python tools/model_check.py gpurun_out/mc.jsonl gpurun_out/mc.csv > profiles/model_check_r02.json

Per case, three numbers at each level:
  measured   ncu: dram__bytes_{read,write} (HBM boundary); 32 B x
             lts__t_sectors_srcunit_tex_op_{read,write} (L2 <-> SM)
  gpu model  LoopNest.gpu_model of the same plan and options: the schedule's
             own task list -- FIFO-SMEM traffic exact over the tasks, HBM
             bytes from a lockstep run through an LRU of the physical L2
  reference  multilevel_cost (costmodel.hpp:163-229) of the same plan on the
             derived hierarchy it was planned with
The models are recomputed here (no GPU needed) from the recorded plan.
"""
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
        "s": 1.0, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "sector": 1.0}


def launches_of(csv_path):
    lines = [ln for ln in open(csv_path) if not ln.startswith("==")]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    h = rows[0]
    ki, ni, vi, ui = h.index("ID"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    kn = h.index("Kernel Name")
    per = {}
    for r in rows[1:]:
        v = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
        d = per.setdefault(int(r[ki]), {"kernel": r[kn]})
        d[r[ni]] = v
    return [per[k] for k in sorted(per)]


def main():
    from paper_1904_05717_b200 import tilemul as T

    recs = [json.loads(ln) for ln in open(sys.argv[1]) if ln.strip()]
    recs = [r for r in recs if "error" not in r]
    launches = launches_of(sys.argv[2])
    want = sum(int(r["launch"]["launches"]) for r in recs)
    if want != len(launches):
        raise SystemExit(f"{len(launches)} profiled launches vs {want} expected over {len(recs)} cases")
    out, at = [], 0
    for r in recs:
        nl = int(r["launch"]["launches"])
        g = {}
        for mm in launches[at:at + nl]:
            for key, v in mm.items():
                if key != "kernel":
                    g[key] = g.get(key, 0.0) + v
        at += nl
        shape = T.Shape(*r["shape"])
        hier = T.CacheHierarchy.from_capacities(r["hierarchy"])
        bs = T.BlocksizeSet({(lv, d): v for lv, d, v in r["blocksizes"]})
        nest = T.build_plan(T.parse_name(r["family"]), bs, hier, shape)
        opts = T.ExecOptions(schedule=r["schedule"], split_k=r["split_k"], staging=r["staging"])
        sms, _, l2 = r["facts"]
        gm = nest.gpu_model(opts, sms=sms, l2_bytes=l2)
        ref = nest.model()
        dram = g["dram__bytes_read.sum"] + g["dram__bytes_write.sum"]
        l2sm = 32.0 * (g["lts__t_sectors_srcunit_tex_op_read.sum"] + g["lts__t_sectors_srcunit_tex_op_write.sum"])
        o = {"config": r["config"], "shape": r["shape"], "family": r["family"], "schedule": r["schedule"],
             "split_k": r["split_k"], "staging": r["staging"], "launch": r["launch"],
             "blocksizes": {f"{lv}:{d}": v for lv, d, v in r["blocksizes"]},
             "hbm_measured": dram, "hbm_gpu_model": gm["hbm_total_bytes"],
             "hbm_ref_model": ref.at_level(2).total_bytes(),
             "hbm_over_gpu_model": dram / gm["hbm_total_bytes"],
             "hbm_over_ref_model": dram / ref.at_level(2).total_bytes(),
             "smem_level_measured": l2sm, "smem_gpu_model": gm["smem_bytes"],
             "smem_ref_model": ref.at_level(1).total_bytes(),
             "smem_over_gpu_model": l2sm / gm["smem_bytes"],
             "smem_over_ref_model": l2sm / ref.at_level(1).total_bytes(),
             "kernel_seconds_under_ncu": g.get("gpu__time_duration.sum")}
        out.append(o)
    json.dump({"kernel_id": sys.argv[3] if len(sys.argv) > 3 else None, "cases": out}, sys.stdout, indent=1)
    print()
    for o in out:
        print(f"{o['config']:9s} {str(o['shape']):22s} {o['family']:7s} {o['schedule']:8s} sk={o['split_k']:2d} "
              f"{o['staging']:7s} HBM {o['hbm_measured'] / 1e9:8.3f} GB: /gpu {o['hbm_over_gpu_model']:5.2f}x "
              f"/ref {o['hbm_over_ref_model']:5.2f}x   L2<->SM {o['smem_level_measured'] / 1e9:8.2f} GB: "
              f"/gpu {o['smem_over_gpu_model']:5.2f}x /ref {o['smem_over_ref_model']:5.2f}x", file=sys.stderr)


if __name__ == "__main__":
    main()
