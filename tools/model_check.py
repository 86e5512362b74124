#!/usr/bin/env python
"""Measured vs modelled traffic per family member (the MOMMS I/O model,
costmodel.hpp:163-229, on the B200 hierarchy {CTA tile, SMEM, L2}).

GPU step (under ncu, one launch per case):
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,\\
lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,gpu__time_duration.sum \\
      -k regex:k_dmma --csv --log-file gpurun_out/model_check.csv python tools/sweep.py --once ... \\
      > gpurun_out/model_check.jsonl
CPU step (here):
  python tools/model_check.py gpurun_out/model_check.jsonl gpurun_out/model_check.csv > profiles/model_check_r01.json

HBM level: measured dram bytes vs modelled bytes into L2 (level 2).
SMEM level: measured L2<->SM bytes (32-byte sectors read + written by the
SMs) vs modelled bytes into level 1 (A/B staging + C, which moves between L2
and the register tile directly).
"""
import csv
import io
import json
import sys


def main():
    recs = [json.loads(l) for l in open(sys.argv[1]) if l.strip()]
    recs = [r for r in recs if "error" not in r]
    lines = [l for l in open(sys.argv[2]) if not l.startswith("==")]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    h = rows[0]
    ki, ni, vi, ui = h.index("ID"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    per = {}
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        mult = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6,
                "ms": 1e-3, "s": 1.0, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}.get(u, 1.0)
        per.setdefault(int(r[ki]), {})[r[ni]] = v * mult
    launches = [per[k] for k in sorted(per)]
    if len(launches) != len(recs):
        # a case may be several task-kernel launches (TMA segments): group them by the case's launch count
        want = sum(int(r.get("launch", {}).get("launches", 1)) for r in recs)
        if want != len(launches):
            raise SystemExit(f"{len(launches)} profiled launches vs {len(recs)} cases ({want} launches)")
        grouped, at = [], 0
        for r in recs:
            nl = int(r.get("launch", {}).get("launches", 1))
            g = {}
            for m in launches[at:at + nl]:
                for key, v in m.items():
                    g[key] = g.get(key, 0.0) + v
            grouped.append(g)
            at += nl
        launches = grouped
    out = []
    for rec, m in zip(recs, launches):
        dram = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
        l2sm = 32.0 * (m["lts__t_sectors_srcunit_tex_op_read.sum"] + m["lts__t_sectors_srcunit_tex_op_write.sum"])
        mb = rec["model_bytes"]
        out.append({"config": rec["config"], "shape": rec["shape"], "family": rec["family"],
                    "schedule": rec["schedule"], "blocksizes": rec["blocksizes"],
                    "hbm_measured": dram, "hbm_model": mb["L2"], "hbm_ratio": dram / mb["L2"],
                    "smem_level_measured": l2sm, "smem_level_model": mb["L1"], "smem_ratio": l2sm / mb["L1"],
                    "kernel_seconds_under_ncu": m.get("gpu__time_duration.sum")})
    json.dump(out, sys.stdout, indent=1)
    print()
    for o in out:
        print(f"{o['config']:22s} {str(o['shape']):20s} {o['family']} {o['schedule']:8s} "
              f"HBM {o['hbm_measured']/1e9:8.3f}/{o['hbm_model']/1e9:8.3f} GB = {o['hbm_ratio']:5.2f}x   "
              f"L2<->SM {o['smem_level_measured']/1e9:8.2f}/{o['smem_level_model']/1e9:8.2f} GB = "
              f"{o['smem_ratio']:5.2f}x", file=sys.stderr)


if __name__ == "__main__":
    main()
