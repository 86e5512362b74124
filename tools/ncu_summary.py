#!/usr/bin/env python
"""Summarise an ncu --set full capture (.ncu-rep) and an ncu launch list
(--metrics gpu__time_duration.sum --csv) into profiles/ncu_summary_<tag>.json.

  python tools/ncu_summary.py --rep gpurun_out/prof.ncu-rep --launches gpurun_out/launches.csv \
      --workload "<bench workload string>" --tag r02_x --launches-per-step 14 [--flops F] [--model-bytes B]

Per-step figures (dram_bytes_per_step, ...) sum the first --launches-per-step
task-kernel launches of the capture (capture exactly one step's launches);
the summary is stamped with the library build id, and bench.py only uses its
bytes when that id equals the loaded library's.

Run here (no GPU needed): ncu -i reads the report offline.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_bytes.sum": "l2_bytes",
    "lts__t_sectors_srcunit_tex_op_read.sum": "l2_read_sectors_from_sm",
    "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum": "l2_read_hit_sectors",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct_alt",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "sm__cycles_elapsed.avg": "sm_cycles",
    "smsp__cycles_active.avg": "smsp_cycles_active",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_hz",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active": "dmma_pipe_pct_of_active",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active": "hmma_pipe_pct_of_active",
}
UNIT = {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-9, "usecond": 1e-6,
        "msecond": 1e-3, "second": 1.0, "Ghz": 1e9, "Mhz": 1e6, "hz": 1.0}


def raw(rep):
    """Header, units and rows of an ncu --page raw --csv export: read from a
    .csv made on the GPU box (`ncu -i X.ncu-rep --page raw --csv > X.csv`; a
    full-set report of many launches is too large to bring back) or exported
    here from a .ncu-rep."""
    if rep.endswith(".csv"):
        text = "".join(ln for ln in open(rep) if not ln.startswith("=="))
    else:
        text = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                              check=True).stdout
    rows = list(csv.reader(io.StringIO(text)))
    return rows[0], rows[1], rows[2:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--workload", required=True)
    ap.add_argument("--tag", required=True)
    ap.add_argument("--flops", type=float)
    ap.add_argument("--staging", default="cpasync", help="DMMA kernel staging the capture ran with")
    ap.add_argument("--model-bytes", type=float)
    ap.add_argument("--launches-per-step", type=int, default=1,
                    help="task-kernel launches in one step of the workload (TMA segments): the first N kernels "
                         "matching --kernel-regex in the capture are summed into *_per_step")
    ap.add_argument("--kernel-regex", default=r"k_dmma|k_tc|k_simt", help="which captured kernels are task kernels")
    ap.add_argument("--kernel-id", default=None, help="library kernel id the capture ran (default: the local build)")
    ap.add_argument("--blocksizes", default=None, help="JSON of the plan's blocksizes (bench config.blocksizes)")
    ap.add_argument("--out-dir", default=os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                      "profiles"))
    a = ap.parse_args()
    hdr, units, data = raw(a.rep)
    kernels = []
    for row in data:
        k = {"kernel": row[hdr.index("Kernel Name")]}
        for name, short in KEYS.items():
            if name in hdr:
                i = hdr.index(name)
                v = row[i].replace(",", "")
                try:
                    k[short] = float(v) * UNIT.get(units[i], 1.0)
                except ValueError:
                    pass
        stalls = {}
        for i, name in enumerate(hdr):
            if name.startswith("smsp__average_warps_issue_stalled_") and name.endswith("_per_issue_active.ratio"):
                try:
                    val = float(row[i])
                except ValueError:
                    continue
                if val >= 0.01:
                    stalls[name[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = val
        k["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
        if "dram_read" in k and "dram_write" in k:
            k["dram_bytes"] = k["dram_read"] + k["dram_write"]
        kernels.append(k)
    import re

    task = [k for k in kernels if re.search(a.kernel_regex, k["kernel"])]
    if len(task) < a.launches_per_step:
        raise SystemExit(f"capture holds {len(task)} task-kernel launches, fewer than --launches-per-step "
                         f"{a.launches_per_step}")
    step = task[:a.launches_per_step]
    top = step[0]
    bid = a.kernel_id
    if bid is None:
        import sys

        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from paper_1904_05717_b200 import _native

        bid = _native.kernel_id()
    per_step = {
        "launches_per_step": a.launches_per_step,
        "dram_bytes_per_step": sum(k.get("dram_bytes", 0.0) for k in step),
        "duration_s_per_step_under_ncu": sum(k.get("duration", 0.0) for k in step),
        "l2_read_sectors_from_sm_per_step": sum(k.get("l2_read_sectors_from_sm", 0.0) for k in step),
    }
    summary = {
        "workload": a.workload,
        "tag": a.tag,
        "staging": a.staging,
        "report": os.path.basename(a.rep),
        "kernel_id": bid,
        "blocksizes": json.loads(a.blocksizes) if a.blocksizes else None,
        **per_step,
        "kernel": top["kernel"],
        "duration_s_under_ncu": top.get("duration"),
        "dram_bytes_per_launch": per_step["dram_bytes_per_step"] / a.launches_per_step,
        "tensor_pipe_pct": top.get("tensor_pipe_pct", top.get("tensor_pipe_pct_alt")),
        "kernels": kernels,
        "note": "ncu per-launch times are serialised and cold-cache (clock-control none); compare shares, "
                "not absolutes, with bench.py's CUDA-event numbers",
    }
    if a.flops and per_step["duration_s_per_step_under_ncu"]:
        summary["tflops_under_ncu"] = a.flops / per_step["duration_s_per_step_under_ncu"] / 1e12
    if a.model_bytes and per_step["dram_bytes_per_step"]:
        summary["model_hbm_bytes"] = a.model_bytes
        summary["measured_over_model"] = per_step["dram_bytes_per_step"] / a.model_bytes
    if a.launches and os.path.exists(a.launches):
        lines = [ln for ln in open(a.launches) if not ln.startswith("==")]
        rows = list(csv.reader(io.StringIO("".join(lines))))
        h = rows[0]
        ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
        launches = [(r[ki], float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)) for r in rows[1:] if len(r) > vi]
        tot = sum(t for _, t in launches)
        by = {}
        for name, t in launches:
            short = name.split("(")[0].replace("void ", "").replace("mmm::gpu::<unnamed>::", "")
            d = by.setdefault(short, {"launches": 0, "seconds": 0.0})
            d["launches"] += 1
            d["seconds"] += t
        for d in by.values():
            d["share"] = d["seconds"] / tot if tot else None
        summary["launch_list"] = {"total_seconds": tot, "by_kernel": by, "source": os.path.basename(a.launches)}
    os.makedirs(a.out_dir, exist_ok=True)
    path = os.path.join(a.out_dir, f"ncu_summary_{a.tag}.json")
    json.dump(summary, open(path, "w"), indent=1)
    print(path)
    print(json.dumps({k: v for k, v in summary.items() if k not in ("kernels", "launch_list")}, indent=1))


if __name__ == "__main__":
    main()
