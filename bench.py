#!/usr/bin/env python
"""Benchmark of the hot path: one FP64 multilevel-blocked C += A·B per step.

Workload (BASELINE.json configs[1], the largest square of the sweep that the
metric is quoted on): m = n = k = 16384, FP64, column-major, A, B, C
uniform[-1,1) from a seeded counter-based generator on the device (synthetic;
the reference has no dataset), family member C2A1C0 lowered with the fused
schedule onto the DMMA task kernel. Inputs are 6.4 GB (> 126 MB L2), so no
L2 flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One JSON line from rank 0. `value` = whole-job TFLOP/s with inputs resident
in HBM (CUDA events on the launch stream, max over ranks); `e2e` = the same
metric through the C ABI's host-buffer entry (tm_execute_host: pinned host
A,B,C copied in, C copied out, inside the timed region); `roofline` = the
task kernel's achieved FLOP/s over the FP64 DMMA peak measured live on this
device; `cpu_baseline` = the reference's own execute() (oracle/_ref, built
from the unmodified reference headers, -O2) on the host cores, on a bounded
sub-problem. `--impl reference` times that same reference arm on the same
config/metric.

N > 1 (torchrun): the 2-D C partition of BASELINE configs[4] — each rank owns
a 16384 x 16384 block of C (weak scaling), A row-panels and B column-panels
are all-gathered over NCCL in k-chunks overlapped with the local GEMM.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

M = N = K = 16384
FAMILY = "C2A1C0"
METRIC = "GEMM TFLOP/s (FP64) and % of FP64 peak"  # both arms report this metric on this workload


def workload_name(m):
    return f"fp64 C+=A*B m=n=k={m} column-major, family {FAMILY} fused/DMMA"
CPU_SAMPLE = (2048, 2048, 8192)      # bounded sub-problem of the same workload for the CPU reference
CPU_SAMPLE_REF_ARM = (2048, 2048, 4096)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--size", type=int, default=M, help="square size (default 16384 = configs[1] max)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--staging", default="auto", choices=["auto", "cpasync", "tma"],
                   help="DMMA kernel staging (auto = TMA whenever it applies)")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--summa", action="store_true",
                   help="run the multi-GPU 2-D partition driver even at N=1 (exercises the N>1 code path)")
    return p.parse_args()


# ----------------------------------------------------------------- helpers
def host_hierarchy():
    """The host's cache hierarchy in FP64 elements, from sysfs (level 0 =
    64 register elements as in the reference's CPU configs)."""
    caps = [64]
    base = "/sys/devices/system/cpu/cpu0/cache"
    sizes = {}
    try:
        for idx in sorted(os.listdir(base)):
            if not idx.startswith("index"):
                continue
            d = os.path.join(base, idx)
            typ = open(os.path.join(d, "type")).read().strip()
            lvl = int(open(os.path.join(d, "level")).read().strip())
            if typ == "Instruction":
                continue
            s = open(os.path.join(d, "size")).read().strip()
            mult = {"K": 1024, "M": 1024 * 1024}.get(s[-1], 1)
            sizes[lvl] = int(s.rstrip("KM")) * mult
    except OSError:
        sizes = {1: 48 * 1024, 2: 2 * 1024 * 1024, 3: 32 * 1024 * 1024}
    for lvl in sorted(sizes):
        caps.append(sizes[lvl] // 8)
    return caps


def cpu_reference_run(shape, reps, workers):
    """The reference's own execute() (oracle/_ref) on host buffers; returns
    (TFLOP/s, seconds per rep, blocksizes)."""
    from oracle import oracle as O

    if not O.have_ref():
        raise FileNotFoundError("oracle/_ref/libtilemul_ref.so not built")
    m, n, k = shape
    caps = host_hierarchy()
    rc, bs = O.ref_derive(FAMILY, caps, shape)
    if rc != 0:
        raise RuntimeError(f"reference derive failed: {bs}")
    a, b, c = O.fill_uniform(7, [(m, k), (k, n), (m, n)])
    secs = []
    for _ in range(reps):
        secs.append(O.ref_execute(FAMILY, caps, shape, bs, a, b, c, workers=workers))
    t = statistics.median(secs)
    return 2.0 * m * n * k / t / 1e12, t, bs, caps


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def ncu_traffic(workload, staging="cpasync"):
    """Per-launch DRAM bytes of the task kernel from the committed ncu
    --set full summary of this workload and staging (profiles/), or None."""
    for name in sorted(os.listdir(os.path.join(ROOT, "profiles")), reverse=True) if os.path.isdir(
            os.path.join(ROOT, "profiles")) else []:
        if name.startswith("ncu_summary") and name.endswith(".json"):
            try:
                d = json.load(open(os.path.join(ROOT, "profiles", name)))
            except (OSError, ValueError):
                continue
            if d.get("workload") == workload and d.get("staging", "cpasync") == staging and d.get(
                    "dram_bytes_per_launch"):
                return d["dram_bytes_per_launch"], name
    return None, None


# ------------------------------------------------------------ reference arm
def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    workers = os.cpu_count() or 1
    shape = CPU_SAMPLE_REF_ARM
    from oracle import oracle as O

    if not O.have_ref():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtilemul_ref.so was not built"}))
        return 0
    for _ in range(args.warmup):
        cpu_reference_run(shape, 1, workers)
    times = []
    for _ in range(args.steps):
        tf, t, bs, caps = cpu_reference_run(shape, 1, workers)
        times.append(t)
    total = sum(times)
    flops = 2.0 * shape[0] * shape[1] * shape[2]
    value = flops * len(times) / total / 1e12
    sample = (f"reference execute() {FAMILY} on the {shape[0]}x{shape[1]}x{shape[2]} sub-problem of the "
              f"{M}^3 workload per step, host-derived blocksizes {sorted(bs.items())}, -O2 reference build")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args.size), "sample": list(shape)},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": workers, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))
    return 0


# ------------------------------------------------------------------ our arm
def make_plan(T, m, n, k, tile=128):
    """C2A1C0 on the B200 hierarchy with the L2 level at its effective
    capacity for residency (planner.L2_EFFECTIVE, measured), blocksizes from
    the reference's derivation with the GPU pins (planner.derive_for_gpu)."""
    from paper_1904_05717_b200 import planner as P

    hier = P.gpu_hierarchy_effective(tile)
    bs = P.derive_for_gpu(FAMILY, (m, n, k), hier, (tile, tile))
    return T.build_plan(T.parse_name(FAMILY), bs, hier, T.Shape(m, n, k)), bs, hier


def our_arm(args):
    import torch
    import torch.distributed as dist

    from paper_1904_05717_b200 import tilemul as T

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1 or args.summa:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29541")
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
        from paper_1904_05717_b200 import multigpu

        return multigpu.bench(args, T, make_plan, world, rank, local)

    m = n = k = args.size
    nest, bs, hier = make_plan(T, m, n, k)
    stream = torch.cuda.current_stream()
    A = torch.empty(m * k, dtype=torch.float64, device="cuda")
    B = torch.empty(k * n, dtype=torch.float64, device="cuda")
    C = torch.empty(m * n, dtype=torch.float64, device="cuda")
    T.fill_uniform_device(A, 1)
    T.fill_uniform_device(B, 2)
    T.fill_uniform_device(C, 3)
    # auto split_k: only the last partial wave's tiles are k-split (tail split)
    opts = T.ExecOptions(numerics="dmma", schedule="fused", split_k=0, staging=args.staging)
    for _ in range(args.warmup):
        T.execute(nest, A, B, C, opts)
    torch.cuda.synchronize()
    launches_per_step = nest.last_launch()["launches"]
    staging = nest.last_launch()["staging"]
    kernel_name = ("k_dmma_tma<BM=128,BN=128,BK=32,WM=32,WN=32,stages=3> (16 warps, TMA 128B-swizzled slabs"
                   + (f"; {launches_per_step} launches per step, segments of whole rounds" if launches_per_step > 1 else "")
                   + ")" if staging == "tma" else
                   "k_dmma<BM=128,BN=128,BK=32,WM=32,WN=32,stages=3,vec16> (16 warps, cp.async)")

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for i in range(args.steps):
            ev[i][0].record(stream)
            T.execute(nest, A, B, C, opts)
            ev[i][1].record(stream)
        t_end.record(stream)
        torch.cuda.synchronize()
    total_ms = t_start.elapsed_time(t_end)
    step_ms = [s.elapsed_time(e) for s, e in ev]
    flops = 2.0 * m * n * k
    value = flops * args.steps / (total_ms * 1e-3) / 1e12
    kernel_ms = sum(step_ms) / len(step_ms)  # per step: the task kernel (+ a tile reduction when tail-split)
    achieved = flops / (kernel_ms * 1e-3) / 1e12

    peak = T.measure_fp64_peak(30)
    workload = workload_name(m)
    traffic, traffic_src = ncu_traffic(workload, staging)
    model = nest.model()
    hbm_model_bytes = model.at_level(hier.top_level()).total_bytes()

    # ---- e2e: host buffers through the C ABI, copies inside the timed region
    e2e = None
    if not args.no_e2e:
        Ah = A.cpu().pin_memory().numpy()
        Bh = B.cpu().pin_memory().numpy()
        Ch = C.cpu().pin_memory().numpy()
        T.execute(nest, Ah, Bh, Ch, opts)  # warm (allocates the plan's device buffers)
        e2e_steps = max(1, min(args.steps, 3))
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            T.execute(nest, Ah, Bh, Ch, opts)
        dt = (time.perf_counter() - t0) / e2e_steps
        e2e = {"value": flops / dt / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": 8 * (m * k + k * n + m * n),
               "d2h_bytes_per_step": 8 * m * n, "ms_per_step": dt * 1e3,
               "path": "tm_execute_host (pinned host A,B,C -> device, C back; one persistent launch fed by the copy engine)"}
        del Ah, Bh, Ch

    # ---- CPU baseline: the reference's execute() on the host cores
    cpu = None
    if not args.no_cpu:
        try:
            workers = os.cpu_count() or 1
            tf, t, cbs, caps = cpu_reference_run(CPU_SAMPLE, 3, workers)
            cpu = {"value": tf, "unit": "TFLOP/s", "cores": workers, "kind": "reference",
                   "sample": f"reference execute() {FAMILY}, {CPU_SAMPLE[0]}x{CPU_SAMPLE[1]}x{CPU_SAMPLE[2]} "
                             f"sub-problem of the same workload, median of 3 ({t:.2f} s each), host hierarchy "
                             f"{caps} elements, -O2 unmodified reference headers"}
        except Exception as exc:  # reported, never silently replaced
            cpu = {"value": None, "unit": "TFLOP/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    out = {
        "metric": METRIC,
        "value": value, "unit": "TFLOP/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded counter-based uniform[-1,1) on device)",
        "config": {"workload": workload, "m": m, "n": n, "k": k, "family": FAMILY,
                   "blocksizes": {f"{lv}:{d}": v for (lv, d), v in bs.entries()},
                   "schedule": "fused", "numerics": "dmma (mma.sync m8n8k4 f64)", "cta_tile": "128x128",
                   "staging": staging,
                   "split_k": "auto (tail split of the last partial wave)",
                   "l2_flush": "not needed: inputs 6.4 GB > 126 MB L2", "parallelism": "1 GPU",
                   "hierarchy_elements": [hier.capacity(i) for i in range(hier.size())],
                   "l2_effective_fraction": 0.25},
        "pct_of_fp64_peak": 100.0 * value / peak,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "peak_source": "FP64 DMMA issue-rate probe run live in this bench (MEASURED_PEAKS.json has no "
                                    "FP64 figure); nominal 148 SM x 64 FMA/clk x 1.965 GHz = 37.2",
                     "kernel": kernel_name, "algorithmic_flops_per_launch": flops / launches_per_step,
                     "algorithmic_flops_per_step": flops, "launches_per_step": launches_per_step,
                     "traffic_source": traffic_src},
        "model": {"hbm_bytes_model": hbm_model_bytes,
                  "hbm_bytes_measured": traffic,
                  "measured_over_model": (traffic / hbm_model_bytes) if traffic else None},
        "e2e": e2e,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "gpu_launches": launches_per_step * args.steps,
        "step_ms": step_ms,
    }
    print(json.dumps(out))
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    return our_arm(args)


if __name__ == "__main__":
    sys.exit(main())
