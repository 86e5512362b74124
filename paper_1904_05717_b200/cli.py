"""Command-line surface on the GPU, mirroring the reference CLI's `run`,
`analyze`, `simulate`, `plan`, `roofline` and `pareto` subcommands
(/root/reference/proj/tools/tilemul_main.cpp:163-229, :231-304, :306-431):
same flags where they apply,
same JSON keys, same exit codes — 0 ok, 1 validation/parse/infeasible or a
failed correctness check, 2 usage/config error (:519-535).

    python -m paper_1904_05717_b200 run --alg C2A1C0 --shape 2048 --format json
    python -m paper_1904_05717_b200 analyze --alg C2A1C0 --shape 16384 [--hier gpu.json]
    python -m paper_1904_05717_b200 simulate --alg B3A2C0 --hier h.json --shape 384 --bs 3:n=192 ...
    python -m paper_1904_05717_b200 plan --shape 65536x256x1024

Differences, by design: the hierarchy defaults to the current B200's
{CTA tile, SMEM, L2} (tilemul.gpu_hierarchy); --mr/--nr default to the
128 x 128 CTA tile; `run` verifies (when m*n*k <= --verify-max) against the
exact-numerics kernel, which is bit-identical to the reference's execute()
(tests/test_gpu_exec.py), instead of a CPU reference_gemm.
"""
from __future__ import annotations

import argparse
import json
import math
import sys

from . import planner as P
from . import tilemul as T


class ConfigError(Exception):
    pass


HIER_KEYS = {"index", "capacity_elements", "granularity", "inclusive", "write_allocate", "write_back"}


def load_hierarchy(path: str) -> T.CacheHierarchy:
    """serialize.hpp:55-92: {"levels": [{index, capacity_elements, ...}]}, unknown fields rejected."""
    try:
        j = json.load(open(path))
    except OSError:
        raise ConfigError(f"cannot open hierarchy config: {path}")
    except ValueError as e:
        raise ConfigError(f"bad JSON in {path}: {e}")
    if not isinstance(j, dict) or not isinstance(j.get("levels"), list):
        raise ConfigError("hierarchy config must be an object with a 'levels' array")
    for k in j:
        if k != "levels":
            raise ConfigError(f"unknown field '{k}' in hierarchy config")
    levels = []
    for e in j["levels"]:
        for k in e:
            if k not in HIER_KEYS:
                raise ConfigError(f"unknown field '{k}' in hierarchy level")
        if "index" not in e or "capacity_elements" not in e:
            raise ConfigError("hierarchy level needs 'index' and 'capacity_elements'")
        levels.append(T.CacheLevel(int(e["index"]), int(e["capacity_elements"]), int(e.get("granularity", 1)),
                                   bool(e.get("inclusive", False)), bool(e.get("write_allocate", True)),
                                   bool(e.get("write_back", True))))
    try:
        return T.CacheHierarchy(levels)
    except ValueError as e:
        raise ConfigError(str(e))


def parse_shape(text: str):  # tilemul_main.cpp:25-43
    parts = text.lower().split("x")
    if not all(p.isdigit() for p in parts) or len(parts) not in (1, 3):
        raise ConfigError(f"bad shape '{text}', expected MxNxK")
    v = [int(p) for p in parts]
    return T.Shape(v[0], v[0], v[0]) if len(v) == 1 else T.Shape(*v)


def parse_bs(items):  # tilemul_main.cpp:90-103
    bs = {}
    for s in items or []:
        if ":" not in s or "=" not in s or s.index("=") < s.index(":"):
            raise ConfigError(f"bad --bs '{s}', expected level:dim=value")
        lv, rest = s.split(":", 1)
        dim, val = rest.split("=", 1)
        if dim not in ("m", "n", "k"):
            raise ConfigError(f"bad --bs dimension in '{s}'")
        bs[(int(lv), dim)] = int(val)
    return bs


def defaults(a):
    # a hierarchy file means the reference's own conventions (micro tile
    # 4 x 12, tilemul_main.cpp:54); no file means the current B200 with its
    # 128 x 128 CTA tile
    if a.mr is None:
        a.mr = 4 if a.hier else 128
    if a.nr is None:
        a.nr = 12 if a.hier else 128


def resolve(a):
    defaults(a)
    hier = load_hierarchy(a.hier) if a.hier else T.gpu_hierarchy(a.mr if a.mr in (64, 128) else 128)
    shape = parse_shape(a.shape)
    if not a.alg:
        raise ConfigError("pass --alg")
    d = T.parse_name(a.alg)
    pins = T.BlocksizeSet(parse_bs(a.bs))
    if not a.hier and not a.bs:  # GPU defaults: the planner's pins
        bs = P.derive_for_gpu(a.alg, (shape.m, shape.n, shape.k), hier, (a.mr, a.nr), wave_block=True)
    else:
        bs = T.derive_blocksizes(d, hier, shape, T.AccessCosts(a.beta_a, a.beta_b, a.beta_c),
                                 T.DeriveOptions(a.slack, T.MicroTile(a.mr, a.nr)), pins)
    return d, bs, hier, shape


def emit(a, text):
    if a.out:
        open(a.out, "w").write(text)
    else:
        sys.stdout.write(text)


# What `run` checks against (the product may not load oracle/): the repo's own
# EXACT-numerics GPU kernel (DMUL then DADD per step, ascending k), which the
# GPU tests pin bitwise to the reference's execute() (tests/test_gpu_exec.py,
# tests/test_gpu_dropin.py) -- not an independent CPU oracle at run time.
VERIFY_AGAINST = ("this library's EXACT-numerics GPU kernel (bitwise equal to the reference's execute() "
                  "in the GPU parity tests), not an independent CPU oracle")


def cmd_run(a) -> int:
    import numpy as np
    import torch

    d, bs, hier, shape = resolve(a)
    nest = T.build_plan(d, bs, hier, shape)
    A, B = T.fill_seeded(a.seed, [(shape.m, shape.k), (shape.k, shape.n)])  # tilemul_main.cpp:236-242
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    dC = torch.zeros(shape.m * shape.n, dtype=torch.float64, device="cuda")
    opts = T.ExecOptions(numerics=a.numerics, schedule=a.schedule, staging=a.staging)
    T.execute(nest, dA, dB, dC.clone(), opts)  # warm: lowering + module load outside the timed window
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    T.execute(nest, dA, dB, dC, opts)
    e1.record()
    torch.cuda.synchronize()
    elapsed = e0.elapsed_time(e1) / 1e3
    verified = shape.m * shape.n * shape.k <= a.verify_max
    rel = None
    if verified:
        ref = torch.zeros_like(dC)
        T.execute(nest, dA, dB, ref, T.ExecOptions(numerics="exact", schedule="fused"))
        torch.cuda.synchronize()
        got, want = dC.cpu().numpy(), ref.cpu().numpy()
        den = float(np.sum(want * want))
        num = float(np.sum((got - want) ** 2))
        rel = math.sqrt(num / den) if den > 0 else math.sqrt(num)
    gflops = shape.flops() / elapsed / 1e9 if elapsed > 0 else 0.0
    if a.format == "json":
        emit(a, json.dumps({"algorithm": T.format_name(d), "shape": {"m": shape.m, "n": shape.n, "k": shape.k},
                            "device": torch.cuda.get_device_name(0), "numerics": a.numerics,
                            "schedule": a.schedule, "verified": verified, "rel_frobenius_error": rel,
                            "verified_against": VERIFY_AGAINST if verified else None,
                            "timing": {"elapsed_s": elapsed, "gflops": gflops}}, indent=2) + "\n")
    else:
        s = f"algorithm {T.format_name(d)}, device {torch.cuda.get_device_name(0)}\n"
        s += f"elapsed: {elapsed} s ({gflops} GFLOP/s)\n"
        s += (f"max relative error vs reference: {rel} ({VERIFY_AGAINST})\n" if verified
              else "reference check skipped (shape above --verify-max)\n")
        emit(a, s)
    if verified and rel > 1e-12:
        sys.stderr.write(f"correctness check failed: relative error {rel}\n")
        return 1
    return 0


def cmd_analyze(a) -> int:  # tilemul_main.cpp:163-177 + costmodel.hpp:163-229
    d, bs, hier, shape = resolve(a)
    rep = T.multilevel_cost(d, bs, hier, shape)
    levels = []
    for lt in rep.levels:
        levels.append({"level": lt.level, "reads": lt.reads(), "writes": lt.writes(),
                       "bytes": lt.total_bytes(),
                       "operands": {o: {"reads": lt.of(o).reads, "writes": lt.of(o).writes} for o in "ABC"}})
    out = {"algorithm": T.format_name(d), "shape": {"m": shape.m, "n": shape.n, "k": shape.k},
           "blocksizes": [{"level": lv, "dim": dd, "value": v} for (lv, dd), v in bs.entries()],
           "flops": shape.flops(), "levels": levels,
           "intensity_flops_per_byte": rep.intensity_flops_per_byte()}
    if a.format == "csv":  # serialize.hpp cost report CSV
        rows = ["level,operand,reads,writes"]
        for lt in rep.levels:
            rows += [f"{lt.level},{o},{lt.of(o).reads},{lt.of(o).writes}" for o in "ABC"]
        emit(a, "\n".join(rows) + "\n")
    else:
        emit(a, json.dumps(out, indent=2) + "\n")
    return 0


def cmd_simulate(a) -> int:  # tilemul_main.cpp:179-229 + serialize.hpp:174-235
    d, bs, hier, shape = resolve(a)
    nest = T.build_plan(d, bs, hier, shape)
    lay = T.TraceLayouts.column_major(shape) if a.colmajor_trace else T.TraceLayouts.packed(nest)
    events = T.trace_event_count(nest)
    if events > a.max_events:
        raise ConfigError(f"trace of {events} events exceeds --max-events; use a smaller shape")
    if a.trace_dump:
        try:
            out = open(a.trace_dump, "w")
        except OSError:
            raise ConfigError(f"cannot write trace to {a.trace_dump}")
        with out:
            T.generate_trace(nest, lay, lambda e: T.write_trace_event(out, e))
    sim = T.simulate(nest, lay, hier, T.SimOptions(include_registers=a.include_registers))
    rep = T.multilevel_cost(d, bs, hier, shape)
    cmp = T.compare_model(sim, rep)
    if a.format == "csv":
        rows = ["level,hits,misses,writebacks,sim_elements,model_elements,rel_error"]
        for c in cmp.levels:
            s = sim.at_level(c.level)
            rows.append(f"{c.level},{s.hits},{s.misses()},{s.writebacks},{c.sim_elements},{c.model_elements},"
                        f"{c.rel_error}")
        emit(a, "\n".join(rows) + "\n")
    elif a.format == "human":
        rows = [f"algorithm {T.format_name(d)}, {sim.events} trace events",
                "level   hits        misses      writebacks  sim elems     model elems   rel error"]
        for c in cmp.levels:
            s = sim.at_level(c.level)
            rows.append(f"  {c.level}   {s.hits}   {s.misses()}   {s.writebacks}   {c.sim_elements}   "
                        f"{c.model_elements}   {c.rel_error}")
        emit(a, "\n".join(rows) + "\n")
    else:
        model = {"shape": {"m": shape.m, "n": shape.n, "k": shape.k}, "flops": rep.flops,
                 "boundary_level": rep.boundary_level,
                 "intensity_flops_per_byte": rep.intensity_flops_per_byte(),
                 "levels": [{"level": lt.level,
                             "operands": {o: {"reads": lt.of(o).reads, "writes": lt.of(o).writes} for o in "ABC"},
                             "total_elements": lt.total_elements(), "total_bytes": lt.total_bytes()}
                            for lt in rep.levels]}
        simj = {"events": sim.events,
                "levels": [{"level": s.level, "capacity_lines": s.capacity_lines, "granularity": s.granularity,
                            "hits": s.hits, "misses": s.misses(), "read_misses": s.read_misses,
                            "write_misses": s.write_misses, "writebacks": s.writebacks,
                            "transferred_elements": s.transferred_elements()} for s in sim.levels]}
        cmpj = {"max_rel_error": cmp.max_rel_error,
                "levels": [{"level": c.level, "model_elements": c.model_elements, "sim_elements": c.sim_elements,
                            "rel_error": c.rel_error} for c in cmp.levels]}
        emit(a, json.dumps({"algorithm": T.format_name(d), "simulation": simj, "model": model, "comparison": cmpj},
                           indent=2, default=lambda x: None if x == float("inf") else x) + "\n")
    return 0


def _num(x: float) -> str:  # std::ostream's default formatting (6 significant digits)
    return f"{x:g}"


def cmd_roofline(a) -> int:  # tilemul_main.cpp:355-388
    rows, csv = [], ["name,intensity_flops_per_byte,bound_flops_per_s,regime"]
    for p in a.point or []:
        if "=" not in p:
            raise ConfigError(f"bad --point '{p}', expected name=intensity")
        name, val = p.split("=", 1)
        try:
            intensity = float(val)
        except ValueError:
            raise ConfigError(f"bad --point '{p}', expected name=intensity")
        bound = T.roofline_bound(intensity, a.peak, a.bw)
        regime = "compute-bound" if intensity * a.bw >= a.peak else "bandwidth-bound"
        csv.append(f"{name},{_num(intensity)},{_num(bound)},{regime}")
        rows.append({"name": name, "intensity_flops_per_byte": intensity, "bound_flops_per_s": bound, "regime": regime})
    breakpoint_ = a.peak / a.bw
    csv.append(f"_breakpoint,{_num(breakpoint_)},{_num(a.peak)},breakpoint")
    if a.format == "json":
        emit(a, json.dumps({"peak_flops_per_s": a.peak, "bandwidth_bytes_per_s": a.bw,
                            "breakpoint_intensity": breakpoint_, "points": rows}, indent=2) + "\n")
    else:
        emit(a, "\n".join(csv) + "\n")
    return 0


def cmd_pareto(a) -> int:  # tilemul_main.cpp:390-431
    shape = parse_shape(a.shape)
    try:
        ratios = [float(x) for x in a.ratios.split(",") if x]
    except ValueError:
        raise ConfigError(f"bad --ratios '{a.ratios}'")
    if not ratios:
        raise ConfigError("--ratios needs at least one value")
    pts = T.pareto_sweep(a.cache, ratios, shape,
                         T.DeriveOptions(a.slack, T.MicroTile(a.mr if a.mr else 4, a.nr if a.nr else 12)))
    keys = ["ratio", "inner_capacity", "outer_block_k", "outer_block_n", "inner_block_m", "inner_block_k",
            "eff_outer_flops_per_element", "eff_inner_flops_per_element"]
    if a.format == "json":
        emit(a, json.dumps({"outer_capacity": a.cache, "points": [{k: getattr(p, k) for k in keys} for p in pts]},
                           indent=2) + "\n")
    else:
        lines = [",".join(keys)] + [",".join(_num(getattr(p, k)) if isinstance(getattr(p, k), float)
                                             else str(getattr(p, k)) for k in keys) for p in pts]
        emit(a, "\n".join(lines) + "\n")
    return 0


def cmd_plan(a) -> int:  # tilemul_main.cpp:306-360, re-targeted (planner.py)
    defaults(a)
    shape = parse_shape(a.shape)
    hier = load_hierarchy(a.hier) if a.hier else T.gpu_hierarchy(128)
    nest, pick, ranked = P.select_for_gpu((shape.m, shape.n, shape.k), hier, (a.mr, a.nr))
    out = {"recommended": pick.name,
           "reference_select_algorithm": T.select_algorithm(shape, hier.capacity(hier.top_level())),
           "blocksizes": [{"level": lv, "dim": dd, "value": v} for (lv, dd), v in pick.blocksizes.entries()],
           "ranking": [{"algorithm": c.name, "model_bytes_into_L2": c.hbm_bytes, "model_bytes_into_SMEM": c.smem_bytes,
                        "note": c.note} for c in ranked]}
    emit(a, json.dumps(out, indent=2, default=lambda x: None if x == float("inf") else x) + "\n")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1904_05717_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("run", "analyze", "simulate", "plan"):
        p = sub.add_parser(name)
        p.add_argument("--alg")
        p.add_argument("--hier")
        p.add_argument("--shape", default="1024")
        p.add_argument("--bs", action="append")
        p.add_argument("--slack", type=float, default=1.0 / 16.0)
        p.add_argument("--beta-a", dest="beta_a", type=float, default=1.0)
        p.add_argument("--beta-b", dest="beta_b", type=float, default=1.0)
        p.add_argument("--beta-c", dest="beta_c", type=float, default=1.0)
        p.add_argument("--mr", type=int, default=None)
        p.add_argument("--nr", type=int, default=None)
        p.add_argument("--format", default="json", choices=["json", "human", "csv"])
        p.add_argument("--out")
        if name == "run":
            p.add_argument("--seed", type=int, default=12345)
            p.add_argument("--verify-max", dest="verify_max", type=int, default=1 << 27)
            p.add_argument("--numerics", default="dmma", choices=["dmma", "fma", "exact"])
            p.add_argument("--schedule", default="fused", choices=["fused", "faithful"])
            p.add_argument("--staging", default="auto", choices=["auto", "cpasync", "tma"],
                           help="DMMA kernels: how A/B k-slabs reach shared memory (auto: by measured evidence)")
            p.add_argument("--colmajor", action="store_true", help="accepted; the GPU path is column-major")
        if name == "simulate":
            p.add_argument("--trace-dump", dest="trace_dump", help="write the plain-text trace to a file")
            p.add_argument("--include-registers", dest="include_registers", action="store_true")
            p.add_argument("--colmajor-trace", dest="colmajor_trace", action="store_true",
                           help="address the trace in column-major instead of prepacked layout")
            p.add_argument("--max-events", dest="max_events", type=int, default=4 * 10 ** 9)
    r = sub.add_parser("roofline")  # tilemul_main.cpp:482-488
    r.add_argument("--peak", type=float, required=True, help="peak flops per second")
    r.add_argument("--bw", type=float, required=True, help="memory bandwidth in bytes per second")
    r.add_argument("--point", action="append", help="name=intensity_flops_per_byte (repeatable)")
    r.add_argument("--format", default="csv", choices=["json", "human", "csv"])
    r.add_argument("--out")
    q = sub.add_parser("pareto")  # tilemul_main.cpp:492-501
    q.add_argument("--cache", type=int, required=True, help="outer cache capacity in elements")
    q.add_argument("--ratios", required=True, help="comma list of capacity ratios > 1")
    q.add_argument("--shape", default="1024")
    q.add_argument("--slack", type=float, default=1.0 / 16.0)
    q.add_argument("--mr", type=int, default=4)
    q.add_argument("--nr", type=int, default=12)
    q.add_argument("--format", default="csv", choices=["json", "human", "csv"])
    q.add_argument("--out")
    a = ap.parse_args(argv)
    try:
        return {"run": cmd_run, "analyze": cmd_analyze, "simulate": cmd_simulate, "plan": cmd_plan,
                "roofline": cmd_roofline, "pareto": cmd_pareto}[a.cmd](a)
    except (T.ValidationFailure, T.ParseError, T.InfeasibleError) as e:
        sys.stderr.write(f"{e}\n")
        return 1
    except (ConfigError, ValueError, KeyError, T.CudaError) as e:
        sys.stderr.write(f"{e}\n")
        return 2


if __name__ == "__main__":
    sys.exit(main())
