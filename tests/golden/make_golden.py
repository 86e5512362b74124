"""Generates the golden fixtures in tests/golden/ from the REFERENCE ITSELF
(oracle/_ref/libtilemul_ref.so = /root/reference/proj/include compiled
unmodified). Run in the container that has /root/reference:

    python tests/golden/make_golden.py

config1_2048.json — BASELINE config 1: FP64 2048^3, mt19937_64(12345)
  uniform(-1,1) A then B, C = 0, family member C2A1C0 executed by the
  reference's execute() (bitwise equal to reference_gemm here).
  Stores checksums, 4096 sampled entries and their (|A||B|)_ij.
cachesim_cases.json — reference LruSimulator / simulate / generate_trace
  outputs (seeded event lists, acceptance and unit nests, random plans).
host_cases.json — reference outputs of parse_name / derive_blocksizes /
  validate_blocksizes / nest_steps / multilevel_cost on seeded random
  configurations, for the host-library parity tests where _ref is absent.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402

GPU_HIER = [128 * 128, 232448 // 8, 132644864 // 8]  # B200: CTA tile, smem opt-in, L2 (FP64 elements)


def config1():
    m = n = k = 2048
    a, b = O.fill_uniform(12345, [(m, k), (k, n)], lib_=O.ref())
    rc, bs = O.ref_derive("C2A1C0", GPU_HIER, (m, n, k), mr=128, nr=128, pinned={(1, "m"): 128})
    assert rc == 0, bs
    c = np.zeros(m * n)
    secs = O.ref_execute("C2A1C0", GPU_HIER, (m, n, k), bs, a, b, c, workers=os.cpu_count() or 1)
    rng = np.random.default_rng(2048)
    ii = rng.integers(0, m, 4096)
    jj = rng.integers(0, n, 4096)
    _, ab = O.entries(k, a, m, b, k, None, m, ii, jj)
    out = {
        "what": "reference execute(), C2A1C0, FP64 2048^3, seed 12345, C=0",
        "reference_seconds": secs,
        "A": a[:3].tolist() + [a[-1]], "B": b[:3].tolist() + [b[-1]],
        "C0": c[0], "C1": c[1], "Clast": c[-1],
        "sum_abs": float(sum(abs(x) for x in c)),  # sequential index-order sum
        "max_abs": float(np.abs(c).max()),
        "gpu_hierarchy": GPU_HIER,
        "gpu_blocksizes": [[lv, d, v] for (lv, d), v in sorted(bs.items())],
        "sample_i": ii.tolist(), "sample_j": jj.tolist(),
        "sample_c": c[ii + jj * m].tolist(), "sample_absprod": ab.tolist(),
    }
    json.dump(out, open(os.path.join(HERE, "config1_2048.json"), "w"))
    print("config1: C0", c[0], "secs", secs)


def host_cases():
    sys.path.insert(0, os.path.join(os.path.dirname(HERE)))
    import helpers as H  # tests/helpers.py (random generators)
    rng = np.random.default_rng(4242)
    cases = []
    names = ["C2A1C0", "B2A1C0", "A2B1C0", "C2B1C0", "A2C0", "B2C0", "A1C0", "B1C0", "C0", "B3A2C0", "C3A2C0",
             "A3B2C0", "C4A2C0", "A3C0", "B3A1C0", "C3B1C0"]
    hiers = [[64, 8192, 32768, 786432], [64, 6144, 262144, 13762560], GPU_HIER + [GPU_HIER[-1] * 8],
             [16, 512, 4096, 65536, 1 << 22]]
    for t in range(160):
        name = names[t % len(names)]
        caps = hiers[int(rng.integers(0, len(hiers)))]
        top = int(name[-3]) if len(name) > 2 else 0
        if top >= len(caps):
            caps = hiers[3]
        shape = tuple(int(x) for x in rng.integers(1, 5000, size=3))
        mr, nr = [(4, 12), (8, 6), (2, 2), (128, 128), (16, 8)][t % 5]
        if mr * nr > caps[0]:
            mr, nr = 4, 8
        slack = [1 / 16, 0.0, 0.25][t % 3]
        betas = [(1, 1, 1), (1, 2, 1), (2, 1, 3)][t % 3]
        inclusive = [int(x) for x in rng.integers(0, 2, size=len(caps))] if t % 4 == 0 else [0] * len(caps)
        pinned = {}
        if t % 7 == 0:
            pinned = {(1, "m"): mr * 2} if name.endswith("A1C0") else {}
        rc, bs = O.ref_derive(name, caps, shape, slack=slack, mr=mr, nr=nr, betas=betas, pinned=pinned,
                              inclusive=inclusive)
        case = {"name": name, "caps": caps, "inclusive": inclusive, "shape": shape, "slack": slack, "mr": mr,
                "nr": nr, "betas": betas, "pinned": [[l, d, v] for (l, d), v in pinned.items()], "derive_rc": rc}
        if rc == 0:
            case["blocksizes"] = [[l, d, v] for (l, d), v in sorted(bs.items())]
            loops, cells = O.ref_nest(name, caps, shape, bs, inclusive=inclusive)
            case["loops"] = [list(x) for x in loops]
            case["cells"] = cells
            case["model"] = O.ref_cost(name, caps, shape, bs, inclusive=inclusive).tolist()
            # a perturbed set for validate_blocksizes
            bad = dict(bs)
            key = sorted(bad)[int(rng.integers(0, len(bad)))]
            bad[key] = bad[key] * int(rng.integers(2, 9))
            n, rules = O.ref_validate(name, caps, shape, bad, inclusive=inclusive)
            case["perturbed"] = [[l, d, v] for (l, d), v in sorted(bad.items())]
            case["perturbed_rules"] = [list(r) for r in rules]
        else:
            case["error"] = bs
        cases.append(case)
    json.dump(cases, open(os.path.join(HERE, "host_cases.json"), "w"))
    print("host cases:", len(cases), "derive ok:", sum(c["derive_rc"] == 0 for c in cases))


def _roomy_caps(top):
    return [(1 << 20) * 4 ** h for h in range(top + 1)]


def cachesim_cases():
    """Reference LruSimulator / simulate / generate_trace outputs:
    * events: seeded random event lists over random hierarchies (regenerated
      in the test from the seed by helpers.random_sim_case; a checksum guards
      against generator drift);
    * plans: the acceptance-suite nests (criteria 2, 4, 5), the desk-scale
      B3A2C0 and two-level Resident C unit cases, and seeded random plans;
    * traces: event-stream hashes of seeded random plans, both layouts."""
    import hashlib
    sys.path.insert(0, os.path.join(os.path.dirname(HERE)))
    import helpers as H
    out = {"events": [], "plans": [], "traces": []}
    for seed in range(60):
        c = H.random_sim_case(seed)
        stats, ev = O.ref_sim_events(c["levels"], c["shape"], c["ops"], c["idx"], c["writes"],
                                     c["include_registers"], c["flush"])
        out["events"].append({"seed": seed, "checksum": int(sum((i + 1) * (v + 7) for i, v in enumerate(c["idx"]))),
                              "stats": stats, "events": ev})

    def plan(label, name, caps, shape, bs, sim_levels, packed=False):
        case = {"label": label, "name": name, "caps": caps, "shape": list(shape),
                "bs": [[l, d, v] for (l, d), v in sorted(bs.items())], "sim_levels": sim_levels, "packed": packed}
        try:
            case["stats"], case["events"] = O.ref_simulate(name, caps, shape, bs, sim_levels, packed=packed)
        except ValueError as e:  # e.g. packed layouts whose same-axis steps do not divide
            case["error"] = str(e)
        out["plans"].append(case)

    for lbl, name, shape, bs, reg in [
            ("criterion2_resident_C", "C0", (96, 96, 768), {(0, "m"): 96, (0, "n"): 96}, 9216),
            ("criterion2_resident_A", "A1C0", (96, 768, 96), {(1, "m"): 96, (1, "k"): 96, (0, "n"): 1, (0, "m"): 96}, 128),
            ("criterion2_resident_B", "B1C0", (768, 96, 96), {(1, "k"): 96, (1, "n"): 96, (0, "m"): 1, (0, "n"): 96}, 128)]:
        caps = [reg, 10240]
        plan(lbl, name, caps, shape, bs, [(reg, 1, False, True, True), (10240, 1, False, False, True)])
    plan("criterion4_right_resident", "C0", [4096, 8192], (64, 64, 1024), {(0, "m"): 64, (0, "n"): 64},
         [(1, 1, False, True, True), (4096, 1, False, False, True)])
    c5 = [(64, 1, False, True, True), (2048, 1, False, False, True), (49152, 1, False, False, True)]
    plan("criterion5_b_outer", "B2A1C0", [64, 2048, 49152], (816, 816, 816),
         {(2, "n"): 204, (2, "k"): 192, (1, "m"): 24, (1, "k"): 48, (0, "n"): 12, (0, "m"): 4}, c5, packed=True)
    plan("criterion5_goto", "A1C0", [64, 2048, 49152], (816, 816, 816),
         {(1, "m"): 24, (1, "k"): 48, (0, "n"): 12, (0, "m"): 4, (2, "n"): 660}, c5, packed=True)
    desk = [(16, 1, False, True, True), (512, 1, False, False, True), (2048, 1, False, False, True),
            (49152, 1, False, False, True)]
    plan("unit_desk_scale_B3A2C0", "B3A2C0", [16, 512, 2048, 49152], (384, 384, 384),
         {(3, "n"): 192, (3, "k"): 192, (2, "m"): 24, (2, "k"): 48, (0, "n"): 6, (0, "m"): 2}, desk, packed=True)
    plan("unit_two_level_resident_C", "C0", [2304, 2560], (48, 48, 384), {(0, "m"): 48, (0, "n"): 48},
         [(2304, 1, False, True, True), (2560, 1, False, False, True)])
    for seed in range(40):
        p = H.random_sim_plan(1000 + seed)
        bs = {(l, d): v for l, d, v in p["bs"]}
        plan(f"random_{1000 + seed}", p["name"], _roomy_caps(p["top"]), p["shape"], bs, p["sim_levels"],
             packed=p["packed"])
    for seed in range(12):
        p = H.random_sim_plan(2000 + seed)
        bs = {(l, d): v for l, d, v in p["bs"]}
        for packed in (False, True):
            try:
                ops, idx, wr, n = O.ref_trace(p["name"], _roomy_caps(p["top"]), p["shape"], bs, packed=packed)
            except ValueError as e:
                out["traces"].append({"seed": 2000 + seed, "packed": packed, "error": str(e)})
                continue
            h = hashlib.sha256(ops.encode() + idx.astype("<i8").tobytes() + wr.tobytes()).hexdigest()
            out["traces"].append({"seed": 2000 + seed, "packed": packed, "count": n, "sha256": h,
                                  "head": [[ops[i], int(idx[i]), int(wr[i])] for i in range(min(24, len(ops)))]})
    json.dump(out, open(os.path.join(HERE, "cachesim_cases.json"), "w"))
    print("cachesim:", len(out["events"]), "event cases,", len(out["plans"]), "plans,", len(out["traces"]), "traces")


def pareto_cases():
    """Reference pareto_sweep outputs over seeded cache sizes, ratios and shapes."""
    rng = np.random.default_rng(77)
    out = []
    for t in range(24):
        outer = int(rng.choice([4096, 49152, 262144, 786432, 1 << 22]))
        ratios = sorted(set(float(x) for x in rng.choice([1.5, 2, 4, 8, 16, 24, 64, 256], size=3)))
        shape = tuple(int(x) for x in rng.integers(64, 8192, size=3))
        slack = [1 / 16, 0.0, 0.25][t % 3]
        mr, nr = [(4, 12), (8, 6), (2, 2)][t % 3]
        case = {"outer": outer, "ratios": ratios, "shape": shape, "slack": slack, "mr": mr, "nr": nr}
        try:
            case["points"] = [list(p) for p in O.ref_pareto(outer, ratios, shape, slack, mr, nr)]
        except ValueError as e:
            case["error"] = str(e)
        out.append(case)
    json.dump(out, open(os.path.join(HERE, "pareto_cases.json"), "w"))
    print("pareto:", len(out), "cases,", sum("error" in c for c in out), "rejected")


if __name__ == "__main__":
    which = sys.argv[1:] or ["host", "config1", "cachesim", "pareto"]
    if "host" in which:
        host_cases()
    if "config1" in which:
        config1()
    if "cachesim" in which:
        cachesim_cases()
    if "pareto" in which:
        pareto_cases()
