"""Generates the golden fixtures in tests/golden/ from the REFERENCE ITSELF
(oracle/_ref/libtilemul_ref.so = /root/reference/proj/include compiled
unmodified). Run in the container that has /root/reference:

    python tests/golden/make_golden.py

config1_2048.json — BASELINE config 1: FP64 2048^3, mt19937_64(12345)
  uniform(-1,1) A then B, C = 0, family member C2A1C0 executed by the
  reference's execute() (bitwise equal to reference_gemm here).
  Stores checksums, 4096 sampled entries and their (|A||B|)_ij.
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


if __name__ == "__main__":
    host_cases()
    config1()
