#!/usr/bin/env python
"""One config through T.execute for an ncu capture: a warm-up launch, then
`--reps` profiled launches (capture with --launch-skip 1 -k regex:k_dmma).

  python tools/profile_one.py --shape 16384,16384,256 --tile 128 --tile-n 64 --staging tma
"""
from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="16384,16384,256")
    ap.add_argument("--family", default="C2A1C0")
    ap.add_argument("--tile", type=int, default=0)
    ap.add_argument("--tile-n", type=int, default=0)
    ap.add_argument("--split", type=int, default=0)
    ap.add_argument("--staging", default="auto")
    ap.add_argument("--reps", type=int, default=1)
    a = ap.parse_args()
    import torch
    from paper_1904_05717_b200 import planner, tilemul as T

    m, n, k = (int(x) for x in a.shape.split(","))
    hier = planner.gpu_hierarchy_effective(128)
    bs = planner.derive_for_gpu(a.family, (m, n, k), hier)
    nest = T.build_plan(T.parse_name(a.family), bs, hier, T.Shape(m, n, k))
    A = torch.empty(m * k, dtype=torch.float64, device="cuda")
    B = torch.empty(k * n, dtype=torch.float64, device="cuda")
    C = torch.empty(m * n, dtype=torch.float64, device="cuda")
    for x, s in ((A, 1), (B, 2), (C, 3)):
        T.fill_uniform_device(x, s)
    opts = T.ExecOptions(numerics="dmma", split_k=a.split, tile=a.tile, tile_n=a.tile_n, staging=a.staging)
    for _ in range(1 + a.reps):
        T.execute(nest, A, B, C, opts)
    torch.cuda.synchronize()
    print(nest.last_launch())


if __name__ == "__main__":
    main()
